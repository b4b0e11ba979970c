"""Precision probe: GPU teacher prefix vs float64 (tests/np_ref) per TF32 mode."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2012_03096_b200 as P
from oracle.oracle import Oracle
from tests.np_ref import prefix_f64
o = Oracle("orc")
ctx = P.Context(0)
for name in ["vgg16_cifar", "resnet18_cifar"]:
    spec = open(f"configs/{name}.json").read(); tw = o.teacher_init(spec, 5)
    ctx.teacher_load(spec, tw)
    x = np.random.default_rng(3).random((3, 3, 32, 32), dtype=np.float32)
    nb = o.teacher_num_blocks(spec)
    for k in sorted({1, 2, nb // 2, nb}):
        e = prefix_f64(spec, tw, x, k); r = o.prefix_infer(spec, tw, x, k, True)
        g = ctx.prefix_infer(x, k, True, r.size)
        print(os.environ.get("PBKD_TF32_TERMS"), name, k, "gpu", np.abs(g - e).max(), "ref", np.abs(r - e).max(), "scale", np.abs(e).max(), flush=True)
rng = np.random.default_rng(0)
for (rows, cin, cout) in [(4096, 64, 64), (4096, 512, 512), (4096, 3, 64)]:
    import torch
    x = rng.uniform(-1, 1, (rows, cin)).astype(np.float32); w = rng.uniform(-1, 1, (cout, cin)).astype(np.float32)
    xd, wd = torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda(); y = torch.zeros(rows, cout, device="cuda")
    ctx.k("pw_fwd", P.DevPtr(xd.data_ptr()), P.DevPtr(wd.data_ptr()), P.DevPtr(y.data_ptr()), rows, cin, cout, None, None)
    ex = x.astype(np.float64) @ w.astype(np.float64).T
    f32 = (x @ w.T)
    print(os.environ.get("PBKD_TF32_TERMS"), "gemm", rows, cin, cout, "gpu", np.abs(y.cpu().numpy() - ex).max(), "np32", np.abs(f32 - ex).max(), "scale", np.abs(ex).max(), flush=True)
