"""Helper for test_gpu_parity.test_gemm_kernels_agree_bitwise: runs the
pointwise GEMM entry points (pbkd_k_pw_fwd / pbkd_k_pw_bwd) and the teacher
prefix (implicit-GEMM convs) on seeded inputs and saves every output.  Run once with PBKD_GEMM_TMA=0 PBKD_CONV_TMA=0
(register-staged umma.cu kernel) and once with the defaults (TMA
umma_tma.cu kernel)."""
import sys

import numpy as np
import torch

import paper_2012_03096_b200 as P

SHAPES = [(32768, 64, 64), (8192, 64, 128), (2048, 128, 256), (512, 256, 512), (128, 512, 512),
          (1000, 20, 48), (300, 96, 40), (4096, 3, 64), (2048, 16, 16), (1000, 24, 20), (2048, 16, 32)]


def main(out):
    ctx = P.Context(0)
    res = {}
    for rows, cin, cout in SHAPES:
        rng = np.random.default_rng(rows + cin * 7 + cout * 13)
        x = torch.from_numpy(rng.uniform(-1, 1, (rows, cin)).astype(np.float32)).cuda()
        w = torch.from_numpy(rng.uniform(-1, 1, (cout, cin)).astype(np.float32)).cuda()
        gy = torch.from_numpy(rng.uniform(-1, 1, (rows, cout)).astype(np.float32)).cuda()
        y = torch.zeros(rows, cout, device="cuda")
        cs, cq = torch.zeros(cout, device="cuda"), torch.zeros(cout, device="cuda")
        gx, gw = torch.zeros(rows, cin, device="cuda"), torch.zeros(cout, cin, device="cuda")
        D = lambda t: P.DevPtr(t.data_ptr())  # noqa: E731
        ctx.k("pw_fwd", D(x), D(w), D(y), rows, cin, cout, D(cs), D(cq))
        ctx.k("pw_bwd", D(x), D(w), D(gy), D(gx), D(gw), rows, cin, cout)
        key = f"{rows}_{cin}_{cout}"
        for name, t in (("y", y), ("cs", cs), ("cq", cq), ("gx", gx), ("gw", gw)):
            res[f"{key}_{name}"] = t.cpu().numpy()
        # fp64 reference for the dump's own sanity
        xd, wd, gyd = (t.double().cpu().numpy() for t in (x, w, gy))
        yd = xd @ wd.T
        for name, want in (("y", yd), ("gx", gyd @ wd), ("gw", gyd.T @ xd), ("cs", yd.sum(0)), ("cq", (yd * yd).sum(0))):
            got = res[f"{key}_{name}"].astype(np.float64)
            err = np.max(np.abs(got - want)) / max(np.max(np.abs(want)), 1e-30)
            if err > 1e-5:
                raise SystemExit(f"{key} {name}: rel err {err:.2e} vs fp64 (max|got| {np.max(np.abs(got)):.3e}, "
                                 f"max|want| {np.max(np.abs(want)):.3e}, got[0,:4] {got.ravel()[:4]}, "
                                 f"want[0,:4] {want.ravel()[:4]})")
    # teacher implicit-GEMM convs (register-staged vs TMA 4-D im2col boxes):
    # every boundary of VGG-16 and ResNet-18 on 5 samples
    import os
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for name in ("vgg16_cifar", "resnet18_cifar"):
        spec = open(os.path.join(root, "configs", name + ".json")).read()
        ctx.teacher_init(spec, 77)
        x = np.random.default_rng(5).random((5, 3, 32, 32), dtype=np.float32)
        nb = P.spec_num_blocks(spec)
        for k in range(1, nb + 1):
            res[f"{name}_{k}"] = ctx.prefix_infer(x, k, True, 5 * 64 * 32 * 32)
    # ResNet-50 / 224x224: 56/28/14/7-pixel outputs, whose TMA conv tiles are
    # 112 or 98 rows (whole output rows / images), every bottleneck block
    spec = open(os.path.join(root, "configs", "resnet50_imagenet.json")).read()
    ctx.teacher_init(spec, 78)
    x = np.random.default_rng(6).random((2, 3, 224, 224), dtype=np.float32)
    for k in range(1, P.spec_num_blocks(spec) + 1):
        res[f"resnet50_{k}"] = ctx.prefix_infer(x, k, True, 2 * 256 * 56 * 56)
    np.savez(out, **res)


if __name__ == "__main__":
    main(sys.argv[1])
