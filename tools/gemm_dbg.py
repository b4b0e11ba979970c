"""Time the teacher conv (bench_kernel 0) and pointwise GEMM (1) under
PBKD_GEMM_DBG masks (run one process per mask)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2012_03096_b200 as P
ctx = P.Context(0)
spec = open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "configs", "vgg16_cifar.json")).read()
ctx.teacher_init(spec, 1)
for which, b in ((0, 256), (0, 900), (1, 32)):
    ms, by, fl = ctx.bench_kernel(which, b, 20)
    print(f"dbg={os.environ.get('PBKD_GEMM_DBG','0')} which={which} batch={b}: {ms*1e3:8.1f} us  {fl/ms/1e9:7.1f} TF/s  {by/ms/1e6:7.1f} GB/s", flush=True)
