"""Phase breakdown of the bench's e2e leg (PBKD_TRACE=1 prints engine phases)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2012_03096_b200 as P
import bench

spec, classes, images, labels, tr, ev, blocks = bench.workload("vgg16", 1000, P)
ctx = P.Context(0)
ctx.teacher_init(spec, P.mix_seed(42, 0x7E11))
ctx.dataset_load(images, labels, classes)
tw = ctx.teacher_weights(P.spec_num_floats(spec))
pin = lambda a: torch.from_numpy(a).pin_memory().numpy()
img_p, tw_p = pin(images), pin(tw)
tasks = [P.make_task(k, epochs=int(os.environ.get("EP", "1")), eval_every=1, seed=P.mix_seed(42, k), batch_size=32) for k in blocks]
for i in range(4):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    ctx.teacher_load(spec, tw_p); torch.cuda.synchronize(); t1 = time.perf_counter()
    ctx.dataset_load(img_p, labels, classes); torch.cuda.synchronize(); t2 = time.perf_counter()
    r = ctx.run(tasks, tr, ev, plan=[blocks], workers=1, policy="wfd"); torch.cuda.synchronize(); t3 = time.perf_counter()
    print(f"iter {i}: teacher_load {1e3*(t1-t0):.1f} ms, dataset_load {1e3*(t2-t1):.1f} ms, run {1e3*(t3-t2):.1f} ms", flush=True)
