import sys, numpy as np
sys.path.insert(0, '.')
import paper_2012_03096_b200 as P
B = int(sys.argv[1]); n = int(sys.argv[2]); blocks = [int(x) for x in sys.argv[3].split(",")]
spec = open("configs/resnet50_imagenet.json").read()
ctx = P.Context(0)
ctx.teacher_init(spec, 11)
img = np.random.default_rng(50).random((n, 3, 224, 224), dtype=np.float32)
lab = (np.arange(n) % 1000).astype(np.int32)
ctx.dataset_load(img, lab, 1000)
tr = np.arange(0, n - 8, dtype=np.int32); ev = np.arange(n - 8, n, dtype=np.int32)
for k in blocks:
    try:
        r = ctx.run([P.make_task(k, epochs=1, eval_every=10**6, seed=1, batch_size=B, max_steps=1)], tr, ev, flags=P.RUN_STEP_ONLY)["results"][0]
        print("block", k, "ok", r["step_losses"], flush=True)
    except Exception as e:
        print("block", k, "FAIL", e, flush=True); break
