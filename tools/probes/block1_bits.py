"""Diagnosis: dump the grouped engine's results for VGG-16 blocks 1-3 (block 1
reads the 3-channel network input) so two library builds can be compared bit
for bit.  usage: block1_bits.py <libpbkd_b200.so> <out.npz>"""
import sys
import numpy as np
import paper_2012_03096_b200 as P

P.LIB_PATH = sys.argv[1]
from tests.conftest import spec_text  # noqa: E402

spec = spec_text("vgg16_cifar")
ctx = P.Context(0)
ctx.teacher_init(spec, P.mix_seed(42, 0x7E11))
n = 160
img = np.random.default_rng(5).random((n, 3, 32, 32), dtype=np.float32)
lab = (np.arange(n) % 10).astype(np.int32)
tr, ev = P.stratified_split(lab, 0.2, 3)
ctx.dataset_load(img, lab)
out = {}
for tag, kw in (("three", dict(kind=1)), ("two", dict())):
    tasks = [P.make_task(k, epochs=2, eval_every=1, seed=P.mix_seed(9, k), batch_size=32, **kw) for k in (1, 2, 3)]
    res = ctx.run(tasks, tr, ev)["results"]
    for r in res:
        k = r["block_index"]
        out[f"{tag}_b{k}_final"] = r["final_block"]
        out[f"{tag}_b{k}_block"] = r["block"]
        out[f"{tag}_b{k}_loss"] = np.array(r["loss_history"])
        out[f"{tag}_b{k}_eval"] = np.array([a for _, a in r["eval_history"]])
        out[f"{tag}_b{k}_steps"] = r["step_losses"]
np.savez(sys.argv[2], **out)
print("dumped", len(out))
