"""C5 vocabulary (BASELINE configs[4]): bottleneck blocks, the
7x7 stride-2 stem with 3x3/2 max pooling, ImageNet 224x224 input.

The reference has no such blocks (parity is not pinnable against it); the
arbiter is the float64 restatement in tests/torch_f64.py:
  * teacher boundaries (prefix_infer) of a small bottleneck network
    (configs/bottleneck_demo.json, 64x64 input): GPU vs float64 within
    2e-6 of the boundary's scale (fp32-level; 3xTF32 convs);
  * student step replays on bottleneck blocks: per-step losses 1e-5
    relative, weights norm-wise 1e-4 per parameter group;
  * the full ResNet-50 / 224x224 / batch-256 shape trains (all 16
    bottleneck blocks grouped, finite losses) -- the benchmark workload.
"""
import json

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2012_03096_b200 as P  # noqa: E402
from tests.conftest import spec_text  # noqa: E402


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    return P.Context(0)


def geometry(spec):
    d = json.loads(spec)
    c, out = d["input_shape"][0], []
    for b in d["blocks"]:
        out.append((c, b["out_channels"], b.get("stride", 1)))
        c = b["out_channels"]
    return out


def test_bottleneck_prefix_matches_float64(ctx):
    from tests import torch_f64
    spec = spec_text("bottleneck_demo")
    ctx.teacher_init(spec, 5)
    tw = ctx.teacher_weights(P.spec_num_floats(spec))
    x = np.random.default_rng(3).random((4, 3, 64, 64), dtype=np.float32)
    nb = P.spec_num_blocks(spec)
    bnd = torch_f64.boundaries(spec, tw, x, nb)
    for k in range(1, nb + 1):
        want = bnd[k].cpu().numpy()
        got = ctx.prefix_infer(x, k, True, want.size).reshape(want.shape)
        err = np.abs(got - want).max() / np.abs(want).max()
        assert err < 2e-6, (k, err)


def test_bottleneck_step_replay_matches_float64(ctx, orc):
    from tests import torch_f64
    from oracle.oracle import make_task as orc_task
    spec = spec_text("bottleneck_demo")
    ctx.teacher_init(spec, 7)
    tw = ctx.teacher_weights(P.spec_num_floats(spec))
    n = 48
    img = np.random.default_rng(8).random((n, 3, 64, 64), dtype=np.float32)
    lab = (np.arange(n) % 10).astype(np.int32)
    tr, ev = P.stratified_split(lab, 0.25, 12)
    ctx.dataset_load(img, lab)
    geo = geometry(spec)
    blocks, B, steps = [2, 4, 6], 12, 5
    tasks = [P.make_task(k, epochs=2, seed=P.mix_seed(3, k), batch_size=B, max_steps=steps) for k in blocks]
    res = ctx.run(tasks, tr, ev, flags=P.RUN_STEP_ONLY)["results"]
    otasks = [orc_task(k, seed=P.mix_seed(3, k), batch_size=B) for k in blocks]
    x64 = torch_f64.replay(orc, spec, tw, img, tr, otasks, geo, steps, [steps])
    for r, (l64, snaps), k in zip(res, x64, blocks):
        assert np.all(np.abs(r["step_losses"] - l64) <= 1e-5 * l64), (k, r["step_losses"], l64)
        got, want = r["final_block"].astype(np.float64), snaps[steps]
        cin, cout, _ = geo[k - 1]
        at = 0
        for u in range(2):
            ci = cin if u == 0 else cout
            for size in (ci * 9, cout * ci, 2 * cout, 2 * cout):  # dw, pw, BN affine, BN stats
                a, b = got[at:at + size], want[at:at + size]
                assert np.linalg.norm(a - b) <= 1e-4 * np.linalg.norm(b) + 1e-12, (k, u, size)
                at += size


def test_resnet50_imagenet_shape_trains(ctx):
    spec = spec_text("resnet50_imagenet")
    ctx.teacher_init(spec, P.mix_seed(42, 0x7E11))
    n = 300
    img = np.random.default_rng(50).random((n, 3, 224, 224), dtype=np.float32)
    lab = (np.arange(n) % 1000).astype(np.int32)
    tr = np.arange(0, 280, dtype=np.int32)
    ev = np.arange(280, 300, dtype=np.int32)
    ctx.dataset_load(img, lab, 1000)
    blocks = list(range(2, 18))  # every bottleneck block (the stem is not replaceable)
    tasks = [P.make_task(k, epochs=1, eval_every=10 ** 6, seed=P.mix_seed(42, k), batch_size=256, max_steps=2)
             for k in blocks]
    res = ctx.run(tasks, tr, ev, flags=P.RUN_STEP_ONLY)["results"]
    assert [r["block_index"] for r in res] == blocks
    for r in res:
        assert not r["failed"], r["failure"]
        assert r["step_losses"].size == 2 and np.all(np.isfinite(r["step_losses"]))
        assert np.all(np.isfinite(r["final_block"]))
