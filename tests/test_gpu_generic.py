"""GPU parity of the layer-by-layer paths (csrc/netexec.cu, csrc/nettrain.cu)
against the REFERENCE build (golden tests/golden/toy_generic_paths.npz, made
by tests/golden/make_golden.py from oracle/_ref):

* train_block with the Combined objective  lambda*MSE + CE through the frozen
  teacher remainder (distill.cpp:57-84, :135-262), SURVEY 8f-2;
* train_block with the skip candidates TwoLayerSkip / ThreeLayerSkip
  (replacement.cpp:55-72), SURVEY 8a-11;
* reassemble + finetune, frozen and unfrozen, and train_teacher
  (distill.cpp:297-441), SURVEY 8f-1.

Tolerances: loss histories 1e-4 relative; evaluation accuracies exact
(integer counts over 10 samples); weights |gpu - ref| <= 1e-4 |ref| +
5e-4 rms(ref) per element.
"""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2012_03096_b200 as P  # noqa: E402
from tests.conftest import ROOT, spec_text  # noqa: E402

G = np.load(os.path.join(ROOT, "tests", "golden", "toy_generic_paths.npz"))
SPEC = spec_text("toy_teacher")


@pytest.fixture(scope="module")
def ctx():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    c = P.Context(0)
    c.teacher_load(SPEC, G["teacher_w"])
    c.dataset_load(G["images"], G["labels"])
    return c


def weights_close(got, want):
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    assert got.shape == want.shape
    rms = float(np.sqrt(np.mean(want * want)))
    bar = 1e-4 * np.abs(want) + 5e-4 * rms
    assert np.all(np.abs(got - want) <= bar), float(np.max(np.abs(got - want) / bar))


@pytest.mark.parametrize("name,task", [
    ("combined", dict(block=2, kind=0, seed=1234, loss_mode=1, lambda_local=0.5)),
    ("skip2", dict(block=2, kind=2, seed=99)),
    ("skip3", dict(block=3, kind=3, seed=98)),
])
def test_train_block_generic_matches_reference(ctx, name, task):
    t = P.make_task(task["block"], kind=task["kind"], epochs=2, eval_every=1, seed=task["seed"], batch_size=16,
                    lr=0.02, loss_mode=task.get("loss_mode", 0), lambda_local=task.get("lambda_local", 1.0))
    r = ctx.run([t], G["train_idx"], G["eval_idx"])["results"][0]
    assert not r["failed"], r["failure"]
    lh = G[f"{name}_loss_history"]
    assert np.all(np.abs(np.array(r["loss_history"]) - lh) <= 1e-4 * np.abs(lh)), (r["loss_history"], lh)
    eh = G[f"{name}_eval_history"]
    assert [e for e, _ in r["eval_history"]] == eh[:, 0].astype(int).tolist()
    assert np.allclose([a for _, a in r["eval_history"]], eh[:, 1]), (r["eval_history"], eh)
    assert r["best_eval"] == pytest.approx(float(G[f"{name}_best_eval"]))
    weights_close(r["block"], G[f"{name}_block"])


@pytest.mark.parametrize("name,kw", [
    ("ft_frozen", dict(epochs=2, freeze=1, lr=0.01, momentum=0.9, batch=16, seed=77, teacher_mode=False)),
    ("ft_all", dict(epochs=1, freeze=0, lr=0.01, momentum=0.9, batch=16, seed=78, teacher_mode=False)),
    ("teacher", dict(epochs=2, freeze=0, lr=0.05, momentum=0.9, batch=24, seed=900, teacher_mode=True)),
])
def test_finetune_and_teacher_training_match_reference(ctx, orc, name, kw):
    geo = {1: (3, 16, 1), 2: (16, 32, 2), 3: (32, 32, 1)}
    reps = [] if name == "teacher" else [
        (int(k), int(kind), orc.build_candidate(int(kind), *geo[int(k)], int(seed))) for k, kind, seed in G["reps"]]
    r = ctx.fit_assembled(SPEC, G["teacher_w"], reps, G["train_idx"], G["eval_idx"], **kw)
    lh = G[f"{name}_loss_history"]
    assert np.all(np.abs(r["loss_history"] - lh) <= 1e-4 * np.abs(lh)), (r["loss_history"], lh)
    assert np.allclose([a for _, a in r["eval_history"]], G[f"{name}_eval_history"])
    want = np.zeros(r["net"].size, np.float32)
    g = G[f"{name}_net"]
    want[:g.size] = g  # the golden is stored without trailing zeros
    weights_close(r["net"], want)
    if name == "ft_frozen":  # frozen teacher block 2 and the classifier stay bitwise unchanged
        base = ctx.fit_assembled(SPEC, G["teacher_w"], reps, G["train_idx"], G["eval_idx"], **{**kw, "epochs": 0})
        nb1 = reps[0][2].size
        nb2 = 16 * 32 * 9 + 4 * 32  # teacher block 2: conv + batch norm
        assert np.array_equal(r["net"][nb1:nb1 + nb2], base["net"][nb1:nb1 + nb2])
        cls = 32 * 10 + 10
        assert np.array_equal(r["net"][-cls:], base["net"][-cls:])


def test_combined_objective_is_linear_in_lambda(ctx):
    """test_distill.cpp:147-166: obj(lambda=2) = 2*obj(local) + obj(lambda=0)
    after one optimizer step (LocalOnly on the grouped path, Combined on the
    layer-by-layer path: the step losses agree to the bit)."""
    def run(mode, lam):
        t = P.make_task(2, epochs=1, eval_every=2, seed=1234, batch_size=16, lr=0.02, loss_mode=mode,
                        lambda_local=lam, max_steps=1)
        return ctx.run([t], G["train_idx"], G["eval_idx"])["results"][0]["loss_history"]
    ce_only, both, local = run(1, 0.0), run(1, 2.0), run(0, 0.0)
    assert both[1] == pytest.approx(2.0 * local[1] + ce_only[1], rel=1e-9)


def test_mixed_paths_in_one_run_match_single_runs(ctx):
    """Grouped (LocalOnly two-layer) and layer-by-layer (Combined, skip)
    tasks in one run / one run_parallel give each task's single-run bits."""
    def tasks():
        return [P.make_task(1, epochs=2, eval_every=1, seed=11, batch_size=16, lr=0.02),
                P.make_task(2, epochs=2, eval_every=1, seed=12, batch_size=16, lr=0.02, loss_mode=1,
                            lambda_local=0.5),
                P.make_task(3, kind=2, epochs=2, eval_every=1, seed=13, batch_size=16, lr=0.02)]
    alone = [ctx.run([t], G["train_idx"], G["eval_idx"])["results"][0] for t in tasks()]
    grouped = ctx.run(tasks(), G["train_idx"], G["eval_idx"])["results"]
    par = ctx.run(tasks(), G["train_idx"], G["eval_idx"], plan=[[1, 3], [2]], workers=2, policy="wfd")["results"]
    for a, b, c in zip(alone, grouped, par):
        for x in (b, c):
            assert x["block_index"] == a["block_index"] and not x["failed"]
            assert np.array_equal(x["block"], a["block"]) and x["loss_history"] == a["loss_history"]


def test_divergence_is_reported_like_the_reference(ctx, orc):
    """distill.cpp:236-244 on the grouped engine: a non-finite local loss
    (targets from a teacher block holding +inf) marks the task failed with
    the reference's message instead of throwing; the CPU restatement fails
    the same task at the same epoch and batch."""
    tw = np.array(G["teacher_w"], np.float32)
    tw[16 * 3 * 9 + 4 * 16 + 5] = np.inf  # block 2's first conv weight: boundary 2 non-finite
    ctx.teacher_load(SPEC, tw)
    try:
        t = P.make_task(2, epochs=2, eval_every=1, seed=1234, batch_size=16, lr=0.02)
        r = ctx.run([t], G["train_idx"], G["eval_idx"])["results"][0]
        from oracle.oracle import make_task as orc_task
        want = orc.train_block(SPEC, tw, G["images"], G["labels"], G["train_idx"], G["eval_idx"],
                               orc_task(2, epochs=2, eval_every=1, seed=1234, batch_size=16, lr=0.02), 1 << 16)
        assert want["failed"] and r["failed"], (want["failure"], r["failure"])
        prefix = want["failure"].split(" (loss")[0]
        assert r["failure"].startswith(prefix), (r["failure"], want["failure"])
    finally:
        ctx.teacher_load(SPEC, G["teacher_w"])
