"""Pins the CPU oracle (oracle/pbkd_oracle.cpp) before anything is compared to it.

* known-answer values from the reference's own tests (test_tensor_ops.cpp,
  test_scheduler.cpp, test_replacement.cpp, test_distill.cpp),
* golden fixtures generated from the reference build (tests/golden/),
* bit-for-bit agreement with the reference library itself where it is built
  (oracle/_ref, this container only).
"""
import os

import numpy as np
import pytest

from tests.conftest import spec_text

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


# ---------------------------------------------------------------- KATs ----
def test_kat_kernels(orc):
    # conv worked example: 1..9 with all-ones 3x3 -> 45; padded corner 12 (test_tensor_ops.cpp:40-56)
    x = np.arange(1, 10, dtype=np.float32).reshape(1, 1, 3, 3)
    k = np.ones((1, 1, 3, 3), np.float32)
    assert orc.conv_fwd(x, k, 1, 0).ravel()[0] == 45.0
    yp = orc.conv_fwd(x, k, 1, 1)
    assert yp[0, 0, 1, 1] == 45.0 and yp[0, 0, 0, 0] == 12.0
    # depthwise: per-channel 2x2 sums -> 10, 26 (:86-95)
    x = np.arange(1, 9, dtype=np.float32).reshape(1, 2, 2, 2)
    y = orc.dw_fwd(x, np.ones((2, 1, 2, 2), np.float32), 1, 0)
    assert y.ravel().tolist() == [10.0, 26.0]
    # pointwise: 1*1 + 2*3 = 7; stride 2 keeps top-left (:117-145)
    assert orc.pw_fwd(np.array([1, 2], np.float32).reshape(1, 2, 1, 1),
                      np.array([1, 3], np.float32).reshape(1, 2, 1, 1)).ravel()[0] == 7.0
    y = orc.pw_fwd(np.array([1, 2, 3, 4], np.float32).reshape(1, 1, 2, 2),
                   np.ones((1, 1, 1, 1), np.float32), 2)
    assert y.shape == (1, 1, 1, 1) and y.ravel()[0] == 1.0
    # batch norm moments (:147-163)
    x = np.array([1, 2, 3, 4], np.float32).reshape(1, 1, 2, 2)
    y, xhat, inv, mm, mv = orc.bn_train_fwd(x, [2.0], [1.0], [0.0], [1.0])
    ref_inv = 1.0 / np.sqrt(1.25 + 1e-5)
    assert y.ravel()[0] == pytest.approx(2 * (1 - 2.5) * ref_inv + 1, rel=1e-5)
    assert mm[0] == pytest.approx(0.25) and mv[0] == pytest.approx(0.9 + 0.125)
    assert abs(float(xhat.sum())) < 1e-5
    # MSE 2.5 and its gradient -1, -2; scale 3 (:239-257)
    s, t = np.array([1, 2], np.float32), np.array([2, 4], np.float32)
    assert orc.mse(s, t) == 2.5
    assert orc.mse_bwd(s, t).tolist() == [-1.0, -2.0]
    assert orc.mse_bwd(s, t, 3.0).tolist() == [-3.0, -6.0]
    # SGD recursion 0.8 / 2.8 / 0.52 (:259-269)
    w, v = orc.sgd([1.0], [2.0], [0.0], 0.1, 0.9)
    assert v[0] == pytest.approx(2.0) and w[0] == pytest.approx(0.8)
    w, v = orc.sgd(w, [1.0], v, 0.1, 0.9)
    assert v[0] == pytest.approx(2.8) and w[0] == pytest.approx(0.52)


def test_kat_scheduler(orc):
    five = ([1, 2, 3, 4, 5], [8.0, 7.0, 6.0, 5.0, 4.0])
    plan, mk = orc.wfd(*five, 2)  # test_scheduler.cpp:53-60
    assert plan == [[1, 4, 5], [2, 3]] and mk == 17.0
    assert orc.round_robin(five[0], 2) == [[1, 3, 5], [2, 4]]  # :32-36 (makespan 18)
    plan, _ = orc.wfd([4, 2, 3, 1], [2.0] * 4, 2)  # tie-breaking (:66-71)
    assert plan == [[1, 3], [2, 4]]
    assert orc.wfd(*five, 1)[0] == [[1, 2, 3, 4, 5]]


def test_kat_model(orc):
    toy = spec_text("toy_teacher")
    # toy total MACs 995648 (test_cli.cpp:104): 3 conv blocks + dense 32*10
    total = sum(orc.block_macs(toy, k) for k in (1, 2, 3)) + 32 * 10
    assert total == 995648
    vgg = spec_text("vgg16_cifar")
    assert orc.block_macs(vgg, 1) == 32 * 32 * 64 * 3 * 9  # test_model.cpp:209-211
    # two-layer candidate at C=64 has 2*(9*64 + 64*64) conv params (test_replacement.cpp:133-138)
    w = orc.build_candidate(0, 64, 64, 1, 1)
    assert w.size == 2 * (9 * 64 + 64 * 64) + 2 * 4 * 64
    # seed determinism and sensitivity (:82-94)
    assert np.array_equal(orc.build_candidate(3, 16, 32, 2, 77), orc.build_candidate(3, 16, 32, 2, 77))
    assert not np.array_equal(orc.build_candidate(3, 16, 32, 2, 77),
                              orc.build_candidate(3, 16, 32, 2, 78))


def test_kat_mix_seed(orc):
    assert orc.mix_seed(42, 0) != orc.mix_seed(42, 1)
    assert orc.mix_seed(42, 7) == orc.mix_seed(42, 7)


# -------------------------------------------------------------- golden ----
def test_golden_toy_train_block(orc):
    g = np.load(os.path.join(GOLD, "toy_train_block.npz"))
    toy = spec_text("toy_teacher")
    tw = orc.teacher_init(toy, 404)
    assert np.array_equal(tw, g["teacher_w"])
    img, lab = orc.synthetic_dataset(60, 11, 2)
    assert np.array_equal(img, g["images"]) and np.array_equal(lab, g["labels"])
    tr, ev = orc.stratified_split(lab, 0.2, 12)
    assert np.array_equal(tr, g["train_idx"]) and np.array_equal(ev, g["eval_idx"])
    from oracle.oracle import make_task
    task = make_task(2, epochs=4, eval_every=2, seed=1234, batch_size=16, lr=0.02)
    r = orc.train_block(toy, tw, img, lab, tr, ev, task, g["block"].size)
    assert r["loss_history"] == g["loss_history"].tolist()
    assert [list(e) for e in r["eval_history"]] == g["eval_history"].tolist()
    assert np.array_equal(r["block"], g["block"])


def test_golden_kernels(orc):
    g = np.load(os.path.join(GOLD, "c2_replay_and_kernels.npz"))
    for s in (1, 2):
        assert np.array_equal(orc.dw_fwd(g[f"dw_s{s}_x"], g[f"dw_s{s}_k"], s, 1), g[f"dw_s{s}_y"])
        gx, gk = orc.dw_bwd(g[f"dw_s{s}_x"], g[f"dw_s{s}_k"], g[f"dw_s{s}_gy"], s, 1)
        assert np.array_equal(gx, g[f"dw_s{s}_gx"]) and np.array_equal(gk, g[f"dw_s{s}_gk"])
    assert np.array_equal(orc.pw_fwd(g["pw_x"], g["pw_w"]), g["pw_y"])
    gx, gw = orc.pw_bwd(g["pw_x"], g["pw_w"], g["pw_gy"])
    assert np.array_equal(gx, g["pw_gx"]) and np.array_equal(gw, g["pw_gw"])
    y, xhat, inv, mm, mv = orc.bn_train_fwd(g["bn_x"], g["bn_gamma"], g["bn_beta"],
                                            np.zeros(8), np.ones(8))
    for a, b in [(y, "bn_y"), (xhat, "bn_xhat"), (inv, "bn_inv"), (mm, "bn_mm"), (mv, "bn_mv")]:
        assert np.array_equal(a, g[b])
    gx, gg, gb = orc.bn_train_bwd(g["bn_xhat"], g["bn_inv"], g["bn_gamma"], g["bn_gy"])
    assert np.array_equal(gx, g["bn_gx"]) and np.array_equal(gg, g["bn_gg"])
    assert np.array_equal(gb, g["bn_gb"])
    assert orc.mse(g["bn_x"], g["mse_t"]) == g["mse_loss"]
    assert np.array_equal(orc.mse_bwd(g["bn_x"], g["mse_t"]), g["mse_g"])
    assert np.array_equal(orc.conv_fwd(g["bn_x"], g["conv_k"], 2, 1), g["conv_y"])


@pytest.mark.slow
def test_golden_vgg_replay(orc):
    from oracle.oracle import make_task
    from tests.golden.make_golden import cifar_like
    g = np.load(os.path.join(GOLD, "c2_replay_and_kernels.npz"))
    vgg = spec_text("vgg16_cifar")
    tw = orc.teacher_init(vgg, orc.mix_seed(42, 0x7E11))
    img = cifar_like(40, 7)
    lab = (np.arange(40) % 10).astype(np.int32)
    tr, ev = orc.stratified_split(lab, 0.1, orc.mix_seed(42, 0x5711))
    assert np.array_equal(tr, g["vgg_train_idx"])
    for k in (2, 9):  # 64- and 512-channel blocks
        task = make_task(k, seed=orc.mix_seed(42, k), batch_size=8)
        losses, fw = orc.train_replay(vgg, tw, img, lab, tr, ev, task, 3, g[f"vgg_b{k}_final"].size)
        assert np.array_equal(losses, g[f"vgg_b{k}_losses"]), k
        assert np.array_equal(fw, g[f"vgg_b{k}_final"]), k
    # the grouped replay (teacher boundaries once per sample) gives the same bits
    tasks = [make_task(k, seed=orc.mix_seed(42, k), batch_size=8) for k in (2, 9)]
    nfs = [g["vgg_b2_final"].size, g["vgg_b9_final"].size]
    losses, _, snaps = orc.train_replay_multi(vgg, tw, img, lab, tr, ev, tasks, 3, nfs, ck_steps=[3])
    for i, k in enumerate((2, 9)):
        assert np.array_equal(losses[i], g[f"vgg_b{k}_losses"]), k
        assert np.array_equal(snaps[i][0], g[f"vgg_b{k}_final"]), k


# ---------------------------------------------------- vs the reference ----
def test_bitwise_vs_reference_ops(orc, ref):
    rng = np.random.default_rng(11)
    for (n, c, h, w, s) in [(2, 4, 8, 8, 1), (1, 3, 7, 7, 2), (2, 16, 5, 6, 2), (3, 64, 4, 4, 1)]:
        x = rng.uniform(-1, 1, (n, c, h, w)).astype(np.float32)
        k = rng.uniform(-1, 1, (c, 1, 3, 3)).astype(np.float32)
        y = orc.dw_fwd(x, k, s, 1)
        assert np.array_equal(y, ref.dw_fwd(x, k, s, 1))
        gy = rng.uniform(-1, 1, y.shape).astype(np.float32)
        for a, b in zip(orc.dw_bwd(x, k, gy, s, 1), ref.dw_bwd(x, k, gy, s, 1)):
            assert np.array_equal(a, b)
        wp = rng.uniform(-1, 1, (5, c, 1, 1)).astype(np.float32)
        assert np.array_equal(orc.pw_fwd(x, wp, s), ref.pw_fwd(x, wp, s))
        gyp = rng.uniform(-1, 1, orc.pw_fwd(x, wp, s).shape).astype(np.float32)
        for a, b in zip(orc.pw_bwd(x, wp, gyp, s), ref.pw_bwd(x, wp, gyp, s)):
            assert np.array_equal(a, b)


def test_bitwise_vs_reference_indexing(orc, ref):
    lab = (np.arange(1000) % 10).astype(np.int32)
    for seed in (1, 42, 0x5711):
        a, b = orc.stratified_split(lab, 0.1, seed), ref.stratified_split(lab, 0.1, seed)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
        assert np.array_equal(orc.shuffle(a[0], seed), ref.shuffle(a[0], seed))
    rng = np.random.default_rng(5)
    for _ in range(20):
        n, w = int(rng.integers(1, 18)), int(rng.integers(1, 9))
        wt = rng.uniform(0.5, 20, n)
        assert orc.wfd(list(range(1, n + 1)), wt, w) == ref.wfd(list(range(1, n + 1)), wt, w)


@pytest.mark.parametrize("name", ["c1_small_vgg", "resnet18_cifar", "vgg16_cifar", "resnet_blocks_demo"])
def test_bitwise_vs_reference_model(orc, ref, name):
    spec = spec_text(name)
    assert np.array_equal(orc.teacher_init(spec, 99), ref.teacher_init(spec, 99))
    nb = orc.teacher_num_blocks(spec)
    for k in range(1, nb + 1):
        assert orc.block_macs(spec, k) == ref.block_macs(spec, k)
    for kind in range(4):
        assert np.array_equal(orc.build_candidate(kind, 16, 32, 2, 5),
                              ref.build_candidate(kind, 16, 32, 2, 5))


def test_bitwise_vs_reference_prefix_resnet(orc, ref):
    spec = spec_text("resnet_blocks_demo")
    tw = orc.teacher_init(spec, 3)
    x = np.random.default_rng(2).random((3, 3, 16, 16), dtype=np.float32)
    for k in (1, 2, 3, 4):
        assert np.array_equal(orc.prefix_infer(spec, tw, x, k, True),
                              ref.prefix_infer(spec, tw, x, k, True))


def test_replay_multi_matches_single(orc):
    """orc.train_replay_multi (boundaries cached per sample, tasks threaded,
    weight checkpoints) == orc.train_replay task by task, bit for bit."""
    from oracle.oracle import make_task
    for name, seed in (("toy_teacher", 404), ("resnet_blocks_demo", 3)):
        spec = spec_text(name)
        tw = orc.teacher_init(spec, seed)
        if name == "toy_teacher":
            img, lab = orc.synthetic_dataset(50, 11, 2)
        else:
            img = np.random.default_rng(4).random((30, 3, 16, 16), dtype=np.float32)
            lab = (np.arange(30) % 10).astype(np.int32)
        tr, ev = orc.stratified_split(lab, 0.2, 12)
        nb = orc.teacher_num_blocks(spec)
        tasks = [make_task(k, seed=orc.mix_seed(7, k), batch_size=6, lr=0.02) for k in range(1, nb + 1)]
        steps = 9  # buffers of 2^18 floats, zero beyond each block's arrays on both sides
        losses, l64, snaps = orc.train_replay_multi(spec, tw, img, lab, tr, ev, tasks, steps,
                                                    [1 << 18] * nb, ck_steps=[2, steps], threads=4)
        for k in range(1, nb + 1):
            for ck in (2, steps):
                l1, fw = orc.train_replay(spec, tw, img, lab, tr, ev, tasks[k - 1], ck, 1 << 18)
                assert np.array_equal(l1, losses[k - 1][:ck]), (name, k)
                assert np.array_equal(fw, snaps[k - 1][[2, steps].index(ck)]), (name, k, ck)


def test_run_parallel_vs_reference(orc, ref):
    """orc.run_parallel == the reference's own run_parallel (runtime.cpp), bit for bit."""
    from oracle.oracle import make_task
    spec = spec_text("toy_teacher")
    tw = orc.teacher_init(spec, 2025)
    img, lab = orc.synthetic_dataset(40, 21, 2)
    tr, ev = orc.stratified_split(lab, 0.25, 3)
    tasks = [make_task(k, epochs=2, eval_every=1, seed=orc.mix_seed(99, k), batch_size=10, lr=0.02)
             for k in (1, 2, 3)]
    nfs = [orc.candidate_num_floats(0, ci, co, s) for ci, co, s in ((3, 16, 1), (16, 32, 2), (32, 32, 1))]
    a = orc.run_parallel(spec, tw, img, lab, tr, ev, tasks, [[1, 3], [2]], nfs)
    b = ref.run_parallel(spec, tw, img, lab, tr, ev, tasks, [[1, 3], [2]], nfs, policy=1)
    for x, y in zip(a, b):
        assert x["loss_history"] == y["loss_history"] and x["eval_history"] == y["eval_history"]
        assert x["best_eval"] == y["best_eval"] and np.array_equal(x["block"], y["block"])


def test_golden_c1_run_parallel(orc):
    """The restatement's run_parallel reproduces the reference's C1 run
    (tests/golden/c1_run_parallel.npz, made by oracle/_ref) bit for bit."""
    from tests.golden.make_golden import c1_run_parallel
    g = np.load(os.path.join(GOLD, "c1_run_parallel.npz"))
    mine = c1_run_parallel(orc, int(g["epochs"]))
    for key in mine:
        assert np.array_equal(np.asarray(mine[key]), g[key]), key
