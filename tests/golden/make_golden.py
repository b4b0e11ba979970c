"""Regenerates tests/golden/*.npz from the REFERENCE build (oracle/_ref).

Run here (where /root/reference exists):  python tests/golden/make_golden.py
The fixtures pin the CPU restatement (oracle/liboracle.so) when the reference
library is not available (e.g. on the GPU box): tests/test_oracle.py checks the
restatement against them bit for bit.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
from oracle.oracle import Oracle, make_task  # noqa: E402


def spec(name):
    return open(os.path.join(ROOT, "configs", name + ".json")).read()


def cifar_like(n, seed):
    """Seeded CIFAR-shape synthetic images in [0,1) (PCG64 stream is stable)."""
    return np.random.default_rng(seed).random((n, 3, 32, 32), dtype=np.float32)


def main():
    ref = Oracle("ref")
    out = {}

    # 1. Toy teacher train_block end to end (test_distill.cpp:30-53 fixture).
    toy = spec("toy_teacher")
    tw = ref.teacher_init(toy, 404)
    img, lab = ref.synthetic_dataset(60, 11, 2)
    tr, ev = ref.stratified_split(lab, 0.2, 12)
    task = make_task(2, epochs=4, eval_every=2, seed=1234, batch_size=16, lr=0.02)
    nf = ref.candidate_num_floats(0, 16, 32, 2)
    r = ref.train_block(toy, tw, img, lab, tr, ev, task, nf)
    np.savez_compressed(os.path.join(HERE, "toy_train_block.npz"),
                        teacher_w=tw, images=img, labels=lab, train_idx=tr, eval_idx=ev,
                        loss_history=np.array(r["loss_history"]),
                        eval_history=np.array(r["eval_history"]),
                        final_local_loss=r["final_local_loss"], best_eval=r["best_eval"],
                        block=r["block"])

    # 2. VGG-16 step-loop replays (C2 shapes), B=8, 3 steps, blocks 2 and 9.
    vgg = spec("vgg16_cifar")
    tw = ref.teacher_init(vgg, ref.mix_seed(42, 0x7E11))
    img = cifar_like(40, 7)
    lab = (np.arange(40) % 10).astype(np.int32)
    tr, ev = ref.stratified_split(lab, 0.1, ref.mix_seed(42, 0x5711))
    for k, cin, cout, s in [(2, 64, 64, 1), (9, 512, 512, 1)]:
        task = make_task(k, seed=ref.mix_seed(42, k), batch_size=8)
        nf = ref.candidate_num_floats(0, cin, cout, s)
        losses, fw = ref.train_replay(vgg, tw, img, lab, tr, ev, task, 3, nf)
        out[f"vgg_b{k}_losses"] = losses
        out[f"vgg_b{k}_final"] = fw
    out["vgg_train_idx"], out["vgg_eval_idx"] = tr, ev

    # 3. Kernel outputs on seeded inputs (ops.hpp), shapes from C2 blocks.
    rng = np.random.default_rng(3)
    x = rng.uniform(-1, 1, (2, 8, 9, 7)).astype(np.float32)
    k = rng.uniform(-1, 1, (8, 1, 3, 3)).astype(np.float32)
    for s in (1, 2):
        y = ref.dw_fwd(x, k, s, 1)
        gy = rng.uniform(-1, 1, y.shape).astype(np.float32)
        gx, gk = ref.dw_bwd(x, k, gy, s, 1)
        out[f"dw_s{s}_x"], out[f"dw_s{s}_k"], out[f"dw_s{s}_y"] = x, k, y
        out[f"dw_s{s}_gy"], out[f"dw_s{s}_gx"], out[f"dw_s{s}_gk"] = gy, gx, gk
    w = rng.uniform(-1, 1, (6, 8, 1, 1)).astype(np.float32)
    y = ref.pw_fwd(x, w, 1)
    gy = rng.uniform(-1, 1, y.shape).astype(np.float32)
    gx, gw = ref.pw_bwd(x, w, gy, 1)
    out.update(pw_x=x, pw_w=w, pw_y=y, pw_gy=gy, pw_gx=gx, pw_gw=gw)
    gamma = rng.uniform(0.5, 1.5, 8).astype(np.float32)
    beta = rng.uniform(-0.5, 0.5, 8).astype(np.float32)
    yb, xhat, inv, mm, mv = ref.bn_train_fwd(x, gamma, beta, np.zeros(8), np.ones(8))
    gyb = rng.uniform(-1, 1, x.shape).astype(np.float32)
    gxb, gg, gb = ref.bn_train_bwd(xhat, inv, gamma, gyb)
    out.update(bn_x=x, bn_gamma=gamma, bn_beta=beta, bn_y=yb, bn_xhat=xhat, bn_inv=inv,
               bn_mm=mm, bn_mv=mv, bn_gy=gyb, bn_gx=gxb, bn_gg=gg, bn_gb=gb)
    t = rng.uniform(-1, 1, x.shape).astype(np.float32)
    out.update(mse_t=t, mse_loss=np.float32(ref.mse(x, t)), mse_g=ref.mse_bwd(x, t, 1.0))
    kc = rng.uniform(-1, 1, (5, 8, 3, 3)).astype(np.float32)
    out.update(conv_k=kc, conv_y=ref.conv_fwd(x, kc, 2, 1))
    np.savez_compressed(os.path.join(HERE, "c2_replay_and_kernels.npz"), **out)
    print("wrote", os.listdir(HERE))


def c1_run_parallel(O, n_epochs=2, f64=None):
    """4. C1 (BASELINE configs[0]) through the reference's run_parallel:
    4 blocks, batch 32, dataset 1000 (900 train / 100 eval), n_epochs epochs,
    eval every epoch, WFD plan over 2 workers."""
    c1 = spec("c1_small_vgg")
    tw = O.teacher_init(c1, O.mix_seed(42, 0x7E11))
    img = cifar_like(1000, 2012)
    lab = (np.arange(1000) % 10).astype(np.int32)
    tr, ev = O.stratified_split(lab, 0.1, O.mix_seed(42, 0x5711))
    geo = [(3, 16, 1), (16, 32, 2), (32, 64, 2), (64, 64, 1)]
    tasks = [make_task(k, epochs=n_epochs, eval_every=1, seed=O.mix_seed(42, k), batch_size=32)
             for k in range(1, 5)]
    nfs = [O.candidate_num_floats(0, *g) for g in geo]
    res = O.run_parallel(c1, tw, img, lab, tr, ev, tasks, [[1, 4], [2, 3]], nfs, policy=1)
    out = dict(teacher_w=tw, train_idx=tr, eval_idx=ev, epochs=n_epochs)
    for k, r in zip(range(1, 5), res):
        out[f"b{k}_loss_history"] = np.array(r["loss_history"])
        out[f"b{k}_eval_history"] = np.array(r["eval_history"])
        out[f"b{k}_best_eval"] = r["best_eval"]
        out[f"b{k}_block"] = r["block"]
        assert not r["failed"], r["failure"]
    if f64 is not None:
        # the reference's loss history is a mean of per-batch fp32 serial sums
        # (ops.hpp:522-527) with their own rounding; the restatement (bitwise
        # equal to the reference) also sums the same outputs in fp64
        for k, t, nf in zip(range(1, 5), tasks, nfs):
            r = f64.train_block(c1, tw, img, lab, tr, ev, t, nf, with_f64=True)
            assert r["loss_history"] == out[f"b{k}_loss_history"].tolist(), k
            out[f"b{k}_loss_history64"] = np.array(r["loss_history64"])
    return out


def generic_paths(O):
    """5. The layer-by-layer GPU paths against the reference on the toy
    teacher (test_distill.cpp fixture): train_block with the Combined
    objective and with the skip candidates, reassemble + finetune (frozen and
    not), train_teacher."""
    toy = spec("toy_teacher")
    tw = O.teacher_init(toy, 404)
    img, lab = O.synthetic_dataset(60, 11, 2)
    tr, ev = O.stratified_split(lab, 0.2, 12)
    out = dict(teacher_w=tw, images=img, labels=lab, train_idx=tr, eval_idx=ev)
    geo = {1: (3, 16, 1), 2: (16, 32, 2), 3: (32, 32, 1)}
    cases = {"combined": make_task(2, epochs=2, eval_every=1, seed=1234, batch_size=16, lr=0.02, loss_mode=1,
                                   lambda_local=0.5),
             "skip2": make_task(2, kind=2, epochs=2, eval_every=1, seed=99, batch_size=16, lr=0.02),
             "skip3": make_task(3, kind=3, epochs=2, eval_every=1, seed=98, batch_size=16, lr=0.02)}
    for name, t in cases.items():
        nf = O.candidate_num_floats(t.kind, *geo[t.block_index])
        r = O.train_block(toy, tw, img, lab, tr, ev, t, nf)
        assert not r["failed"], r["failure"]
        out[f"{name}_loss_history"] = np.array(r["loss_history"])
        out[f"{name}_eval_history"] = np.array(r["eval_history"])
        out[f"{name}_best_eval"] = r["best_eval"]
        out[f"{name}_block"] = r["block"]
    reps = [(1, 0, 7), (3, 1, 9)]
    out["reps"] = np.array(reps, np.int64)
    for name, kw in {"ft_frozen": dict(epochs=2, freeze=1, lr=0.01, momentum=0.9, batch=16, seed=77, teacher_mode=0),
                     "ft_all": dict(epochs=1, freeze=0, lr=0.01, momentum=0.9, batch=16, seed=78, teacher_mode=0),
                     "teacher": dict(epochs=2, freeze=0, lr=0.05, momentum=0.9, batch=24, seed=900,
                                     teacher_mode=1)}.items():
        r = O.fit_network(toy, tw, img, lab, tr, ev, [] if name == "teacher" else reps, **kw)
        n = int(np.max(np.nonzero(r["net"])[0])) + 1
        out[f"{name}_loss_history"] = r["loss_history"]
        out[f"{name}_eval_history"] = r["eval_history"]
        out[f"{name}_net"] = r["net"][:n]
    return out


if __name__ == "__main__":
    if sys.argv[1:] == ["generic"]:
        np.savez_compressed(os.path.join(HERE, "toy_generic_paths.npz"), **generic_paths(Oracle("ref")))
    elif sys.argv[1:] == ["c1"]:
        np.savez_compressed(os.path.join(HERE, "c1_run_parallel.npz"),
                            **c1_run_parallel(Oracle("ref"), f64=Oracle("orc")))
    else:
        main()
