"""Multi-GPU path: sample-sharded teacher + one exchange of boundary rows.

* CPU, world_size 2 over gloo: every rank derives the exchange layout from
  pbkd_exchange_plan (the same C++ BoundaryPlan the engine uses), computes
  synthetic boundary rows of its shard, exchanges them with send/recv in the
  plan's issue order straight between full-size boundary buffers (as
  NcclComm::exchange does), and checks every boundary its blocks read is
  complete and that shared boundaries travel once.
* GPU (one device): virtual_shards > 1 computes the teacher boundaries shard
  by shard; training results must be bitwise identical to the unsharded run
  (teacher rows are per-sample, so sharding must not move a single bit).
"""
import os
import socket

import numpy as np
import pytest

import paper_2012_03096_b200 as P


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _value(t, j, col):
    return float(t * 1000 + j * 10) + col * 1e-3


def _worker(rank, world, port, share, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        blocks = [1, 2, 3, 4, 5, 6]
        weights = [3.0, 8.0, 2.0, 5.0, 4.0, 1.0]
        plan, _ = P.wfd_bin_pack(blocks, weights, world)
        owner = {k: w for w, q_ in enumerate(plan) for k in q_}
        owners = [owner[k] for k in blocks]
        rows = [3, 5, 2, 4, 6, 1, 7]  # floats per sample of boundaries 0..6
        n_train = 37
        plans = {(a, b): P.exchange_plan(blocks, owners, rows, world, n_train, a, b, share)
                 for a in range(world) for b in range(world)}
        sb = plans[(0, 0)][2]
        # 1) layout agreement: what I send to d must be what d expects from me
        mine = [plans[(rank, d)][:2] for d in range(world)]
        gathered = [None] * world
        dist.all_gather_object(gathered, mine)
        for s_ in range(world):
            assert tuple(gathered[s_][rank]) == tuple(plans[(s_, rank)][:2])
        # 2) boundary buffers: boundary 0 (images) complete everywhere, j >= 1
        #    only on this rank's shard rows; exchange in the plan's issue order
        bnd = [np.full((n_train, r), -1.0, np.float32) for r in rows]
        bnd[0][:] = [[_value(t, 0, c) for c in range(rows[0])] for t in range(n_train)]
        for j in range(1, len(rows)):
            for t in range(sb[rank], sb[rank + 1]):
                bnd[j][t] = [_value(t, j, c) for c in range(rows[j])]
        reqs, inbox = [], []
        for p_ in range(world):
            if p_ == rank:
                continue
            for j, r0, nr in plans[(rank, p_)][1]:
                reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(bnd[j][r0:r0 + nr])), p_))
            for j, r0, nr in plans[(p_, rank)][1]:
                buf = torch.zeros(nr, rows[j])
                reqs.append(dist.irecv(buf, p_))
                inbox.append((j, r0, buf))
        for r in reqs:
            r.wait()
        got = 0
        for j, r0, buf in inbox:
            bnd[j][r0:r0 + buf.shape[0]] = buf.numpy()
            got += buf.numel()
        assert got == sum(plans[(p_, rank)][0] for p_ in range(world) if p_ != rank)
        # 3) every boundary my blocks read is complete; each travels once per peer
        mine_blocks = [k for k in blocks if owner[k] == rank]
        for k in mine_blocks:
            for j in (k - 1, k):
                want = np.array([[_value(t, j, c) for c in range(rows[j])] for t in range(n_train)], np.float32)
                assert np.array_equal(bnd[j], want), (rank, k, j)
        for p_ in range(world):
            js = [x[0] for x in plans[(p_, rank)][1]]
            assert len(js) == len(set(js)) and 0 not in js
        q.put((rank, len(mine_blocks), None))
    except Exception as e:  # surface the failure in the parent
        q.put((rank, -1, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("share", [None, [1.0, 2.5]])
def test_exchange_plan_gloo_world2(share):
    import torch.multiprocessing as mp
    if not os.path.exists(P.LIB_PATH):
        P.build()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, share, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    for rank, ok, err in res:
        assert err is None, err
        assert ok >= 1
    assert sum(ok for _, ok, _ in res) == 6  # every block checked by its owner


def test_exchange_plan_shares_boundaries():
    """Blocks k and k+1 on one owner read boundary k once (no duplicate rows)."""
    if not os.path.exists(P.LIB_PATH):
        P.build()
    rows = [3, 4, 5, 6]
    cnt, xs, sb = P.exchange_plan([1, 2, 3], [1, 1, 0], rows, 2, 10, 0, 1)
    assert [x[0] for x in xs] == [1, 2] and cnt == sum(rows[j] * (sb[1] - sb[0]) for j in (1, 2))
    cnt, xs, sb = P.exchange_plan([1, 2, 3], [1, 1, 0], rows, 2, 10, 1, 0)
    assert [x[0] for x in xs] == [2, 3]


@pytest.mark.gpu
@pytest.mark.parametrize("shards,share", [(2, None), (3, [1.0, 3.0, 0.5])])
def test_virtual_shards_bitwise(orc, shards, share):
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from tests.conftest import spec_text
    spec = spec_text("c1_small_vgg")
    ctx = P.Context(0)
    ctx.teacher_load(spec, orc.teacher_init(spec, 11))
    img = np.random.default_rng(4).random((70, 3, 32, 32), dtype=np.float32)
    lab = (np.arange(70) % 10).astype(np.int32)
    ctx.dataset_load(img, lab)
    tr, ev = orc.stratified_split(lab, 0.1, 3)
    tasks = lambda: [P.make_task(k, epochs=2, seed=P.mix_seed(7, k), batch_size=16) for k in (1, 2, 3, 4)]  # noqa: E731
    base = ctx.run(tasks(), tr, ev, flags=P.RUN_STEP_ONLY)["results"]
    shd = ctx.run(tasks(), tr, ev, flags=P.RUN_STEP_ONLY, virtual_shards=shards, share=share,
                  global_blocks=[(k, 0) for k in (1, 2, 3, 4)])["results"]
    for a, b in zip(base, shd):
        assert np.array_equal(a["step_losses"], b["step_losses"])
        assert np.array_equal(a["final_block"], b["final_block"])


@pytest.mark.gpu
@pytest.mark.parametrize("policy", ["round_robin", "wfd", "work_stealing"])
def test_context_over_gpu_list_run_parallel(orc, policy):
    """A context over a GPU list (pbkd_ctx_create_multi: one engine per GPU,
    one in-process NCCL clique, a host thread per GPU).  On this one-GPU box
    the list is [0]: a one-rank communicator, so the teacher boundaries still
    go through the NCCL exchange (self send/recv), and run_parallel with 2
    workers and evaluations must give the single-GPU context's bits."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from tests.conftest import spec_text
    spec = spec_text("toy_teacher")
    tw = orc.teacher_init(spec, 2025)
    img, lab = orc.synthetic_dataset(40, 21, 2)
    tr, ev = orc.stratified_split(lab, 0.25, 3)
    tasks = lambda: [P.make_task(k, epochs=2, eval_every=1, seed=P.mix_seed(99, k), batch_size=10, lr=0.02)  # noqa: E731
                     for k in (1, 2, 3)]
    plan = [[1, 2, 3], []] if policy == "work_stealing" else P.round_robin([1, 2, 3], 2)
    one = P.Context(0)
    one.teacher_load(spec, tw)
    one.dataset_load(img, lab)
    base = one.run(tasks(), tr, ev, plan=plan, workers=2, policy=policy)
    one.close()
    multi = P.Context(devices=[0])
    multi.teacher_load(spec, tw)
    multi.dataset_load(img, lab)
    got = multi.run(tasks(), tr, ev, plan=plan, workers=2, policy=policy)
    assert [x["block_index"] for x in got["results"]] == [1, 2, 3]
    for a, b in zip(base["results"], got["results"]):
        assert not b["failed"], b["failure"]
        assert np.array_equal(a["block"], b["block"]) and np.array_equal(a["final_block"], b["final_block"])
        assert a["loss_history"] == b["loss_history"] and a["eval_history"] == b["eval_history"]
    kinds = [e[3] for e in got["trace"]]
    assert kinds.count(0) == 3 and kinds.count(1) == 3 and kinds.count(2) == 3 and kinds.count(4) == 1
