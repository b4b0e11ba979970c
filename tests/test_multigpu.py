"""Multi-GPU path: sample-sharded teacher + all-to-all-v of boundary rows.

* CPU, world_size 2 over gloo: every rank derives the exchange layout from
  pbkd_exchange_plan (the same C++ code the engine uses); the ranks pack
  synthetic teacher rows by that layout, exchange them with all_to_all_single
  and unpack them into epoch-ordered streams.  Checks the layout agrees
  across ranks and every row lands where its owner expects it.
* GPU (one device): virtual_shards > 1 runs the engine's real pack / scatter
  kernels with local shards; training results must be bitwise identical to
  the unsharded run (teacher rows are per-sample, so sharding must not move a
  single bit).
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


def _value(t, b, kind, j):
    return float(t * 1000 + b * 10 + kind) + j * 1e-3


def _worker(rank, world, port, share, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        blocks = [1, 2, 3, 4, 5]
        weights = [3.0, 8.0, 2.0, 5.0, 4.0]
        plan, _ = P.wfd_bin_pack(blocks, weights, world)
        owner = {k: w for w, q_ in enumerate(plan) for k in q_}
        owners = [owner[k] for k in blocks]
        in_row, out_row = [3, 5, 2, 4, 6], [5, 2, 4, 6, 1]
        n_train = 37
        plans = {}
        for a in range(world):
            for b in range(world):
                plans[(a, b)] = P.exchange_plan(blocks, owners, in_row, out_row, world, n_train, a, b, share)
        sb = plans[(0, 0)][3]
        # 1) layout agreement: what I send to d must be what d expects from me
        mine = [(plans[(rank, d)][0], plans[(rank, d)][1].tolist()) for d in range(world)]
        gathered = [None] * world
        dist.all_gather_object(gathered, mine)
        for s in range(world):
            cnt, off = gathered[s][rank]
            assert cnt == plans[(s, rank)][0] and off == plans[(s, rank)][1].tolist()
        # 2) pack my shard's rows for every block's owner
        rows = range(sb[rank], sb[rank + 1])
        send_parts = []
        for d in range(world):
            buf = np.zeros(plans[(rank, d)][0], np.float32)
            for bp, b in enumerate(blocks):
                if owners[bp] != d:
                    continue
                oi, ot = int(plans[(rank, d)][1][bp]), int(plans[(rank, d)][2][bp])
                for i, t in enumerate(rows):
                    for j in range(in_row[bp]):
                        buf[oi + i * in_row[bp] + j] = _value(t, b, 0, j)
                    for j in range(out_row[bp]):
                        buf[ot + i * out_row[bp] + j] = _value(t, b, 1, j)
            send_parts.append(buf)
        send = torch.from_numpy(np.concatenate(send_parts))
        recv_counts = [plans[(s, rank)][0] for s in range(world)]
        recv = torch.zeros(sum(recv_counts))
        dist.all_to_all_single(recv, send, recv_counts, [len(p_) for p_ in send_parts])
        recv = recv.numpy()
        # 3) unpack into epoch-ordered streams (pos = a random permutation)
        pos = np.random.default_rng(5).permutation(n_train)
        roff = np.concatenate([[0], np.cumsum(recv_counts)])
        ok = 0
        for bp, b in enumerate(blocks):
            if owners[bp] != rank:
                continue
            stream_in = np.full((n_train, in_row[bp]), -1.0, np.float32)
            for s in range(world):
                oi = int(roff[s] + plans[(s, rank)][1][bp])
                nrows = sb[s + 1] - sb[s]
                part = recv[oi:oi + nrows * in_row[bp]].reshape(nrows, in_row[bp])
                stream_in[pos[sb[s]:sb[s + 1]]] = part
            for t in range(n_train):
                want = [_value(t, b, 0, j) for j in range(in_row[bp])]
                assert np.allclose(stream_in[pos[t]], want)
            ok += 1
        q.put((rank, ok, None))
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
    assert sum(ok for _, ok, _ in res) == 5  # every block unpacked by its owner


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
def test_boundary_buffers_match_streams(orc, monkeypatch):
    """Single-GPU boundary-buffer path (teacher boundaries stored once, student
    batches gathered through the epoch order) against the per-task stream +
    scatter path: identical bits, baseline and evaluations included."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from tests.conftest import spec_text
    spec = spec_text("c1_small_vgg")
    ctx = P.Context(0)
    ctx.teacher_load(spec, orc.teacher_init(spec, 5))
    img = np.random.default_rng(9).random((90, 3, 32, 32), dtype=np.float32)
    lab = (np.arange(90) % 10).astype(np.int32)
    ctx.dataset_load(img, lab)
    tr, ev = orc.stratified_split(lab, 0.2, 4)
    tasks = lambda: [P.make_task(k, epochs=2, eval_every=1, seed=P.mix_seed(3, k), batch_size=16)  # noqa: E731
                     for k in (1, 2, 3, 4)]
    monkeypatch.delenv("PBKD_STREAMS", raising=False)
    bnd = ctx.run(tasks(), tr, ev)["results"]
    monkeypatch.setenv("PBKD_STREAMS", "1")
    stm = ctx.run(tasks(), tr, ev)["results"]
    for a, b in zip(bnd, stm):
        assert a["loss_history"] == b["loss_history"]
        assert a["eval_history"] == b["eval_history"]
        assert np.array_equal(a["block"], b["block"])
        assert np.array_equal(a["final_block"], b["final_block"])
