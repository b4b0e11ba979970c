"""pbkd-b200: B200-native parallel blockwise knowledge distillation.

Python front end over the C ABI (include/pbkd_b200.h) of libpbkd_b200.so --
the in-tree CUDA (sm_100a) + C++ library.  There is no Python or CPU fallback:
if the shared library is missing, importing :class:`Lib` raises.

The C++ host API (include/pbkd/*.hpp, same signatures as the reference's
pbkd:: API) is the primary interface; this module exists for the test suite,
the benchmark and Python callers.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
# PBKD_LIB: another build of the same library (A/B diagnosis runs)
LIB_PATH = os.environ.get("PBKD_LIB") or os.path.join(HERE, "libpbkd_b200.so")

KINDS = {"two_layer": 0, "three_layer": 1, "two_layer_skip": 2, "three_layer_skip": 3}
POLICIES = {"round_robin": 0, "wfd": 1, "work_stealing": 2}
RUN_STEP_ONLY, RUN_NO_GRAPH, RUN_PROFILE = 1, 2, 4
class WeightsError(RuntimeError):
    """pbkd::WeightsError: unreadable or inconsistent PBKD weight file."""


ERR_KINDS = {1: ValueError, 2: ValueError, 3: IndexError, 4: RuntimeError, 5: RuntimeError,
             6: RuntimeError, 7: WeightsError}


class Task(C.Structure):
    """pbkd_task == pbkd::DistillTask (reference distill.hpp:24-37)."""
    _fields_ = [("block_index", C.c_int), ("kind", C.c_int), ("epochs", C.c_int),
                ("eval_every", C.c_int), ("seed", C.c_uint64), ("threshold", C.c_double),
                ("loss_mode", C.c_int), ("lambda_local", C.c_float), ("lr", C.c_float),
                ("momentum", C.c_float), ("batch_size", C.c_int), ("max_steps", C.c_longlong)]


def make_task(block_index, kind=0, epochs=30, eval_every=2, seed=0, threshold=0.0, loss_mode=0,
              lambda_local=1.0, lr=0.05, momentum=0.9, batch_size=50, max_steps=0):
    return Task(block_index, kind, epochs, eval_every, seed, threshold, loss_mode, lambda_local,
                lr, momentum, batch_size, max_steps)


class ResultInfo(C.Structure):
    _fields_ = [("block_index", C.c_int), ("failed", C.c_int), ("kind", C.c_char * 32),
                ("failure", C.c_char * 256), ("n_loss", C.c_int), ("n_eval", C.c_int),
                ("n_steps", C.c_longlong), ("n_block_floats", C.c_size_t), ("has_best", C.c_int),
                ("final_local_loss", C.c_double), ("best_eval", C.c_double),
                ("wall_time_s", C.c_double)]


class TraceEvent(C.Structure):
    _fields_ = [("timestamp_s", C.c_double), ("worker_id", C.c_int), ("task_id", C.c_int),
                ("kind", C.c_int)]


def build(jobs: int = 8) -> None:
    """Compile libpbkd_b200.so in-tree for sm_100a (make -C paper_2012_03096_b200)."""
    subprocess.run(["make", "-s", "-C", HERE, f"-j{jobs}"], check=True)


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is not built; run paper_2012_03096_b200.build() "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        vp, ip, fp, dp = C.c_void_p, C.POINTER(C.c_int), C.POINTER(C.c_float), C.POINTER(C.c_double)
        sig = {
            "pbkd_last_error": (C.c_char_p, []), "pbkd_last_error_kind": (C.c_int, []),
            "pbkd_version": (C.c_char_p, []),
            "pbkd_ctx_create": (C.c_int, [C.c_int, C.POINTER(vp)]),
            "pbkd_ctx_destroy": (None, [vp]), "pbkd_device_count": (C.c_int, [ip]),
            "pbkd_spec_num_floats": (C.c_int, [C.c_char_p, C.POINTER(C.c_size_t)]),
            "pbkd_spec_num_blocks": (C.c_int, [C.c_char_p, ip]),
            "pbkd_teacher_load": (C.c_int, [vp, C.c_char_p, vp, C.c_size_t]),
            "pbkd_teacher_init": (C.c_int, [vp, C.c_char_p, C.c_uint64]),
            "pbkd_teacher_weights": (C.c_int, [vp, vp, C.c_size_t]),
            "pbkd_dataset_load": (C.c_int, [vp, vp, vp] + [C.c_int] * 5),
            "pbkd_dataset_load_device": (C.c_int, [vp, vp, vp] + [C.c_int] * 5),
            "pbkd_run": (C.c_int, [vp, vp, C.c_int, vp, C.c_int, vp, C.c_int, C.c_int,
                                   C.POINTER(vp)]),
            "pbkd_run_parallel": (C.c_int, [vp, vp, C.c_int, vp, C.c_int, vp, C.c_int, C.c_int,
                                            C.c_int, vp, vp, C.c_int, C.POINTER(vp)]),
            "pbkd_run_count": (C.c_int, [vp]),
            "pbkd_run_info": (C.c_int, [vp, C.c_int, C.POINTER(ResultInfo)]),
            "pbkd_run_loss_history": (C.c_int, [vp, C.c_int, vp, C.c_int]),
            "pbkd_run_eval_history": (C.c_int, [vp, C.c_int, vp, vp, C.c_int]),
            "pbkd_run_block": (C.c_int, [vp, C.c_int, C.c_int, vp, C.c_size_t]),
            "pbkd_run_step_losses": (C.c_int, [vp, C.c_int, vp, C.c_longlong]),
            "pbkd_run_trace": (C.c_int, [vp, vp, C.c_int, ip]),
            "pbkd_run_wall_time": (C.c_double, [vp]), "pbkd_run_epoch_ms": (C.c_double, [vp]),
            "pbkd_run_free": (None, [vp]),
            "pbkd_run_timed": (C.c_int, [vp, vp, C.c_int, vp, C.c_int, vp, C.c_int, C.c_int,
                                         C.c_int, C.POINTER(vp)]),
            "pbkd_run_timing": (C.c_int, [vp, dp, ip, C.POINTER(C.c_longlong), vp, C.c_int, ip]),
            "pbkd_run_profile_count": (C.c_int, [vp]),
            "pbkd_run_profile_entry": (C.c_int, [vp, C.c_int, C.c_char_p, C.c_size_t, ip, dp, dp, dp]),
            "pbkd_bench_kernel": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, dp, dp, dp]),
            "pbkd_nccl_unique_id": (C.c_int, [vp]),
            "pbkd_ctx_set_comm": (C.c_int, [vp, vp, C.c_int, C.c_int]),
            "pbkd_run_sharded": (C.c_int, [vp, vp, C.c_int, vp, C.c_int, vp, C.c_int, C.c_int, C.c_int,
                                           vp, vp, C.c_int, C.c_int, vp, C.c_int, C.POINTER(vp)]),
            "pbkd_exchange_plan": (C.c_int, [vp, vp, C.c_int, vp, C.c_int, C.c_int, C.c_int, vp,
                                             C.c_int, C.c_int, C.POINTER(C.c_size_t), vp, vp, vp,
                                             C.c_int, ip, vp]),
            "pbkd_prefix_infer": (C.c_int, [vp, vp, C.c_int, C.c_int, C.c_int, vp, C.c_size_t, vp]),
            "pbkd_candidate_infer": (C.c_int, [vp] + [C.c_int] * 4 + [vp, vp] + [C.c_int] * 3 +
                                     [vp, C.c_size_t]),
            "pbkd_eval_with_student": (C.c_int, [vp, C.c_int, C.c_int, vp, vp, C.c_int, C.c_int,
                                                 dp]),
            "pbkd_mix_seed": (C.c_uint64, [C.c_uint64, C.c_uint64]),
            "pbkd_stratified_split": (C.c_int, [vp, C.c_int, C.c_double, C.c_uint64, vp, ip, vp,
                                                ip]),
            "pbkd_epoch_order": (C.c_int, [vp, C.c_int, C.c_uint64, C.c_int, vp]),
            "pbkd_build_candidate": (C.c_int, [C.c_int] * 4 + [C.c_uint64, vp, C.c_size_t,
                                                               C.POINTER(C.c_size_t)]),
            "pbkd_round_robin": (C.c_int, [vp, C.c_int, C.c_int, vp, vp]),
            "pbkd_wfd_bin_pack": (C.c_int, [vp, vp, C.c_int, C.c_int, vp, vp, dp]),
            "pbkd_makespan": (C.c_int, [vp, vp, C.c_int, vp, vp, C.c_int, dp]),
            "pbkd_mac_proxy_weights": (C.c_int, [C.c_char_p, vp, C.c_int, vp]),
            "pbkd_k_dw_fwd": (C.c_int, [vp, vp, vp, vp] + [C.c_int] * 6),
            "pbkd_k_dw_bwd": (C.c_int, [vp] + [vp] * 11 + [C.c_int] * 4),
            "pbkd_k_dw_gk": (C.c_int, [vp, vp, vp, vp] + [C.c_int] * 6),
            "pbkd_k_pw_fwd": (C.c_int, [vp, vp, vp, vp, C.c_int, C.c_int, C.c_int, vp, vp]),
            "pbkd_k_pw_bwd": (C.c_int, [vp, vp, vp, vp, vp, vp, C.c_int, C.c_int, C.c_int]),
            "pbkd_k_sgd": (C.c_int, [vp, vp, vp, vp, C.c_size_t, C.c_float, C.c_float]),
            "pbkd_sgd_host": (C.c_int, [vp, vp, vp, C.c_size_t, C.c_float, C.c_float]),
            "pbkd_teacher_save_file": (C.c_int, [vp, C.c_char_p]),
            "pbkd_teacher_load_file": (C.c_int, [vp, C.c_char_p, C.c_char_p]),
            "pbkd_save_student_network": (C.c_int, [C.c_char_p, vp, C.c_size_t, C.c_int, C.c_int, vp,
                                                    C.c_size_t, C.c_char_p]),
            "pbkd_load_network_file": (C.c_int, [C.c_char_p, C.c_char_p, vp, C.c_int, vp, C.c_size_t,
                                                 C.POINTER(C.c_size_t)]),
            "pbkd_file_hash": (C.c_int, [C.c_char_p, C.POINTER(C.c_uint64)]),
            "pbkd_fit_assembled": (C.c_int, [vp, C.c_char_p, vp, C.c_size_t, vp, vp, vp, C.c_int, vp, C.c_int,
                                             vp, C.c_int, C.c_int, C.c_int, C.c_float, C.c_float, C.c_int,
                                             C.c_uint64, C.c_int, dp, dp, vp, vp, vp, ip, vp, C.c_size_t,
                                             C.POINTER(C.c_size_t)]),
            "pbkd_mse_local_loss": (C.c_int, [vp, vp, vp, C.c_size_t, fp]),
            "pbkd_ctx_create_multi": (C.c_int, [vp, C.c_int, C.POINTER(vp)]),
            "pbkd_ctx_device_count": (C.c_int, [vp, ip]),
            "pbkd_softmax_ce": (C.c_int, [vp, vp, C.c_int, C.c_int, vp, fp, vp]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype, f.argtypes = res, args
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc != 0:
        L = lib()
        raise ERR_KINDS.get(L.pbkd_last_error_kind(), RuntimeError)(L.pbkd_last_error().decode())


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _i32(a):
    return np.ascontiguousarray(a, np.int32)


def _f32(a):
    return np.ascontiguousarray(a, np.float32)


# ----------------------------------------------------------- host helpers --
def mix_seed(a: int, b: int) -> int:
    return lib().pbkd_mix_seed(a, b)


def stratified_split(labels, frac, seed):
    lab = _i32(labels)
    tr, ev = np.zeros(len(lab), np.int32), np.zeros(len(lab), np.int32)
    nt, ne = C.c_int(), C.c_int()
    check(lib().pbkd_stratified_split(_ptr(lab), len(lab), frac, seed, _ptr(tr), C.byref(nt),
                                      _ptr(ev), C.byref(ne)))
    return tr[:nt.value].copy(), ev[:ne.value].copy()


def epoch_order(train_idx, seed, epoch):
    tr = _i32(train_idx)
    out = np.zeros_like(tr)
    check(lib().pbkd_epoch_order(_ptr(tr), len(tr), seed, epoch, _ptr(out)))
    return out


def build_candidate(kind, cin, cout, stride, seed):
    n = C.c_size_t()
    check(lib().pbkd_build_candidate(kind, cin, cout, stride, seed, None, 0, C.byref(n)))
    out = np.zeros(n.value, np.float32)
    check(lib().pbkd_build_candidate(kind, cin, cout, stride, seed, _ptr(out), out.size, None))
    return out


def _plan(ids, counts):
    plan, at = [], 0
    for c in counts:
        plan.append([int(v) for v in ids[at:at + c]])
        at += c
    return plan


def round_robin(ids, workers):
    ids = _i32(ids)
    out, cnt = np.zeros(len(ids), np.int32), np.zeros(workers, np.int32)
    check(lib().pbkd_round_robin(_ptr(ids), len(ids), workers, _ptr(out), _ptr(cnt)))
    return _plan(out, cnt)


def wfd_bin_pack(ids, weights, workers):
    ids, w = _i32(ids), np.ascontiguousarray(weights, np.float64)
    out, cnt = np.zeros(len(ids), np.int32), np.zeros(workers, np.int32)
    mk = C.c_double()
    check(lib().pbkd_wfd_bin_pack(_ptr(ids), _ptr(w), len(ids), workers, _ptr(out), _ptr(cnt),
                                  C.byref(mk)))
    return _plan(out, cnt), mk.value


def makespan(plan, ids, weights):
    flat = _i32([i for q in plan for i in q])
    cnt = _i32([len(q) for q in plan])
    ids, w = _i32(ids), np.ascontiguousarray(weights, np.float64)
    out = C.c_double()
    check(lib().pbkd_makespan(_ptr(flat), _ptr(cnt), len(plan), _ptr(ids), _ptr(w), len(ids),
                              C.byref(out)))
    return out.value


def mac_proxy_weights(spec, blocks):
    b = _i32(blocks)
    out = np.zeros(len(b), np.float64)
    check(lib().pbkd_mac_proxy_weights(spec.encode(), _ptr(b), len(b), _ptr(out)))
    return out


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    check(lib().pbkd_nccl_unique_id(buf))
    return buf.raw


def exchange_plan(blocks, owners, rows, world, n_train, src, dst, share=None):
    """Boundary rows rank `src` sends rank `dst` once per run (BoundaryPlan):
    (count in floats, [(boundary j, first train row, rows)], shard bounds)."""
    nb = len(blocks)
    b, o = _i32(blocks), _i32(owners)
    r = np.ascontiguousarray(rows, np.int64)
    sh = np.ascontiguousarray(share, np.float64) if share is not None else None
    cnt, n = C.c_size_t(), C.c_int()
    cap = len(rows) + 1
    xj, x0, xr = np.zeros(cap, np.int32), np.zeros(cap, np.int32), np.zeros(cap, np.int32)
    sbd = np.zeros(world + 1, np.int32)
    check(lib().pbkd_exchange_plan(_ptr(b), _ptr(o), nb, _ptr(r), len(r), world, n_train,
                                   _ptr(sh) if sh is not None else None, src, dst, C.byref(cnt),
                                   _ptr(xj), _ptr(x0), _ptr(xr), cap, C.byref(n), _ptr(sbd)))
    return cnt.value, [(int(xj[i]), int(x0[i]), int(xr[i])) for i in range(n.value)], sbd


def save_student_network(spec, teacher_weights, block_index, kind, block_weights, path):
    """Network of `spec` with block `block_index` replaced by a candidate of
    `kind` holding `block_weights` (e.g. a run result's "block"), as a PBKD file."""
    tw, bw = _f32(teacher_weights), _f32(block_weights)
    check(lib().pbkd_save_student_network(spec.encode(), _ptr(tw), tw.size, block_index, kind, _ptr(bw),
                                          bw.size, os.fsencode(path)))


def load_network_file(spec, path, cap=None):
    """rebuild_network_from_arrays over a PBKD file: (per-block kind, 0 = teacher
    structure / 1 + candidate kind, flat arrays of the rebuilt network)."""
    nb = spec_num_blocks(spec)
    kinds = np.zeros(nb, np.int32)
    cap = cap or 4 * spec_num_floats(spec) + 1024
    out = np.zeros(cap, np.float32)
    n = C.c_size_t()
    check(lib().pbkd_load_network_file(spec.encode(), os.fsencode(path), _ptr(kinds), nb, _ptr(out), cap,
                                       C.byref(n)))
    return kinds, out[:n.value].copy()


def file_hash(path):
    """FNV-1a 64 of the file bytes (weights_io.cpp file_hash)."""
    h = C.c_uint64()
    check(lib().pbkd_file_hash(os.fsencode(path), C.byref(h)))
    return h.value


def spec_num_floats(spec):
    n = C.c_size_t()
    check(lib().pbkd_spec_num_floats(spec.encode(), C.byref(n)))
    return n.value


def spec_num_blocks(spec):
    n = C.c_int()
    check(lib().pbkd_spec_num_blocks(spec.encode(), C.byref(n)))
    return n.value


# ----------------------------------------------------------------- context --
class Context:
    """One GPU (pbkd_ctx), or -- devices=[...] -- a context over a GPU list
    (pbkd_ctx_create_multi: one engine per GPU, one in-process NCCL clique;
    run() with a plan spreads the workers over the GPUs)."""

    def __init__(self, device: int = 0, devices=None):
        self.h = C.c_void_p()
        if devices is None:
            check(lib().pbkd_ctx_create(device, C.byref(self.h)))
        else:
            d = _i32(list(devices))
            check(lib().pbkd_ctx_create_multi(_ptr(d), len(d), C.byref(self.h)))

    def close(self):
        if self.h:
            lib().pbkd_ctx_destroy(self.h)
            self.h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def teacher_init(self, spec: str, seed: int):
        check(lib().pbkd_teacher_init(self.h, spec.encode(), seed))

    def teacher_load(self, spec: str, weights):
        w = _f32(weights)
        check(lib().pbkd_teacher_load(self.h, spec.encode(), _ptr(w), w.size))

    def teacher_weights(self, n):
        out = np.zeros(n, np.float32)
        check(lib().pbkd_teacher_weights(self.h, _ptr(out), n))
        return out

    def teacher_save_file(self, path):
        """The loaded teacher as a PBKD weight file (weights_io.cpp:68-99 layout)."""
        check(lib().pbkd_teacher_save_file(self.h, os.fsencode(path)))

    def teacher_load_file(self, spec: str, path):
        """Teacher of `spec` with its weights from a PBKD file (load_into_network)."""
        check(lib().pbkd_teacher_load_file(self.h, spec.encode(), os.fsencode(path)))

    def dataset_load(self, images, labels, classes=10):
        img, lab = _f32(images), _i32(labels)
        n, c, h, w = img.shape
        check(lib().pbkd_dataset_load(self.h, _ptr(img), _ptr(lab), n, c, h, w, classes))

    def dataset_load_device(self, dev_ptr: int, labels, shape, classes=10):
        lab = _i32(labels)
        n, c, h, w = shape
        check(lib().pbkd_dataset_load_device(self.h, C.c_void_p(dev_ptr), _ptr(lab), n, c, h, w,
                                             classes))

    def set_comm(self, nccl_id: bytes, rank: int, world: int):
        buf = C.create_string_buffer(bytes(nccl_id), 128)
        check(lib().pbkd_ctx_set_comm(self.h, buf, rank, world))

    def run(self, tasks, train_idx, eval_idx, flags=0, plan=None, workers=1, policy="round_robin",
            timed_from_epoch=None, global_blocks=None, virtual_shards=1, share=None):
        arr = (Task * len(tasks))(*tasks)
        tr, ev = _i32(train_idx), _i32(eval_idx)
        out = C.c_void_p()
        if global_blocks is not None or virtual_shards > 1:
            gb = list(global_blocks or [])
            b = _i32([k for k, _ in gb]) if gb else np.zeros(1, np.int32)
            o = _i32([w for _, w in gb]) if gb else np.zeros(1, np.int32)
            sh = np.ascontiguousarray(share, np.float64) if share is not None else None
            check(lib().pbkd_run_sharded(self.h, arr, len(tasks), _ptr(tr), len(tr), _ptr(ev), len(ev),
                                         flags, timed_from_epoch or 1, _ptr(b), _ptr(o), len(gb),
                                         virtual_shards, _ptr(sh) if sh is not None else None,
                                         len(sh) if sh is not None else 0, C.byref(out)))
        elif timed_from_epoch is not None:
            check(lib().pbkd_run_timed(self.h, arr, len(tasks), _ptr(tr), len(tr), _ptr(ev),
                                       len(ev), flags, timed_from_epoch, C.byref(out)))
        elif plan is None:
            check(lib().pbkd_run(self.h, arr, len(tasks), _ptr(tr), len(tr), _ptr(ev), len(ev),
                                 flags, C.byref(out)))
        else:
            ids = _i32([i for q in plan for i in q])
            cnt = _i32([len(q) for q in plan])
            check(lib().pbkd_run_parallel(self.h, arr, len(tasks), _ptr(tr), len(tr), _ptr(ev),
                                          len(ev), workers, POLICIES[policy], _ptr(ids),
                                          _ptr(cnt), flags, C.byref(out)))
        try:
            return self._collect(out)
        finally:
            lib().pbkd_run_free(out)

    def _collect(self, r):
        L = lib()
        res = []
        for i in range(L.pbkd_run_count(r)):
            info = ResultInfo()
            check(L.pbkd_run_info(r, i, C.byref(info)))
            lh = np.zeros(max(info.n_loss, 1), np.float64)
            check(L.pbkd_run_loss_history(r, i, _ptr(lh), info.n_loss))
            ep = np.zeros(max(info.n_eval, 1), np.int32)
            acc = np.zeros(max(info.n_eval, 1), np.float64)
            check(L.pbkd_run_eval_history(r, i, _ptr(ep), _ptr(acc), info.n_eval))
            final = np.zeros(info.n_block_floats, np.float32)
            best = np.zeros(info.n_block_floats, np.float32) if info.has_best else None
            if info.n_block_floats:
                check(L.pbkd_run_block(r, i, 1, _ptr(final), final.size))
                if best is not None:
                    check(L.pbkd_run_block(r, i, 0, _ptr(best), best.size))
            steps = np.zeros(max(info.n_steps, 1), np.float32)
            check(L.pbkd_run_step_losses(r, i, _ptr(steps), info.n_steps))
            res.append({
                "block_index": info.block_index, "kind": info.kind.decode(),
                "failed": bool(info.failed), "failure": info.failure.decode(),
                "loss_history": lh[:info.n_loss].tolist(),
                "eval_history": [(int(e), float(a)) for e, a in zip(ep[:info.n_eval],
                                                                     acc[:info.n_eval])],
                "final_local_loss": info.final_local_loss, "best_eval": info.best_eval,
                "block": best, "final_block": final, "step_losses": steps[:info.n_steps].copy(),
                "wall_time_s": info.wall_time_s,
            })
        n = C.c_int()
        check(L.pbkd_run_trace(r, None, 0, C.byref(n)))
        ev = (TraceEvent * max(n.value, 1))()
        check(L.pbkd_run_trace(r, ev, n.value, C.byref(n)))
        trace = [(e.timestamp_s, e.worker_id, e.task_id, e.kind) for e in ev[:n.value]]
        tms, tep, nl, ne = C.c_double(), C.c_int(), C.c_longlong(), C.c_int()
        check(L.pbkd_run_timing(r, C.byref(tms), C.byref(tep), C.byref(nl), None, 0, C.byref(ne)))
        ems = np.zeros(max(ne.value, 1), np.float64)
        check(L.pbkd_run_timing(r, None, None, None, _ptr(ems), ne.value, C.byref(ne)))
        tt = np.zeros(1, np.float64)
        check(L.pbkd_run_timing(r, None, None, None, _ptr(tt), -1, C.byref(ne)))
        prof = {}
        for i in range(L.pbkd_run_profile_count(r)):
            name = C.create_string_buffer(64)
            nlch, ms, by, fl = C.c_int(), C.c_double(), C.c_double(), C.c_double()
            check(L.pbkd_run_profile_entry(r, i, name, 64, C.byref(nlch), C.byref(ms), C.byref(by), C.byref(fl)))
            prof[name.value.decode()] = {"launches": nlch.value, "ms": ms.value, "bytes": by.value,
                                         "flops": fl.value}
        return {"results": res, "trace": trace, "wall_time_s": L.pbkd_run_wall_time(r),
                "epoch_ms": L.pbkd_run_epoch_ms(r), "timed_ms": tms.value,
                "teacher_ms": float(tt[0]),
                "timed_epochs": tep.value, "launches": nl.value,
                "epoch_ms_list": ems[:ne.value].tolist(), "profile": prof}

    def bench_kernel(self, which, batch, iters=20):
        ms, by, fl = C.c_double(), C.c_double(), C.c_double()
        check(lib().pbkd_bench_kernel(self.h, which, batch, iters, C.byref(ms), C.byref(by),
                                      C.byref(fl)))
        return ms.value, by.value, fl.value

    def prefix_infer(self, x, k, inclusive, out_numel):
        x = _f32(x)
        out = np.zeros(out_numel, np.float32)
        shape = (C.c_int * 4)()
        check(lib().pbkd_prefix_infer(self.h, _ptr(x), x.shape[0], k, int(inclusive), _ptr(out),
                                      out.size, shape))
        shp = tuple(shape)
        return out[:int(np.prod(shp))].reshape(shp)

    def candidate_infer(self, kind, cin, cout, stride, bw, x):
        x, bw = _f32(x), _f32(bw)
        n, _, h, w = x.shape
        ho, wo = (h - 1) // stride + 1, (w - 1) // stride + 1
        out = np.zeros((n, cout, ho, wo), np.float32)
        check(lib().pbkd_candidate_infer(self.h, kind, cin, cout, stride, _ptr(bw), _ptr(x), n, h,
                                         w, _ptr(out), out.size))
        return out

    def fit_assembled(self, spec, teacher_w, reps, train_idx, eval_idx, epochs, freeze, lr, momentum, batch,
                      seed, teacher_mode=False, cap=1 << 24):
        """reassemble + finetune (or train_teacher) on the GPU (pbkd_fit_assembled).
        reps: [(block_index, kind, candidate_weights), ...]"""
        tw = _f32(teacher_w)
        blocks = _i32([r[0] for r in reps] or [0])
        kinds = _i32([r[1] for r in reps] or [0])
        cw = _f32(np.concatenate([np.asarray(r[2], np.float32) for r in reps]) if reps else np.zeros(1))
        tr, ev = _i32(train_idx), _i32(eval_idx)
        lh = np.zeros(max(epochs, 1), np.float64)
        ee = np.zeros(epochs + 1, np.int32)
        ea = np.zeros(epochs + 1, np.float64)
        ne = C.c_int()
        init, fin = C.c_double(), C.c_double()
        out = np.zeros(cap, np.float32)
        n_out = C.c_size_t()
        check(lib().pbkd_fit_assembled(self.h, spec.encode(), _ptr(tw), tw.size, _ptr(blocks), _ptr(kinds),
                                       _ptr(cw), len(reps), _ptr(tr), len(tr), _ptr(ev), len(ev), epochs,
                                       int(freeze), lr, momentum, batch, seed, int(teacher_mode), C.byref(init),
                                       C.byref(fin), _ptr(lh), _ptr(ee), _ptr(ea), C.byref(ne), _ptr(out),
                                       out.size, C.byref(n_out)))
        n = ne.value
        return {"loss_history": lh[:max(n - 1, 0)], "eval_history": list(zip(ee[:n].tolist(), ea[:n].tolist())),
                "initial_eval": init.value, "final_eval": fin.value, "net": out[:n_out.value].copy()}

    def eval_with_student(self, k, kind, sw, eval_idx, batch_size):
        sw, ev = _f32(sw), _i32(eval_idx)
        acc = C.c_double()
        check(lib().pbkd_eval_with_student(self.h, k, kind, _ptr(sw), _ptr(ev), len(ev),
                                           batch_size, C.byref(acc)))
        return acc.value

    # kernel level: arguments are raw device pointers (ints)
    def k(self, name, *args):
        vp = C.c_void_p
        conv = [vp(a) if isinstance(a, DevPtr) else a for a in args]
        check(getattr(lib(), "pbkd_k_" + name)(self.h, *conv))


class DevPtr(int):
    """Marks an integer as a device address for Context.k()."""
