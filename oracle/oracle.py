"""ctypes front end for the CPU oracles -- TEST INFRASTRUCTURE ONLY.

`Oracle("orc")` loads oracle/liboracle.so (the from-scratch restatement of the
reference, oracle/pbkd_oracle.cpp); `Oracle("ref")` loads
oracle/_ref/libpbkd_ref.so (the reference itself, built from
/root/reference/proj by oracle/Makefile; only present where that tree was
available at build time).  Both expose the C ABI in oracle/oracle_api.h.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may use
this module.  The product package never imports it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIBS = {"orc": os.path.join(HERE, "liboracle.so"),
        "ref": os.path.join(HERE, "_ref", "libpbkd_ref.so")}

F32P = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
I32P = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
F64P = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")

KINDS = {"two_layer": 0, "three_layer": 1, "two_layer_skip": 2, "three_layer_skip": 3}


class Task(C.Structure):
    _fields_ = [("block_index", C.c_int), ("kind", C.c_int), ("epochs", C.c_int),
                ("eval_every", C.c_int), ("seed", C.c_uint64), ("threshold", C.c_double),
                ("loss_mode", C.c_int), ("lambda_local", C.c_float), ("lr", C.c_float),
                ("momentum", C.c_float), ("batch_size", C.c_int), ("max_steps", C.c_longlong)]


def make_task(block_index, kind=0, epochs=30, eval_every=2, seed=0, threshold=0.0, loss_mode=0,
              lambda_local=1.0, lr=0.05, momentum=0.9, batch_size=50, max_steps=0):
    """Defaults follow pbkd::DistillTask (distill.hpp:24-37)."""
    return Task(block_index, kind, epochs, eval_every, seed, threshold, loss_mode, lambda_local,
                lr, momentum, batch_size, max_steps)


class Dataset(C.Structure):
    _fields_ = [("images", C.c_void_p), ("labels", C.c_void_p), ("count", C.c_int),
                ("c", C.c_int), ("h", C.c_int), ("w", C.c_int), ("classes", C.c_int)]


class Split(C.Structure):
    _fields_ = [("train_idx", C.c_void_p), ("n_train", C.c_int), ("eval_idx", C.c_void_p),
                ("n_eval", C.c_int)]


class Result(C.Structure):
    _fields_ = [("loss_history", C.c_double * 256), ("n_loss", C.c_int),
                ("eval_epoch", C.c_int * 256), ("eval_acc", C.c_double * 256),
                ("n_eval", C.c_int), ("final_local_loss", C.c_double), ("best_eval", C.c_double),
                ("failed", C.c_int), ("failure", C.c_char * 256)]


def build():
    """Compile both oracles (make -C oracle); the reference one only where its tree exists."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def available(prefix: str) -> bool:
    return os.path.exists(LIBS[prefix])


class Oracle:
    def __init__(self, prefix: str = "orc"):
        if not available(prefix):
            raise FileNotFoundError(f"{LIBS[prefix]} not built (make -C oracle)")
        self.p = prefix
        self.lib = C.CDLL(LIBS[prefix])
        self._keep = []

    def fn(self, name, restype, argtypes):
        f = getattr(self.lib, f"{self.p}_{name}")
        f.restype = restype
        f.argtypes = argtypes
        return f

    def _check(self, rc):
        if rc != 0:
            err = self.fn("last_error", C.c_char_p, [])()
            raise RuntimeError(f"{self.p}: {err.decode()}")

    # ---- seeds / indexing -------------------------------------------------
    def mix_seed(self, a, b):
        return self.fn("mix_seed", C.c_uint64, [C.c_uint64, C.c_uint64])(a, b)

    def shuffle(self, idx, seed):
        a = np.ascontiguousarray(idx, np.int32).copy()
        self.fn("shuffle", None, [I32P, C.c_int, C.c_uint64])(a, len(a), seed)
        return a

    def stratified_split(self, labels, frac, seed):
        lab = np.ascontiguousarray(labels, np.int32)
        tr = np.zeros(len(lab), np.int32)
        ev = np.zeros(len(lab), np.int32)
        nt, ne = C.c_int(), C.c_int()
        f = self.fn("stratified_split", C.c_int, [I32P, C.c_int, C.c_double, C.c_uint64, I32P,
                                                   C.POINTER(C.c_int), I32P, C.POINTER(C.c_int)])
        self._check(f(lab, len(lab), frac, seed, tr, C.byref(nt), ev, C.byref(ne)))
        return tr[:nt.value].copy(), ev[:ne.value].copy()

    def synthetic_dataset(self, count, seed, threads=1):
        img = np.zeros(count * 3 * 16 * 16, np.float32)
        lab = np.zeros(count, np.int32)
        f = self.fn("synthetic_dataset", C.c_int, [C.c_int, C.c_uint64, C.c_int, F32P, I32P])
        self._check(f(count, seed, threads, img, lab))
        return img.reshape(count, 3, 16, 16), lab

    # ---- scheduling -------------------------------------------------------
    def _plan(self, out_ids, counts):
        plan, at = [], 0
        for c in counts:
            plan.append([int(v) for v in out_ids[at:at + c]])
            at += c
        return plan

    def round_robin(self, ids, workers):
        ids = np.ascontiguousarray(ids, np.int32)
        out, cnt = np.zeros(len(ids), np.int32), np.zeros(workers, np.int32)
        f = self.fn("round_robin", C.c_int, [I32P, C.c_int, C.c_int, I32P, I32P])
        self._check(f(ids, len(ids), workers, out, cnt))
        return self._plan(out, cnt)

    def wfd(self, ids, weights, workers):
        ids = np.ascontiguousarray(ids, np.int32)
        w = np.ascontiguousarray(weights, np.float64)
        out, cnt = np.zeros(len(ids), np.int32), np.zeros(workers, np.int32)
        mk = C.c_double()
        f = self.fn("wfd", C.c_int, [I32P, F64P, C.c_int, C.c_int, I32P, I32P,
                                     C.POINTER(C.c_double)])
        self._check(f(ids, w, len(ids), workers, out, cnt, C.byref(mk)))
        return self._plan(out, cnt), mk.value

    # ---- model ------------------------------------------------------------
    def teacher_num_floats(self, spec):
        n = C.c_size_t()
        self._check(self.fn("teacher_num_floats", C.c_int, [C.c_char_p, C.POINTER(C.c_size_t)])(
            spec.encode(), C.byref(n)))
        return n.value

    def teacher_num_blocks(self, spec):
        n = C.c_int()
        self._check(self.fn("teacher_num_blocks", C.c_int, [C.c_char_p, C.POINTER(C.c_int)])(
            spec.encode(), C.byref(n)))
        return n.value

    def teacher_init(self, spec, seed):
        n = self.teacher_num_floats(spec)
        out = np.zeros(n, np.float32)
        self._check(self.fn("teacher_init", C.c_int, [C.c_char_p, C.c_uint64, F32P, C.c_size_t])(
            spec.encode(), seed, out, n))
        return out

    def block_macs(self, spec, k):
        m = C.c_longlong()
        self._check(self.fn("block_macs", C.c_int, [C.c_char_p, C.c_int,
                                                     C.POINTER(C.c_longlong)])(
            spec.encode(), k, C.byref(m)))
        return m.value

    def candidate_num_floats(self, kind, cin, cout, stride):
        n = C.c_size_t()
        self._check(self.fn("candidate_num_floats", C.c_int,
                            [C.c_int, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_size_t)])(
            kind, cin, cout, stride, C.byref(n)))
        return n.value

    def build_candidate(self, kind, cin, cout, stride, seed):
        n = self.candidate_num_floats(kind, cin, cout, stride)
        out = np.zeros(n, np.float32)
        self._check(self.fn("build_candidate", C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int,
                                                          C.c_uint64, F32P, C.c_size_t])(
            kind, cin, cout, stride, seed, out, n))
        return out

    # ---- kernels (NCHW) ---------------------------------------------------
    def dw_fwd(self, x, k, stride, pad):
        n, c, h, w = x.shape
        kk = k.shape[-1]
        ho, wo = (h + 2 * pad - kk) // stride + 1, (w + 2 * pad - kk) // stride + 1
        y = np.zeros((n, c, ho, wo), np.float32)
        self.fn("dw_fwd", None, [F32P] + [C.c_int] * 4 + [F32P] + [C.c_int] * 3 + [F32P])(
            np.ascontiguousarray(x, np.float32), n, c, h, w, np.ascontiguousarray(k, np.float32),
            kk, stride, pad, y)
        return y

    def dw_bwd(self, x, k, gy, stride, pad):
        n, c, h, w = x.shape
        kk = k.shape[-1]
        gx = np.zeros_like(x, dtype=np.float32)
        gk = np.zeros((c, 1, kk, kk), np.float32)
        self.fn("dw_bwd", None, [F32P] + [C.c_int] * 4 + [F32P] + [C.c_int] * 3 + [F32P] * 3)(
            np.ascontiguousarray(x, np.float32), n, c, h, w, np.ascontiguousarray(k, np.float32),
            kk, stride, pad, np.ascontiguousarray(gy, np.float32), gx, gk)
        return gx, gk

    def pw_fwd(self, x, k, stride=1):
        n, c, h, w = x.shape
        co = k.shape[0]
        ho, wo = (h - 1) // stride + 1, (w - 1) // stride + 1
        y = np.zeros((n, co, ho, wo), np.float32)
        self.fn("pw_fwd", None, [F32P] + [C.c_int] * 4 + [F32P, C.c_int, C.c_int, F32P])(
            np.ascontiguousarray(x, np.float32), n, c, h, w, np.ascontiguousarray(k, np.float32),
            co, stride, y)
        return y

    def pw_bwd(self, x, k, gy, stride=1):
        n, c, h, w = x.shape
        co = k.shape[0]
        gx = np.zeros_like(x, dtype=np.float32)
        gk = np.zeros((co, c, 1, 1), np.float32)
        self.fn("pw_bwd", None, [F32P] + [C.c_int] * 4 + [F32P, C.c_int, C.c_int] + [F32P] * 3)(
            np.ascontiguousarray(x, np.float32), n, c, h, w, np.ascontiguousarray(k, np.float32),
            co, stride, np.ascontiguousarray(gy, np.float32), gx, gk)
        return gx, gk

    def conv_fwd(self, x, k, stride, pad):
        n, c, h, w = x.shape
        co, _, kk, _ = k.shape
        ho, wo = (h + 2 * pad - kk) // stride + 1, (w + 2 * pad - kk) // stride + 1
        y = np.zeros((n, co, ho, wo), np.float32)
        self.fn("conv_fwd", None, [F32P] + [C.c_int] * 4 + [F32P] + [C.c_int] * 4 + [F32P])(
            np.ascontiguousarray(x, np.float32), n, c, h, w, np.ascontiguousarray(k, np.float32),
            co, kk, stride, pad, y)
        return y

    def bn_train_fwd(self, x, gamma, beta, mm, mv, momentum=0.9):
        n, c, h, w = x.shape
        y = np.zeros_like(x, dtype=np.float32)
        xhat = np.zeros_like(x, dtype=np.float32)
        inv = np.zeros(c, np.float32)
        mm, mv = np.array(mm, np.float32), np.array(mv, np.float32)
        self.fn("bn_train_fwd", None, [F32P] + [C.c_int] * 4 + [F32P] * 4 + [C.c_float] +
                [F32P] * 3)(np.ascontiguousarray(x, np.float32), n, c, h, w,
                            np.ascontiguousarray(gamma, np.float32),
                            np.ascontiguousarray(beta, np.float32), mm, mv, momentum, y, xhat, inv)
        return y, xhat, inv, mm, mv

    def bn_train_bwd(self, xhat, inv, gamma, gy):
        n, c, h, w = xhat.shape
        gx = np.zeros_like(xhat, dtype=np.float32)
        gg, gb = np.zeros(c, np.float32), np.zeros(c, np.float32)
        self.fn("bn_train_bwd", None, [F32P] * 4 + [C.c_int] * 4 + [F32P] * 3)(
            np.ascontiguousarray(xhat, np.float32), np.ascontiguousarray(inv, np.float32),
            np.ascontiguousarray(gamma, np.float32), np.ascontiguousarray(gy, np.float32),
            n, c, h, w, gx, gg, gb)
        return gx, gg, gb

    def mse(self, s, t):
        s = np.ascontiguousarray(s, np.float32).ravel()
        t = np.ascontiguousarray(t, np.float32).ravel()
        return self.fn("mse", C.c_float, [F32P, F32P, C.c_size_t])(s, t, s.size)

    def mse_bwd(self, s, t, scale=1.0):
        s = np.ascontiguousarray(s, np.float32).ravel()
        t = np.ascontiguousarray(t, np.float32).ravel()
        g = np.zeros_like(s)
        self.fn("mse_bwd", None, [F32P, F32P, C.c_size_t, C.c_float, F32P])(s, t, s.size,
                                                                             scale, g)
        return g

    def sgd(self, w, g, v, lr, momentum):
        w, v = np.array(w, np.float32), np.array(v, np.float32)
        self.fn("sgd", None, [F32P, F32P, F32P, C.c_size_t, C.c_float, C.c_float])(
            w, np.ascontiguousarray(g, np.float32), v, w.size, lr, momentum)
        return w, v

    # ---- block / network --------------------------------------------------
    def prefix_infer(self, spec, tw, x, k, inclusive):
        cap = 1 << 26
        out = np.zeros(cap, np.float32)
        shape = (C.c_int * 4)()
        f = self.fn("prefix_infer", C.c_int, [C.c_char_p, F32P, F32P, C.c_int, C.c_int, C.c_int,
                                               F32P, C.c_size_t, C.c_int * 4])
        self._check(f(spec.encode(), np.ascontiguousarray(tw, np.float32),
                      np.ascontiguousarray(x, np.float32), x.shape[0], k, int(inclusive), out,
                      cap, shape))
        shp = tuple(shape)
        return out[:int(np.prod(shp))].reshape(shp).copy()

    def candidate_infer(self, kind, cin, cout, stride, bw, x):
        n, _, h, w = x.shape
        ho, wo = (h - 1) // stride + 1, (w - 1) // stride + 1
        out = np.zeros((n, cout, ho, wo), np.float32)
        f = self.fn("candidate_infer", C.c_int, [C.c_int] * 4 + [F32P, F32P] + [C.c_int] * 3 +
                    [F32P, C.c_size_t])
        self._check(f(kind, cin, cout, stride, np.ascontiguousarray(bw, np.float32),
                      np.ascontiguousarray(x, np.float32), n, h, w, out, out.size))
        return out

    def _ds(self, images, labels, classes=10):
        images = np.ascontiguousarray(images, np.float32)
        labels = np.ascontiguousarray(labels, np.int32)
        self._keep = [images, labels]
        n, c, h, w = images.shape
        return Dataset(images.ctypes.data, labels.ctypes.data, n, c, h, w, classes)

    def _split(self, train_idx, eval_idx):
        tr = np.ascontiguousarray(train_idx, np.int32)
        ev = np.ascontiguousarray(eval_idx, np.int32)
        self._keep_split = [tr, ev]
        return Split(tr.ctypes.data, len(tr), ev.ctypes.data, len(ev))

    def eval_with_student(self, spec, tw, images, labels, eval_idx, k, kind, sw, batch_size):
        ds = self._ds(images, labels)
        ev = np.ascontiguousarray(eval_idx, np.int32)
        acc = C.c_double()
        f = self.fn("eval_with_student", C.c_int, [C.c_char_p, F32P, C.POINTER(Dataset), I32P,
                                                    C.c_int, C.c_int, C.c_int, F32P, C.c_int,
                                                    C.POINTER(C.c_double)])
        self._check(f(spec.encode(), np.ascontiguousarray(tw, np.float32), C.byref(ds), ev,
                      len(ev), k, kind, np.ascontiguousarray(sw, np.float32), batch_size,
                      C.byref(acc)))
        return acc.value

    def train_block(self, spec, tw, images, labels, train_idx, eval_idx, task, n_block_floats,
                    with_f64=False):
        """with_f64 (orc only): also "loss_history64", every entry's batch MSEs
        summed in fp64 over the same outputs."""
        ds = self._ds(images, labels)
        sp = self._split(train_idx, eval_idx)
        res = Result()
        bw = np.zeros(max(n_block_floats, 1), np.float32)
        h64 = np.zeros(256, np.float64)
        if with_f64:
            f = self.fn("train_block_f64", C.c_int, [C.c_char_p, F32P, C.POINTER(Dataset),
                                                      C.POINTER(Split), C.POINTER(Task),
                                                      C.POINTER(Result), F32P, C.c_size_t, F64P])
            self._check(f(spec.encode(), np.ascontiguousarray(tw, np.float32), C.byref(ds),
                          C.byref(sp), C.byref(task), C.byref(res), bw, bw.size, h64))
        else:
            f = self.fn("train_block", C.c_int, [C.c_char_p, F32P, C.POINTER(Dataset),
                                                  C.POINTER(Split), C.POINTER(Task),
                                                  C.POINTER(Result), F32P, C.c_size_t])
            self._check(f(spec.encode(), np.ascontiguousarray(tw, np.float32), C.byref(ds),
                          C.byref(sp), C.byref(task), C.byref(res), bw, bw.size))
        return {"loss_history64": h64[:res.n_loss].tolist(),
            "loss_history": [res.loss_history[i] for i in range(res.n_loss)],
            "eval_history": [(res.eval_epoch[i], res.eval_acc[i]) for i in range(res.n_eval)],
            "final_local_loss": res.final_local_loss, "best_eval": res.best_eval,
            "failed": bool(res.failed), "failure": res.failure.decode(), "block": bw,
        }

    def train_replay(self, spec, tw, images, labels, train_idx, eval_idx, task, n_steps,
                     n_block_floats, with_f64=False):
        """Returns (float losses, final weights) or, with_f64, also the fp64 losses."""
        ds = self._ds(images, labels)
        sp = self._split(train_idx, eval_idx)
        losses = np.zeros(n_steps, np.float32)
        l64 = np.zeros(n_steps, np.float64)
        fw = np.zeros(n_block_floats, np.float32)
        f = self.fn("train_replay_f64", C.c_int, [C.c_char_p, F32P, C.POINTER(Dataset),
                                                   C.POINTER(Split), C.POINTER(Task), C.c_int,
                                                   F32P, F64P, F32P, C.c_size_t])
        self._check(f(spec.encode(), np.ascontiguousarray(tw, np.float32), C.byref(ds),
                      C.byref(sp), C.byref(task), n_steps, losses, l64, fw, fw.size))
        return (losses, fw, l64) if with_f64 else (losses, fw)

    def train_replay_multi(self, spec, tw, images, labels, train_idx, eval_idx, tasks, n_steps,
                           n_floats, ck_steps=(), threads=None):
        """Grouped replay (orc only): every task's per-step float losses and
        fp64 losses [n_tasks, n_steps], and per task a [len(ck_steps), nf]
        array of student weights after each checkpoint step."""
        ds = self._ds(images, labels)
        sp = self._split(train_idx, eval_idx)
        nt = len(tasks)
        ck = np.ascontiguousarray(sorted(ck_steps) or [n_steps], np.int32)
        off = np.zeros(nt + 1, np.uint64)
        for i, nf in enumerate(n_floats):
            off[i + 1] = off[i] + nf * len(ck)
        buf = np.zeros(max(int(off[-1]), 1), np.float32)
        losses = np.zeros((nt, n_steps), np.float32)
        l64 = np.zeros((nt, n_steps), np.float64)
        arr = (Task * nt)(*tasks)
        f = self.fn("train_replay_multi", C.c_int,
                    [C.c_char_p, F32P, C.POINTER(Dataset), C.POINTER(Split), C.POINTER(Task), C.c_int,
                     C.c_int, I32P, C.c_int, C.c_int, F32P, F64P, F32P,
                     np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")])
        self._check(f(spec.encode(), np.ascontiguousarray(tw, np.float32), C.byref(ds), C.byref(sp), arr,
                      nt, n_steps, ck, len(ck), threads or os.cpu_count() or 1, losses, l64, buf, off))
        snaps = [buf[int(off[i]):int(off[i + 1])].reshape(len(ck), n_floats[i]) for i in range(nt)]
        return losses, l64, snaps

    def run_parallel(self, spec, tw, images, labels, train_idx, eval_idx, tasks, plan, n_floats,
                     policy=0):
        """run_parallel (runtime.cpp:124-243); results in ascending block order,
        n_floats per result in that order."""
        ds = self._ds(images, labels)
        sp = self._split(train_idx, eval_idx)
        nt = len(tasks)
        ids = np.ascontiguousarray([i for q in plan for i in q], np.int32)
        counts = np.ascontiguousarray([len(q) for q in plan], np.int32)
        off = np.zeros(nt + 1, np.uint64)
        for i, nf in enumerate(n_floats):
            off[i + 1] = off[i] + nf
        buf = np.zeros(max(int(off[-1]), 1), np.float32)
        res = (Result * nt)()
        arr = (Task * nt)(*tasks)
        f = self.fn("run_parallel", C.c_int,
                    [C.c_char_p, F32P, C.POINTER(Dataset), C.POINTER(Split), C.POINTER(Task), C.c_int,
                     I32P, I32P, C.c_int, C.c_int, C.POINTER(Result), F32P,
                     np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")])
        self._check(f(spec.encode(), np.ascontiguousarray(tw, np.float32), C.byref(ds), C.byref(sp), arr, nt,
                      ids, counts, len(plan), policy, res, buf, off))
        out = []
        for i in range(nt):
            r = res[i]
            out.append({"loss_history": [r.loss_history[q] for q in range(r.n_loss)],
                        "eval_history": [(r.eval_epoch[q], r.eval_acc[q]) for q in range(r.n_eval)],
                        "final_local_loss": r.final_local_loss, "best_eval": r.best_eval,
                        "failed": bool(r.failed), "failure": r.failure.decode(),
                        "block": buf[int(off[i]):int(off[i + 1])].copy()})
        return out

    def fit_network(self, spec, tw, images, labels, train_idx, eval_idx, reps, epochs, freeze, lr, momentum,
                    batch, seed, teacher_mode, cap=1 << 22):
        """ref only: finetune / train_teacher of the teacher with blocks
        reps = [(k, kind, cand_seed), ...] swapped in (reassemble)."""
        ds = self._ds(images, labels)
        sp = self._split(train_idx, eval_idx)
        ks = np.ascontiguousarray([r[0] for r in reps] or [0], np.int32)
        kinds = np.ascontiguousarray([r[1] for r in reps] or [0], np.int32)
        seeds = np.ascontiguousarray([r[2] for r in reps] or [0], np.uint64)
        lh = np.zeros(max(epochs, 1), np.float64)
        ea = np.zeros(epochs + 1, np.float64)
        ne = C.c_int()
        inf = np.zeros(2, np.float64)
        out = np.zeros(cap, np.float32)
        U64P = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
        f = self.fn("fit_network", C.c_int,
                    [C.c_char_p, F32P, I32P, I32P, U64P, C.c_int, C.POINTER(Dataset), C.POINTER(Split), C.c_int,
                     C.c_int, C.c_float, C.c_float, C.c_int, C.c_uint64, C.c_int, F64P, F64P, C.POINTER(C.c_int),
                     F64P, F32P, C.c_size_t])
        self._check(f(spec.encode(), np.ascontiguousarray(tw, np.float32), ks, kinds, seeds, len(reps), C.byref(ds),
                      C.byref(sp), epochs, int(freeze), lr, momentum, batch, seed, int(teacher_mode), lh, ea,
                      C.byref(ne), inf, out, out.size))
        n = ne.value
        return {"loss_history": lh[:max(n - 1, 0)], "eval_history": ea[:n], "initial_eval": inf[0],
                "final_eval": inf[1], "net": out}
