"""TEST INFRASTRUCTURE: the distillation step in float64 PyTorch (on the GPU).

The reference computes every reduction as a serial fp32 sum (ops.hpp; SURVEY
Appendix B), so its own trajectory carries rounding error that grows with the
step count.  This module recomputes the same trajectory in float64 -- teacher
boundaries (conv3x3 + inference BN + ReLU, residual add with the 1x1 stride
projection; model.cpp:83-119, :498-557), the depthwise-separable candidate
(replacement.cpp:11-16, 59-63) in train-mode BN with the reference's biased
variance E[x^2]-mean^2 clamped at 0 (ops.hpp:261-301), MSE (ops.hpp:518-539),
backward by autograd (the exact derivative the reference's closed forms
implement), SGD with momentum (ops.hpp:545-558) -- from the same float32
inputs (teacher weights, candidate init, images) and the same batches, so
that GPU and reference can both be measured against it.

Only tests/ use this; it is never on the product path.
"""
import json

import numpy as np
import torch
import torch.nn.functional as F

F64 = torch.float64
EPS = float(np.float32(1e-5))       # static_cast<float>(kEps), ops.hpp:245
MOM = float(np.float32(0.9))        # kBnMomentum, model.cpp:15
ONE_MINUS_MOM = float(np.float32(1.0) - np.float32(0.9))


def _teacher(spec, tw, dev):
    """Teacher blocks as lists of float64 tensors, for_each_array order."""
    d = json.loads(spec)
    w = torch.from_numpy(np.asarray(tw, np.float32)).to(dev, F64)
    at = 0

    def take(*shape):
        nonlocal at
        n = int(np.prod(shape))
        t = w[at:at + n].reshape(shape)
        at += n
        return t

    c = d["input_shape"][0]
    blocks = []
    for b in d["blocks"]:
        co, s = b["out_channels"], b.get("stride", 1)
        ks = 1 if b["kind"] == "conv1x1" else 3
        pad = b.get("padding", 0 if ks == 1 else 1)  # model.cpp:281
        if b["kind"] == "bottleneck":  # model.cpp build_bottleneck
            mid = max(1, co // 4)
            blk = {"kind": "bottleneck", "s": s, "w1": take(mid, c, 1, 1), "bn1": [take(mid) for _ in range(4)],
                   "w2": take(mid, mid, 3, 3), "bn2": [take(mid) for _ in range(4)],
                   "w3": take(co, mid, 1, 1), "bn3": [take(co) for _ in range(4)]}
            blk["proj"] = take(co, c, 1, 1) if (s != 1 or c != co) else None
        elif b["kind"] == "stem7x7":
            blk = {"kind": "stem", "s": s, "w1": take(co, c, 7, 7), "bn1": [take(co) for _ in range(4)]}
        elif b["kind"] == "residual3x3":
            blk = {"kind": "res", "s": s, "p": pad, "w1": take(co, c, 3, 3), "bn1": [take(co) for _ in range(4)],
                   "w2": take(co, co, 3, 3), "bn2": [take(co) for _ in range(4)]}
            blk["proj"] = take(co, c, 1, 1) if (s != 1 or c != co) else None  # model.cpp:211-219
        else:
            blk = {"kind": "conv", "s": s, "p": pad, "w1": take(co, c, ks, ks), "bn1": [take(co) for _ in range(4)]}
        blocks.append(blk)
        c = co
    return blocks


def _bn_infer(x, bn):
    g, b, mm, mv = bn
    return g[None, :, None, None] * (x - mm[None, :, None, None]) / torch.sqrt(mv + EPS)[None, :, None, None] \
        + b[None, :, None, None]


def _teacher_block(blk, x):
    if blk["kind"] == "bottleneck":
        y = F.relu(_bn_infer(F.conv2d(x, blk["w1"]), blk["bn1"]))
        y = F.relu(_bn_infer(F.conv2d(y, blk["w2"], stride=blk["s"], padding=1), blk["bn2"]))
        y = _bn_infer(F.conv2d(y, blk["w3"]), blk["bn3"])
        skip = x if blk["proj"] is None else F.conv2d(x, blk["proj"], stride=blk["s"])
        return F.relu(y + skip)
    if blk["kind"] == "stem":
        y = F.relu(_bn_infer(F.conv2d(x, blk["w1"], stride=blk["s"], padding=3), blk["bn1"]))
        return F.max_pool2d(y, 3, stride=2, padding=1)
    y = F.relu(_bn_infer(F.conv2d(x, blk["w1"], stride=blk["s"], padding=blk["p"]), blk["bn1"]))
    if blk["kind"] == "conv":
        return y
    y = _bn_infer(F.conv2d(y, blk["w2"], padding=1), blk["bn2"])
    skip = x if blk["proj"] is None else F.conv2d(x, blk["proj"], stride=blk["s"])
    return F.relu(y + skip)


@torch.no_grad()
def boundaries(spec, tw, images, upto, dev="cuda", chunk=128):
    """Boundary j = 0..upto of every image, float64 [N, C, H, W] on dev."""
    blocks = _teacher(spec, tw, dev)
    x = torch.from_numpy(np.asarray(images, np.float32)).to(dev, F64)
    out = [[] for _ in range(upto + 1)]
    for i in range(0, x.shape[0], chunk):
        cur = x[i:i + chunk]
        out[0].append(cur)
        for j in range(1, upto + 1):
            cur = _teacher_block(blocks[j - 1], cur)
            out[j].append(cur)
    return [torch.cat(o) for o in out]


class Student:
    """A TwoLayer / ThreeLayer candidate from its flat float32 arrays
    (for_each_block_array order: per unit dw, pw, gamma, beta, mm, mv)."""

    def __init__(self, flat, cin, cout, stride, units, dev="cuda"):
        w = torch.from_numpy(np.asarray(flat, np.float32)).to(dev, F64)
        self.stride, self.units, at = stride, units, 0
        self.p, self.stats, self.vel = [], [], []
        for u in range(units):
            ci = cin if u == 0 else cout
            for shape in ((ci, 1, 3, 3), (cout, ci, 1, 1), (cout,), (cout,)):
                n = int(np.prod(shape))
                self.p.append(w[at:at + n].reshape(shape).clone().requires_grad_(True))
                at += n
            self.stats.append([w[at:at + cout].clone(), w[at + cout:at + 2 * cout].clone()])
            at += 2 * cout
        assert at == w.numel()
        self.vel = [torch.zeros_like(t) for t in self.p]

    def step(self, x, t, lr, momentum):
        cur = x
        for u in range(self.units):
            dw, pw, g, b = self.p[4 * u:4 * u + 4]
            cur = F.conv2d(cur, dw, stride=self.stride if u == 0 else 1, padding=1, groups=cur.shape[1])
            cur = F.conv2d(cur, pw)
            mean = cur.mean((0, 2, 3))
            var = torch.clamp((cur * cur).mean((0, 2, 3)) - mean * mean, min=0.0)
            xh = (cur - mean[None, :, None, None]) * (1.0 / torch.sqrt(var + EPS))[None, :, None, None]
            cur = F.relu(g[None, :, None, None] * xh + b[None, :, None, None])
            with torch.no_grad():
                mm, mv = self.stats[u]
                mm.mul_(MOM).add_(ONE_MINUS_MOM * mean)
                mv.mul_(MOM).add_(ONE_MINUS_MOM * var)
        loss = ((cur - t) ** 2).mean()
        grads = torch.autograd.grad(loss, self.p)
        lr, momentum = float(np.float32(lr)), float(np.float32(momentum))
        with torch.no_grad():
            for p, v, gr in zip(self.p, self.vel, grads):
                v.mul_(momentum).add_(gr)
                p.sub_(lr * v)
        return float(loss.detach())

    def flat(self):
        out = []
        for u in range(self.units):
            out += [t.detach().reshape(-1) for t in self.p[4 * u:4 * u + 4]] + [s.reshape(-1) for s in self.stats[u]]
        return torch.cat(out).cpu().numpy()


def replay(orc, spec, tw, images, train_idx, tasks, geo, steps, ck_steps, dev="cuda"):
    """float64 twin of orc.train_replay_multi: per task (losses[steps],
    {step: flat float64 weights})."""
    tr = np.asarray(train_idx)
    upto = max(t.block_index for t in tasks)
    bnd = boundaries(spec, tw, np.asarray(images)[tr], upto, dev)
    out = []
    for t in tasks:
        k = t.block_index
        cin, cout, s = geo[k - 1]
        units = 3 if t.kind == 1 else 2
        st = Student(orc.build_candidate(t.kind, cin, cout, s, orc.mix_seed(t.seed, 0)), cin, cout, s, units, dev)
        losses, snaps, done, epoch = [], {}, 0, 1
        while done < steps:
            pos = orc.shuffle(np.arange(len(tr), dtype=np.int32), orc.mix_seed(t.seed, epoch))
            for at in range(0, len(tr), t.batch_size):
                if done >= steps:
                    break
                b = torch.from_numpy(np.asarray(pos[at:at + t.batch_size], np.int64)).to(dev)
                losses.append(st.step(bnd[k - 1][b], bnd[k][b], t.lr, t.momentum))
                done += 1
                if done in ck_steps:
                    snaps[done] = st.flat()
            epoch += 1
        out.append((np.array(losses), snaps))
    return out
