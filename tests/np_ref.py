"""float64 numpy teacher forward (test-only accuracy yardstick).

Same graph as the reference (model.cpp:83-119 blocks, ops.hpp:37-75 conv,
ops.hpp:304-321 inference batch norm, :460-466 add), evaluated in float64 so
that both the CPU oracle (serial fp32) and the GPU path (tensor cores) can be
measured against the exact result instead of against each other.
"""
import json

import numpy as np


def conv(x, w, stride, pad):
    n, c, h, wd = x.shape
    co, ci, k, _ = w.shape
    ho, wo = (h + 2 * pad - k) // stride + 1, (wd + 2 * pad - k) // stride + 1
    xp = np.zeros((n, c, h + 2 * pad, wd + 2 * pad))
    xp[:, :, pad:pad + h, pad:pad + wd] = x
    cols = np.empty((n, c, k, k, ho, wo))
    for ky in range(k):
        for kx in range(k):
            cols[:, :, ky, kx] = xp[:, :, ky:ky + stride * ho:stride, kx:kx + stride * wo:stride]
    return np.einsum("ncijhw,ocij->nohw", cols, w, optimize=True)


def bn_infer(x, g, b, mm, mv):
    s = g / np.sqrt(mv + 1e-5)
    return x * s[None, :, None, None] + (b - mm * s)[None, :, None, None]


def prefix_f64(spec_text, tw, x, k):
    """Blocks 1..k (inclusive) of the teacher in float64."""
    spec = json.loads(spec_text)
    tw = np.asarray(tw, np.float64)
    at = 0

    def take(*shape):
        nonlocal at
        n = int(np.prod(shape))
        v = tw[at:at + n].reshape(shape)
        at += n
        return v

    cur = np.asarray(x, np.float64)
    c = spec["input_shape"][0]
    for bi, b in enumerate(spec["blocks"]):
        co, s = b["out_channels"], b.get("stride", 1)
        kind = b["kind"]
        if kind in ("conv3x3", "conv1x1"):
            kk = 3 if kind == "conv3x3" else 1
            p = b.get("padding", 1 if kk == 3 else 0)
            w = take(co, c, kk, kk)
            g, be, mm, mv = take(co), take(co), take(co), take(co)
            y = np.maximum(bn_infer(conv(cur, w, s, p), g, be, mm, mv), 0)
        else:
            p = b.get("padding", 1)
            w1 = take(co, c, 3, 3)
            g1, b1, m1, v1 = take(co), take(co), take(co), take(co)
            w2 = take(co, co, 3, 3)
            g2, b2, m2, v2 = take(co), take(co), take(co), take(co)
            skip = cur
            if c != co or s != 1:
                skip = conv(cur, take(co, c, 1, 1), s, 0)
            t = np.maximum(bn_infer(conv(cur, w1, s, p), g1, b1, m1, v1), 0)
            y = np.maximum(bn_infer(conv(t, w2, 1, 1), g2, b2, m2, v2) + skip, 0)
        cur, c = y, co
        if bi + 1 == k:
            return cur
    return cur
