// dw_tile.cuh -- per-tile depthwise routines on a staged shared-memory tile
// (TMA path: channel counts divisible by 4), used by the depthwise kernels
// of ops.cu.
//
// A tile is ni images x th output rows x all columns x 32 channels; its input
// is staged as [ni][tr][tw][32] floats with the zero halo.  Packed layout:
// lane = (channel pair p = lane % 16, half = lane / 16); the 16 row workers
// (2 * warp + half) walk (output row, x segment) items; two channels per
// FFMA2 (exact rn mul / add, common.cuh).  All routines are called by the
// whole CTA (256 threads) and contain their own barriers.
#pragma once
#include "ops.cuh"
#include "tc.cuh"

namespace pbkd_gpu {

constexpr int kDwC = 32;  // channels per tile
constexpr int kDwLanes = kThreads / kDwC;

struct DwPos {
    int n0, y0, c0, tile;
};
__device__ __forceinline__ DwPos dw_pos(const DwTile& t, int local) {
    DwPos q;
    const int cs = local % t.cslices;
    q.tile = local / t.cslices;
    q.n0 = (q.tile / t.tiles_y) * t.ni;
    q.y0 = (q.tile % t.tiles_y) * t.th;
    q.c0 = cs * kDwC;
    return q;
}

// Vectorised in-place map of the staged in-range pixels (padding stays 0):
// a warp pass covers 4 staged pixels x 8 channel quads (512 contiguous
// bytes); f(v, k) maps channel c0 + 4*quad + k.  Rows walked without
// divisions.  The caller synchronises before and after.
template <class F>
__device__ __forceinline__ void dw_map4(float* buf, const DwTile& t, int n, int h, int w, int n0, int iy0, int ix0,
                                        F f) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, quad = lane & 7, sub = lane >> 3;
    int i = 0, rr = warp;
    while (rr >= t.tr) rr -= t.tr, ++i;
    const int cb = max(0, -ix0), ce = min(t.tw, w - ix0);
    for (; i < t.ni;) {
        const int iy = iy0 + rr;
        if (n0 + i < n && iy >= 0 && iy < h) {
            float4* row = reinterpret_cast<float4*>(buf) + (i * t.tr + rr) * t.tw * (kDwC / 4) + quad;
            for (int col = cb + sub; col < ce; col += 4) {
                float4 v = row[col * (kDwC / 4)];
                v.x = f(v.x, 0), v.y = f(v.y, 1), v.z = f(v.z, 2), v.w = f(v.w, 3);
                row[col * (kDwC / 4)] = v;
            }
        }
        rr += kThreads / 32;
        while (rr >= t.tr) rr -= t.tr, ++i;
    }
}

// Train-mode BN + ReLU of the previous unit (ops.hpp:290-293, 380-385) for
// the vectorised prologue: parameters of channels c0 + 4*quad + k.
struct BnRelu4 {
    float m[4], iv[4], g[4], b[4];
    __device__ void load(const float* mean, const float* inv, const float* gam, const float* bet, int c0, int c) {
        const int quad = threadIdx.x & 7;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int ch = c0 + 4 * quad + k;
            const bool ok = ch < c;
            m[k] = ok ? mean[ch] : 0.0f, iv[k] = ok ? inv[ch] : 0.0f;
            g[k] = ok && gam ? gam[ch] : 0.0f, b[k] = ok && bet ? bet[ch] : 0.0f;
        }
    }
    __device__ __forceinline__ float train(float v, int k) const { return relu(bn_train_apply(v, m[k], iv[k], g[k], b[k])); }
    __device__ __forceinline__ float infer(float v, int k) const { return relu(bn_infer_apply(v, m[k], iv[k])); }
};

// CTA-level fixed-order sum over the 16 packed row workers: thread (row
// worker, pair p) holds v[k] for channels 2p, 2p+1; thread ch < 32 gets out[k].
template <int NV>
__device__ __forceinline__ void dw_lane_sum2(float* red, const float2* v, float* out) {
    const int lane = threadIdx.x & 31, rw = 2 * (threadIdx.x >> 5) + (lane >> 4), p = lane & 15;
#pragma unroll
    for (int k = 0; k < NV; ++k) *reinterpret_cast<float2*>(red + (rw * NV + k) * kDwC + 2 * p) = v[k];
    __syncthreads();
    if (threadIdx.x < kDwC) {
        const int ch = threadIdx.x;
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            float acc = 0.0f;
            for (int l = 0; l < 2 * kDwLanes; ++l) acc += red[(l * NV + k) * kDwC + ch];
            out[k] = acc;
        }
    }
}

// Row-worker geometry of a tile: item = (row, x segment); segment seg of
// width sw covers columns [xb, xe).
struct DwRows {
    int rw, xsh, xb, xe, step;
};
__device__ __forceinline__ DwRows dw_rows(const DwTile& t, int width) {
    DwRows r;
    r.rw = 2 * (threadIdx.x >> 5) + ((threadIdx.x & 31) >> 4);
    r.xsh = t.xsh;
    const int seg = r.rw & ((1 << r.xsh) - 1), sw = (width + (1 << r.xsh) - 1) >> r.xsh;
    r.xb = seg * sw;
    r.xe = min(width, r.xb + sw);
    r.step = (2 * (kThreads / 32)) >> r.xsh;
    return r;
}

// ------------------------------------------------------------ forward tile
// Optional prologue (pro 1: train BN + ReLU, pro 2: inference affine + ReLU)
// in place on xs, then the 9-term serial sums in (ky, kx) order
// (ops.hpp:131-140) per lane, written as fp32 or tf32 hi / lo planes.
// wait(): blocks until the staged tile has landed; called after the tile's
// per-channel parameters are in registers (their loads overlap the staging).
template <class Wait>
__device__ __forceinline__ void dw_fwd_tile(const DwFwdOp& o, const DwPos& q, float* xs, Wait wait) {
    const DwTile& t = o.tile;
    const int n = o.n, h = o.h, w = o.wd, C = o.c, ho = o.ho, wo = o.wo, s = o.stride, pad = o.pad, pro = o.pro;
    const int iy0 = q.y0 * s - pad;
    const int p = threadIdx.x & 15, c2 = q.c0 + 2 * p;
    const bool pok = c2 < C;
    const PkConsts K = pk_consts();
    float2 w2[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) w2[k] = pok ? *reinterpret_cast<const float2*>(o.w + k * C + c2) : K.z;
    BnRelu4 p4;
    if (pro != 0) p4.load(o.pa, o.pb, o.pc, o.pd, q.c0, C);
    wait();
    if (pro != 0) {
        if (pro == 1) dw_map4(xs, t, n, h, w, q.n0, iy0, -pad, [&](float v, int k) { return p4.train(v, k); });
        else dw_map4(xs, t, n, h, w, q.n0, iy0, -pad, [&](float v, int k) { return p4.infer(v, k); });
        __syncthreads();
    }
    if (!pok) return;
    float* const yh = o.y_hi;
    float* const yl = o.y_lo;
    float* const yf = o.y;
    const int rs = t.tw * kDwC;
    const DwRows R = dw_rows(t, wo);
    int i = 0, oy = R.rw >> R.xsh;
    while (oy >= t.th) oy -= t.th, ++i;
    for (; i < t.ni;) {
        const int nn = q.n0 + i, yy = q.y0 + oy;
        if (nn < n && yy < ho) {
            const float* base = xs + ((i * t.tr + oy * s) * t.tw) * kDwC + 2 * p;
            long long off = ((static_cast<long long>(nn) * ho + yy) * wo + R.xb) * C + c2;
            auto ld = [&](int r, int col) { return *reinterpret_cast<const float2*>(base + r * rs + col * kDwC); };
            float2 win[3][3];
            if (s == 1) {
#pragma unroll
                for (int r = 0; r < 3; ++r) win[r][1] = ld(r, R.xb), win[r][2] = ld(r, R.xb + 1);
            }
#pragma unroll 3
            for (int ox = R.xb; ox < R.xe; ++ox, off += C) {
                if (s == 1) {
#pragma unroll
                    for (int r = 0; r < 3; ++r) win[r][0] = win[r][1], win[r][1] = win[r][2], win[r][2] = ld(r, ox + 2);
                } else {
#pragma unroll
                    for (int r = 0; r < 3; ++r)
#pragma unroll
                        for (int cc = 0; cc < 3; ++cc) win[r][cc] = ld(r, ox * s + cc);
                }
                float2 acc = K.z;
#pragma unroll
                for (int ky = 0; ky < 3; ++ky)
#pragma unroll
                    for (int kx = 0; kx < 3; ++kx) acc = add2(K, acc, mul2(K, win[ky][kx], w2[ky * 3 + kx]));
                if (yh) {  // tf32 planes for the pointwise GEMMs (3xTF32 operand split)
                    const float2 hv = make_float2(__uint_as_float(tc_split_hi(acc.x)), __uint_as_float(tc_split_hi(acc.y)));
                    const float2 d = sub2(K, acc, hv);
                    *reinterpret_cast<float2*>(yh + off) = hv;
                    *reinterpret_cast<float2*>(yl + off) =  // infinities: lo = 0 (tc_split_lo)
                        make_float2(isinf(acc.x) ? 0.0f : __uint_as_float(tc_split_hi(d.x)),
                                    isinf(acc.y) ? 0.0f : __uint_as_float(tc_split_hi(d.y)));
                    if (o.y_both) *reinterpret_cast<float2*>(yf + off) = acc;
                } else {
                    *reinterpret_cast<float2*>(yf + off) = acc;
                }
            }
        }
        oy += R.step;
        while (oy >= t.th) oy -= t.th, ++i;
    }
}

// ----------------------------------------------------------- backward tile
// gs: gy tile, xs: raw p tile (both with halo).  Pass A: input gradient
// (outputs ascending, tap (1-dy, 1-dx), ops.hpp:156-174), previous ReLU mask
// (from the raw centre), BN-backward partials; xs is then mapped to
// relu(bn(p)); pass B: weight-gradient terms.  The CTA partials (row q.tile)
// are reduced over the row workers in fixed order, through gs.
template <class Wait>
__device__ __forceinline__ void dw_bwd_tile(const DwBwdOp& o, const DwPos& q, float* gs, float* xs, Wait wait) {
    const DwTile& t = o.tile;
    const int n = o.n, h = o.h, w = o.wd, C = o.c;
    const int p = threadIdx.x & 15, c2 = q.c0 + 2 * p;
    const int rs = t.tw * kDwC;
    const bool pok = c2 < C;
    float2 acc2[11];  // gk[9], sg, sgx
#pragma unroll
    for (int k = 0; k < 11; ++k) acc2[k] = make_float2(0.0f, 0.0f);
    const PkConsts K = pk_consts();
    const DwRows R = dw_rows(t, w);
    float2 w2[9], mean2 = K.z, inv2 = K.z, gam2 = K.z, bet2 = K.z;
    bool fin = true;  // finite weights: adding the skipped zero terms is exact
    if (pok) {
#pragma unroll
        for (int k = 0; k < 9; ++k) {
            w2[k] = *reinterpret_cast<const float2*>(o.w + k * C + c2);
            fin = fin && isfinite(w2[k].x) && isfinite(w2[k].y);
        }
        mean2 = *reinterpret_cast<const float2*>(o.mean + c2);
        inv2 = *reinterpret_cast<const float2*>(o.inv + c2);
        gam2 = *reinterpret_cast<const float2*>(o.gamma + c2);
        bet2 = *reinterpret_cast<const float2*>(o.beta + c2);
    }
    BnRelu4 p4;
    p4.load(o.mean, o.inv, o.gamma, o.beta, q.c0, C);
    wait();
    if (pok) {
        float* const gyprev = o.gyprev;
        int i = 0, y = R.rw >> R.xsh;
        while (y >= t.th) y -= t.th, ++i;
        for (; i < t.ni;) {
            const int nn = q.n0 + i, yy = q.y0 + y;
            if (nn < n && yy < h) {
                long long gi = ((static_cast<long long>(nn) * h + yy) * w + R.xb) * C + c2;
                const float* g0 = gs + ((i * t.tr + y) * t.tw) * kDwC + 2 * p;
                const float* x0 = xs + ((i * t.tr + y) * t.tw) * kDwC + 2 * p;
                auto ldg2 = [&](int r, int col) { return *reinterpret_cast<const float2*>(g0 + r * rs + col * kDwC); };
                float2 gw[3][3];
#pragma unroll
                for (int r = 0; r < 3; ++r) gw[r][1] = ldg2(r, R.xb), gw[r][2] = ldg2(r, R.xb + 1);
                for (int x = R.xb; x < R.xe; ++x, gi += C) {
#pragma unroll
                    for (int r = 0; r < 3; ++r) gw[r][0] = gw[r][1], gw[r][1] = gw[r][2], gw[r][2] = ldg2(r, x + 2);
                    float2 gx = K.z;
                    if (fin) {
#pragma unroll
                        for (int r = 0; r < 3; ++r)
#pragma unroll
                            for (int cc = 0; cc < 3; ++cc) gx = add2(K, gx, mul2(K, gw[r][cc], w2[(2 - r) * 3 + (2 - cc)]));
                    } else {  // zero terms skipped per lane (0 * inf would be NaN)
#pragma unroll
                        for (int r = 0; r < 3; ++r)
#pragma unroll
                            for (int cc = 0; cc < 3; ++cc) {
                                const float2 gv = gw[r][cc], wv = w2[(2 - r) * 3 + (2 - cc)];
                                if (gv.x != 0.0f) gx.x = add(gx.x, mul(gv.x, wv.x));
                                if (gv.y != 0.0f) gx.y = add(gx.y, mul(gv.y, wv.y));
                            }
                    }
                    const float2 xpc = *reinterpret_cast<const float2*>(x0 + rs + (x + 1) * kDwC);  // raw centre
                    const float2 xh = mul2(K, sub2(K, xpc, mean2), inv2);
                    const float2 yv = add2(K, mul2(K, gam2, xh), bet2);
                    const float2 gz = add2(K, K.z, gx);
                    const float2 gm = make_float2(yv.x > 0.0f ? gz.x : 0.0f, yv.y > 0.0f ? gz.y : 0.0f);
                    *reinterpret_cast<float2*>(gyprev + gi) = gm;
                    acc2[9] = add2(K, acc2[9], gm);
                    acc2[10] = fma2(gm, xh, acc2[10]);
                }
            }
            y += R.step;
            while (y >= t.th) y -= t.th, ++i;
        }
    }
    __syncthreads();  // pass A read the raw tile
    dw_map4(xs, t, n, h, w, q.n0, q.y0 - 1, -1, [&](float v, int k) { return p4.train(v, k); });
    __syncthreads();
    if (pok) {
        int i = 0, y = R.rw >> R.xsh;
        while (y >= t.th) y -= t.th, ++i;
        for (; i < t.ni;) {
            const int nn = q.n0 + i, yy = q.y0 + y;
            if (nn < n && yy < h) {
                const float* g0 = gs + ((i * t.tr + y) * t.tw) * kDwC + 2 * p;
                const float* x0 = xs + ((i * t.tr + y) * t.tw) * kDwC + 2 * p;
                auto ldx2 = [&](int r, int col) { return *reinterpret_cast<const float2*>(x0 + r * rs + col * kDwC); };
                float2 xw[3][3];
#pragma unroll
                for (int r = 0; r < 3; ++r) xw[r][1] = ldx2(r, R.xb), xw[r][2] = ldx2(r, R.xb + 1);
                for (int x = R.xb; x < R.xe; ++x) {
#pragma unroll
                    for (int r = 0; r < 3; ++r) xw[r][0] = xw[r][1], xw[r][1] = xw[r][2], xw[r][2] = ldx2(r, x + 2);
                    const float2 gyc = *reinterpret_cast<const float2*>(g0 + rs + (x + 1) * kDwC);
                    if (gyc.x != 0.0f || gyc.y != 0.0f) {
#pragma unroll
                        for (int r = 0; r < 3; ++r)
#pragma unroll
                            for (int cc = 0; cc < 3; ++cc) acc2[r * 3 + cc] = fma2(gyc, xw[r][cc], acc2[r * 3 + cc]);
                    }
                }
            }
            y += R.step;
            while (y >= t.th) y -= t.th, ++i;
        }
    }
    __syncthreads();  // the gy tile is reused for the reduction
    float out[11];
    dw_lane_sum2<11>(gs, acc2, out);
    const int c = q.c0 + static_cast<int>(threadIdx.x);
    if (threadIdx.x < kDwC && c < C) {
        for (int k = 0; k < 9; ++k) o.part_gk[(static_cast<long long>(q.tile) * 9 + k) * C + c] = out[k];
        o.part_sg[static_cast<long long>(q.tile) * C + c] = out[9];
        o.part_sgx[static_cast<long long>(q.tile) * C + c] = out[10];
    }
}

// ------------------------------------------------------ weight-grad tile
// xs: input tile with halo, gs: output-gradient tile [ni][th][wo][32];
// red: >= 16 * 9 * 32 floats of shared memory free for the reduction.
template <class Wait>
__device__ __forceinline__ void dw_gk_tile(const DwGkOp& o, const DwPos& q, const float* xs, const float* gs,
                                           float* red, Wait wait) {
    const DwTile& t = o.tile;
    const int n = o.n, C = o.c, ho = o.ho, wo = o.wo, s = o.stride;
    const int p = threadIdx.x & 15, c2 = q.c0 + 2 * p;
    float2 acc2[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) acc2[k] = make_float2(0.0f, 0.0f);
    wait();
    if (c2 < C) {
        const DwRows R = dw_rows(t, wo);
        int i = 0, oy = R.rw >> R.xsh;
        while (oy >= t.th) oy -= t.th, ++i;
        for (; i < t.ni;) {
            const int nn = q.n0 + i, yy = q.y0 + oy;
            if (nn < n && yy < ho) {
                const float* gsr = gs + ((i * t.th + oy) * wo) * kDwC + 2 * p;
                const float* base = xs + ((i * t.tr + oy * s) * t.tw) * kDwC + 2 * p;
#pragma unroll 2
                for (int ox = R.xb; ox < R.xe; ++ox) {
                    const float2 gv = *reinterpret_cast<const float2*>(gsr + ox * kDwC);
                    if (gv.x == 0.0f && gv.y == 0.0f) continue;
                    const float* b = base + ox * s * kDwC;
#pragma unroll
                    for (int ky = 0; ky < 3; ++ky)
#pragma unroll
                        for (int kx = 0; kx < 3; ++kx)
                            acc2[ky * 3 + kx] =
                                fma2(gv, *reinterpret_cast<const float2*>(b + (ky * t.tw + kx) * kDwC), acc2[ky * 3 + kx]);
                }
            }
            oy += R.step;
            while (oy >= t.th) oy -= t.th, ++i;
        }
    }
    __syncthreads();
    float out[9];
    dw_lane_sum2<9>(red, acc2, out);
    const int c = q.c0 + static_cast<int>(threadIdx.x);
    if (threadIdx.x < kDwC && c < C)
        for (int k = 0; k < 9; ++k) o.part_gk[(static_cast<long long>(q.tile) * 9 + k) * C + c] = out[k];
}

}  // namespace pbkd_gpu
