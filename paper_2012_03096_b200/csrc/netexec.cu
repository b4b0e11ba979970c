// netexec.cu -- layer-by-layer block execution on the GPU (see netexec.hpp).
#include <algorithm>
#include <cmath>
#include <cstring>

#include "netexec.hpp"
#include "ops.cuh"

namespace pbkd_gpu {

using pbkd::LayerKind;

namespace {

constexpr float kEps = 1e-5f;         // static_cast<float>(kBnEps), ops.hpp:245
constexpr float kBnMomentum = 0.9f;   // model.cpp:15

int grid_for(long long total, int per = 256) {
    return static_cast<int>(std::max<long long>(1, std::min<long long>(148LL * 16, (total + per - 1) / per)));
}

#define GRID_STRIDE(i, total)                                                                       \
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < (total); \
         i += static_cast<long long>(gridDim.x) * blockDim.x)

// ------------------------------------------------------------- elementwise
__global__ void k_affine(const float* x, float* y, long long total, int c, const float* scale, const float* shift) {
    GRID_STRIDE(i, total) y[i] = bn_infer_apply(x[i], scale[i % c], shift[i % c]);
}
__global__ void k_relu(const float* x, float* y, long long total) {
    GRID_STRIDE(i, total) y[i] = relu(x[i]);
}
__global__ void k_relu_bwd(const float* x, const float* gy, float* gx, long long total) {  // ops.hpp:387-393
    GRID_STRIDE(i, total) gx[i] = x[i] > 0.0f ? gy[i] : 0.0f;
}
__global__ void k_add(const float* a, const float* b, float* y, long long total) {
    GRID_STRIDE(i, total) y[i] = add(a[i], b[i]);
}
__global__ void k_axpy(float* y, const float* x, long long total) {
    GRID_STRIDE(i, total) y[i] = add(y[i], x[i]);
}
// ops.hpp:361-374: gx += gy * gamma / sqrt(mv + eps)
__global__ void k_bn_infer_bwd(const float* gy, const float* gamma, const float* mv, float* gx, long long total,
                               int c) {
    GRID_STRIDE(i, total) {
        const int ch = static_cast<int>(i % c);
        const float sc = __fdiv_rn(gamma[ch], __fsqrt_rn(add(mv[ch], kEps)));
        gx[i] = add(gx[i], mul(sc, gy[i]));
    }
}
// ops.hpp:531-539: g += (scale*2/count) * (s - t)
__global__ void k_mse_bwd(const float* s, const float* t, float* g, long long total, float k) {
    GRID_STRIDE(i, total) g[i] = add(g[i], mul(k, sub(s[i], t[i])));
}
// ops.hpp:545-558 per trainable tensor: v = m*v + g; w -= lr*v
__global__ void k_sgd(float* w, const float* g, float* v, long long n, float lr, float mom) {
    GRID_STRIDE(i, n) {
        const float vv = add(mul(mom, v[i]), g[i]);
        v[i] = vv;
        w[i] = sub(w[i], mul(lr, vv));
    }
}
__global__ void k_sum_parts(const float* part, int parts, long long width, float* out, int accumulate) {
    GRID_STRIDE(i, width) {
        float s = 0.0f;
        for (int p = 0; p < parts; ++p) s = add(s, part[static_cast<long long>(p) * width + i]);
        out[i] = accumulate ? add(out[i], s) : s;
    }
}

// ------------------------------------------------------------- depthwise
// ops.hpp:114-147: per output a serial (ky, kx) sum, out-of-bounds taps skipped
__global__ void k_dw_fwd(const float* x, const float* k9c, float* y, int n, int h, int w, int c, int ho, int wo,
                         int s, int p) {
    const long long total = static_cast<long long>(n) * ho * wo * c;
    GRID_STRIDE(i, total) {
        const int ch = static_cast<int>(i % c);
        long long r = i / c;
        const int ox = static_cast<int>(r % wo);
        r /= wo;
        const int oy = static_cast<int>(r % ho);
        const int b = static_cast<int>(r / ho);
        float acc = 0.0f;
        for (int ky = 0; ky < 3; ++ky) {
            const int iy = oy * s - p + ky;
            if (iy < 0 || iy >= h) continue;
            for (int kx = 0; kx < 3; ++kx) {
                const int ix = ox * s - p + kx;
                if (ix < 0 || ix >= w) continue;
                acc = add(acc, mul(x[((static_cast<long long>(b) * h + iy) * w + ix) * c + ch], k9c[(ky * 3 + kx) * c + ch]));
            }
        }
        y[i] = acc;
    }
}
// ops.hpp:149-178 input gradient: each input pixel gathers g*k from its
// outputs in ascending (oy, ox) order (= descending ky, kx)
__global__ void k_dw_dgrad(const float* gy, const float* k9c, float* gx, int n, int h, int w, int c, int ho, int wo,
                           int s, int p) {
    const long long total = static_cast<long long>(n) * h * w * c;
    GRID_STRIDE(i, total) {
        const int ch = static_cast<int>(i % c);
        long long r = i / c;
        const int ix = static_cast<int>(r % w);
        r /= w;
        const int iy = static_cast<int>(r % h);
        const int b = static_cast<int>(r / h);
        float acc = 0.0f;
        for (int ky = 2; ky >= 0; --ky) {
            const int ty = iy + p - ky;
            if (ty < 0 || ty % s) continue;
            const int oy = ty / s;
            if (oy >= ho) continue;
            for (int kx = 2; kx >= 0; --kx) {
                const int tx = ix + p - kx;
                if (tx < 0 || tx % s) continue;
                const int ox = tx / s;
                if (ox >= wo) continue;
                acc = add(acc, mul(gy[((static_cast<long long>(b) * ho + oy) * wo + ox) * c + ch], k9c[(ky * 3 + kx) * c + ch]));
            }
        }
        gx[i] = acc;
    }
}
// depthwise weight-gradient partials: part[pp][tap][c] over a fixed row slice
__global__ void k_dw_wgrad_part(const float* gy, const float* x, float* part, int n, int h, int w, int c, int ho,
                                int wo, int s, int p, int parts) {
    const long long outs = static_cast<long long>(n) * ho * wo;
    const long long per = (outs + parts - 1) / parts;
    const int pp = blockIdx.y;
    const long long r0 = pp * per, r1 = min(outs, r0 + per);
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < 9 * c; e += gridDim.x * blockDim.x) {
        const int tap = e / c, ch = e % c, ky = tap / 3, kx = tap % 3;
        float acc = 0.0f;
        for (long long r = r0; r < r1; ++r) {
            const int ox = static_cast<int>(r % wo);
            const int oy = static_cast<int>((r / wo) % ho);
            const int b = static_cast<int>(r / (static_cast<long long>(wo) * ho));
            const int iy = oy * s - p + ky, ix = ox * s - p + kx;
            if (iy < 0 || iy >= h || ix < 0 || ix >= w) continue;
            acc = add(acc, mul(gy[r * c + ch], x[((static_cast<long long>(b) * h + iy) * w + ix) * c + ch]));
        }
        part[static_cast<long long>(pp) * 9 * c + e] = acc;
    }
}
// [tap][c] sums -> reference layout [c][1][3][3], accumulated
__global__ void k_dw_wgrad_fin(const float* part, int parts, int c, float* gk) {
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < 9 * c; e += gridDim.x * blockDim.x) {
        float s = 0.0f;
        for (int q = 0; q < parts; ++q) s = add(s, part[static_cast<long long>(q) * 9 * c + e]);
        const int tap = e / c, ch = e % c;
        gk[ch * 9 + tap] = add(gk[ch * 9 + tap], s);
    }
}
// reference [c][1][3][3] -> [9][c]
__global__ void k_dw_relayout(const float* w, float* k9c, int c) {
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < 9 * c; e += gridDim.x * blockDim.x)
        k9c[e] = w[(e % c) * 9 + e / c];
}

// ------------------------------------------------------------- conv helpers
// cols[(b,oy,ox)][(ky*k+kx)*c + j] (zero where the window leaves the image)
__global__ void k_im2col(const float* x, float* cols, int n, int h, int w, int c, int k, int s, int p, int ho,
                         int wo) {
    const long long kc = static_cast<long long>(k) * k * c;
    const long long total = static_cast<long long>(n) * ho * wo * kc;
    GRID_STRIDE(i, total) {
        const long long r = i / kc;
        const int col = static_cast<int>(i % kc);
        const int j = col % c, tap = col / c, ky = tap / k, kx = tap % k;
        const int ox = static_cast<int>(r % wo), oy = static_cast<int>((r / wo) % ho);
        const int b = static_cast<int>(r / (static_cast<long long>(wo) * ho));
        const int iy = oy * s - p + ky, ix = ox * s - p + kx;
        cols[i] = (iy < 0 || iy >= h || ix < 0 || ix >= w) ? 0.0f
                                                           : x[((static_cast<long long>(b) * h + iy) * w + ix) * c + j];
    }
}
// gx[b,iy,ix,j] (+)= sum over taps (ky, kx ascending) of dcols at the output
// position that window tap reads (iy = oy*s - p + ky)
__global__ void k_col2im(const float* dcols, float* gx, int n, int h, int w, int c, int k, int s, int p, int ho,
                         int wo, int accumulate) {
    const long long kc = static_cast<long long>(k) * k * c;
    const long long total = static_cast<long long>(n) * h * w * c;
    GRID_STRIDE(i, total) {
        const int j = static_cast<int>(i % c);
        long long r = i / c;
        const int ix = static_cast<int>(r % w);
        r /= w;
        const int iy = static_cast<int>(r % h);
        const int b = static_cast<int>(r / h);
        float acc = 0.0f;
        for (int ky = 0; ky < k; ++ky) {
            const int ty = iy + p - ky;
            if (ty < 0 || ty % s) continue;
            const int oy = ty / s;
            if (oy >= ho) continue;
            for (int kx = 0; kx < k; ++kx) {
                const int tx = ix + p - kx;
                if (tx < 0 || tx % s) continue;
                const int ox = tx / s;
                if (ox >= wo) continue;
                acc = add(acc, dcols[((static_cast<long long>(b) * ho + oy) * wo + ox) * kc + (ky * k + kx) * c + j]);
            }
        }
        gx[i] = accumulate ? add(gx[i], acc) : acc;
    }
}
// gkt[o][tap*cin + j] -> grad[o][j][tap] (reference layout), accumulated
__global__ void k_conv_wgrad_relayout(const float* gkt, float* grad, int cout, int cin, int kk) {
    const long long total = static_cast<long long>(cout) * cin * kk;
    GRID_STRIDE(i, total) {
        const int tap = static_cast<int>(i % kk);
        const int j = static_cast<int>((i / kk) % cin);
        const int o = static_cast<int>(i / (static_cast<long long>(kk) * cin));
        grad[i] = add(grad[i], gkt[static_cast<long long>(o) * kk * cin + static_cast<long long>(tap) * cin + j]);
    }
}

// ------------------------------------------------------------- batch norm
// Fixed-order column partials: part[q][c] over row slice q of `rows`
// (one thread per channel per slice, serial rows -> schedule independent).
template <int KIND>
__global__ void k_col_part(const float* a, const float* b, int rows_i, int c, int parts, float* p0, float* p1) {
    const long long rows = rows_i;
    const long long per = (rows + parts - 1) / parts;
    const int q = blockIdx.y;
    const long long r0 = q * per, r1 = min(rows, r0 + per);
    for (int ch = blockIdx.x * blockDim.x + threadIdx.x; ch < c; ch += gridDim.x * blockDim.x) {
        float s0 = 0.0f, s1 = 0.0f;
        for (long long r = r0; r < r1; ++r) {
            const float v = a[r * c + ch];
            if (KIND == 0) {  // sum, sum of squares (ops.hpp:273-283)
                s0 = add(s0, v);
                s1 = add(s1, mul(v, v));
            } else {  // sum g, sum g*xhat (ops.hpp:333-342)
                s0 = add(s0, v);
                s1 = add(s1, mul(v, b[r * c + ch]));
            }
        }
        p0[static_cast<long long>(q) * c + ch] = s0;
        p1[static_cast<long long>(q) * c + ch] = s1;
    }
}
// ops.hpp:284-299: mean, var = E[x^2]-mean^2 clamped, inv_std, moving update
__global__ void k_bn_stats(const float* p0, const float* p1, int parts, int c, long long m, float* mean, float* inv,
                           float* mm, float* mv) {
    for (int ch = blockIdx.x * blockDim.x + threadIdx.x; ch < c; ch += gridDim.x * blockDim.x) {
        float s = 0.0f, q = 0.0f;
        for (int i = 0; i < parts; ++i) {
            s = add(s, p0[static_cast<long long>(i) * c + ch]);
            q = add(q, p1[static_cast<long long>(i) * c + ch]);
        }
        const float fm = static_cast<float>(m);
        const float mu = __fdiv_rn(s, fm);
        float var = sub(__fdiv_rn(q, fm), mul(mu, mu));
        if (var < 0.0f) var = 0.0f;
        mean[ch] = mu;
        inv[ch] = __fdiv_rn(1.0f, __fsqrt_rn(add(var, kEps)));
        const float one_m = sub(1.0f, kBnMomentum);
        mm[ch] = add(mul(kBnMomentum, mm[ch]), mul(one_m, mu));
        mv[ch] = add(mul(kBnMomentum, mv[ch]), mul(one_m, var));
    }
}
__global__ void k_bn_apply(const float* x, float* y, float* xhat, long long total, int c, const float* mean,
                           const float* inv, const float* gamma, const float* beta) {
    GRID_STRIDE(i, total) {
        const int ch = static_cast<int>(i % c);
        const float nv = mul(sub(x[i], mean[ch]), inv[ch]);
        if (xhat) xhat[i] = nv;
        y[i] = add(mul(gamma[ch], nv), beta[ch]);
    }
}
// sums -> sg / sgx; parameter gradients accumulate (ops.hpp:343-344)
__global__ void k_bn_bwd_sums(const float* p0, const float* p1, int parts, int c, float* sg, float* sgx,
                              float* ggamma, float* gbeta) {
    for (int ch = blockIdx.x * blockDim.x + threadIdx.x; ch < c; ch += gridDim.x * blockDim.x) {
        float a = 0.0f, b = 0.0f;
        for (int i = 0; i < parts; ++i) {
            a = add(a, p0[static_cast<long long>(i) * c + ch]);
            b = add(b, p1[static_cast<long long>(i) * c + ch]);
        }
        sg[ch] = a;
        sgx[ch] = b;
        if (ggamma) ggamma[ch] = add(ggamma[ch], b);
        if (gbeta) gbeta[ch] = add(gbeta[ch], a);
    }
}
// ops.hpp:345-354: gx += (gamma*inv) * ((g - inv_m*sg) - (xhat*inv_m)*sgx)
__global__ void k_bn_bwd_apply(const float* g, const float* xhat, float* gx, long long total, int c,
                               const float* gamma, const float* inv, const float* sg, const float* sgx, float inv_m) {
    GRID_STRIDE(i, total) {
        const int ch = static_cast<int>(i % c);
        const float kk = mul(gamma[ch], inv[ch]);
        const float v = sub(sub(g[i], mul(inv_m, sg[ch])), mul(mul(xhat[i], inv_m), sgx[ch]));
        gx[i] = add(gx[i], mul(kk, v));
    }
}

// ------------------------------------------------------------- head / losses
// ops.hpp:395-407 (serial sum over the plane, then / plane)
__global__ void k_gap(const float* x, float* y, int n, int hw, int c) {
    GRID_STRIDE(i, static_cast<long long>(n) * c) {
        const long long b = i / c;
        const int ch = static_cast<int>(i % c);
        float s = 0.0f;
        for (int q = 0; q < hw; ++q) s = add(s, x[(b * hw + q) * c + ch]);
        y[i] = __fdiv_rn(s, static_cast<float>(hw));
    }
}
// ops.hpp:410-423: gx += gy / plane
__global__ void k_gap_bwd(const float* gy, float* gx, int n, int hw, int c) {
    const float inv = __fdiv_rn(1.0f, static_cast<float>(hw));
    GRID_STRIDE(i, static_cast<long long>(n) * hw * c) {
        const int ch = static_cast<int>(i % c);
        const long long b = i / (static_cast<long long>(hw) * c);
        gx[i] = add(gx[i], mul(gy[b * c + ch], inv));
    }
}
// ops.hpp:425-442: acc = bias[o]; acc += w[o][j]*x[j] for ascending j
__global__ void k_dense(const float* x, const float* w, const float* bias, float* y, int n, int cin, int cout) {
    GRID_STRIDE(i, static_cast<long long>(n) * cout) {
        const long long b = i / cout;
        const int o = static_cast<int>(i % cout);
        float acc = bias ? bias[o] : 0.0f;
        for (int j = 0; j < cin; ++j) acc = add(acc, mul(w[static_cast<long long>(o) * cin + j], x[b * cin + j]));
        y[i] = acc;
    }
}
// ops.hpp:444-458
__global__ void k_dense_dgrad(const float* gy, const float* w, float* gx, int n, int cin, int cout) {
    GRID_STRIDE(i, static_cast<long long>(n) * cin) {
        const long long b = i / cin;
        const int j = static_cast<int>(i % cin);
        float acc = gx[i];
        for (int o = 0; o < cout; ++o) acc = add(acc, mul(gy[b * cout + o], w[static_cast<long long>(o) * cin + j]));
        gx[i] = acc;
    }
}
__global__ void k_dense_wgrad(const float* gy, const float* x, float* gw, float* gb, int n, int cin, int cout) {
    GRID_STRIDE(i, static_cast<long long>(cout) * cin) {
        const int o = static_cast<int>(i / cin), j = static_cast<int>(i % cin);
        float acc = gw[i];
        for (int b = 0; b < n; ++b) acc = add(acc, mul(gy[static_cast<long long>(b) * cout + o], x[static_cast<long long>(b) * cin + j]));
        gw[i] = acc;
        if (gb && j == 0) {
            float s = gb[o];
            for (int b = 0; b < n; ++b) s = add(s, gy[static_cast<long long>(b) * cout + o]);
            gb[o] = s;
        }
    }
}
// ops.hpp:474-501 per sample: stable log-sum-exp, loss_n = lse - logit[label]
__global__ void k_softmax_ce(const float* logits, const int* labels, float* probs, float* loss, int n, int k) {
    GRID_STRIDE(b, n) {
        const float* row = logits + b * k;
        float mx = row[0];
        for (int j = 1; j < k; ++j) mx = fmaxf(mx, row[j]);
        float s = 0.0f;
        for (int j = 0; j < k; ++j) s = add(s, expf(sub(row[j], mx)));
        const float lse = add(mx, logf(s));
        loss[b] = sub(lse, row[labels[b]]);
        if (probs)
            for (int j = 0; j < k; ++j) probs[b * k + j] = expf(sub(row[j], lse));
    }
}
// ops.hpp:503-514: g += (p - [j == label]) * scale / n
__global__ void k_softmax_ce_bwd(const float* probs, const int* labels, float* g, int n, int k, float inv_n) {
    GRID_STRIDE(i, static_cast<long long>(n) * k) {
        const long long b = i / k;
        const int j = static_cast<int>(i % k);
        float v = probs[i];
        if (j == labels[b]) v = sub(v, 1.0f);
        g[i] = add(g[i], mul(v, inv_n));
    }
}
// distill.cpp:38-55: first maximum wins
__global__ void k_argmax_correct(const float* logits, const int* labels, int n, int k, int* correct) {
    GRID_STRIDE(b, n) {
        const float* row = logits + b * k;
        int best = 0;
        float bv = row[0];
        for (int j = 1; j < k; ++j)
            if (row[j] > bv) bv = row[j], best = j;
        if (best == labels[b]) atomicAdd(correct, 1);  // integer count: order-free
    }
}

__global__ void k_take_samples(const float* src, const int* pos, float* out, int n, long long row) {
    GRID_STRIDE(i, static_cast<long long>(n) * row) {
        const long long s = i / row;
        out[i] = src[static_cast<long long>(pos[s]) * row + i % row];
    }
}

// loss_kernel's partition and order (ops.cu): CTA `local` owns rows
// [local*per, +per); thread (rr, gg) of the geo_of(c) layout accumulates
// rows rr, rr+RP, ... over its V channels; thread 0 sums the 256 lanes
__global__ void k_loss_parts(const float* s, const float* t, int rows, int c, int per, float* part) {
    __shared__ float lred[256];
    const int V = (c % 4 == 0) ? 4 : 1;
    const long long r0 = static_cast<long long>(blockIdx.x) * per;
    const long long r1 = min(static_cast<long long>(rows), r0 + per);
    float lsum = 0.0f;
    for (int cb = 0; cb < c; cb += 256 * V) {  // loss_kernel's channel passes
        const int cw = min(256 * V, c - cb);
        const int G = cw / V, RP = max(1, 256 / G);
        const int rr = threadIdx.x / G, gg = threadIdx.x % G;
        if (rr < RP) {
            const int c0 = cb + gg * V;
            for (long long r = r0 + rr; r < r1; r += RP)
                for (int q = 0; q < V; ++q) {
                    const float d = sub(s[r * c + c0 + q], t[r * c + c0 + q]);
                    lsum += d * d;
                }
        }
    }
    lred[threadIdx.x] = lsum;
    __syncthreads();
    if (threadIdx.x == 0) {
        float a = 0.0f;
        for (int i = 0; i < 256; ++i) a += lred[i];
        part[blockIdx.x] = a;
    }
}
// bn_bwd_fin_kernel's loss tree: one warp, double partials, xor shuffle
__global__ void k_loss_final(const float* part, int ctas, double count, float* out) {
    double a = 0.0;
    for (int p = threadIdx.x; p < ctas; p += 32) a += static_cast<double>(part[p]);
    for (int off = 16; off > 0; off >>= 1) a += __shfl_xor_sync(0xffffffffu, a, off);
    if (threadIdx.x == 0) *out = static_cast<float>(a / count);
}

int parts_for(long long rows) { return static_cast<int>(std::max<long long>(1, std::min<long long>(128, rows / 64))); }

}  // namespace

// ======================================================================== NetExec
NetExec::NetExec(cudaStream_t st) : st_(st) {}

DTensor NetExec::alloc(int n, int c, int h, int w, bool zero) {
    DTensor t;
    t.n = n, t.c = c, t.h = h, t.w = w;
    const size_t bytes = std::max<size_t>(16, static_cast<size_t>(t.size()) * sizeof(float));
    float* p = nullptr;
    PBKD_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&p), bytes, st_));
    cudaStream_t st = st_;
    t.mem = std::shared_ptr<float>(p, [st](float* q) { cudaFreeAsync(q, st); });
    t.p = p;
    if (zero) PBKD_CUDA(cudaMemsetAsync(p, 0, bytes, st_));
    return t;
}

DTensor NetExec::upload_nchw(const float* x, int n, int c, int h, int w) {
    std::vector<float> v(static_cast<size_t>(n) * c * h * w);
    for (int b = 0; b < n; ++b)
        for (int ch = 0; ch < c; ++ch)
            for (int y = 0; y < h; ++y)
                for (int xx = 0; xx < w; ++xx)
                    v[((static_cast<size_t>(b) * h + y) * w + xx) * c + ch] =
                        x[((static_cast<size_t>(b) * c + ch) * h + y) * w + xx];
    DTensor t = alloc(n, c, h, w);
    PBKD_CUDA(cudaMemcpyAsync(t.p, v.data(), v.size() * sizeof(float), cudaMemcpyHostToDevice, st_));
    PBKD_CUDA(cudaStreamSynchronize(st_));  // v is a stack buffer
    return t;
}

void NetExec::download_nchw(const DTensor& t, float* out) {
    std::vector<float> v(static_cast<size_t>(t.size()));
    PBKD_CUDA(cudaMemcpyAsync(v.data(), t.p, v.size() * sizeof(float), cudaMemcpyDeviceToHost, st_));
    PBKD_CUDA(cudaStreamSynchronize(st_));
    for (int b = 0; b < t.n; ++b)
        for (int ch = 0; ch < t.c; ++ch)
            for (int y = 0; y < t.h; ++y)
                for (int x = 0; x < t.w; ++x)
                    out[((static_cast<size_t>(b) * t.c + ch) * t.h + y) * t.w + x] =
                        v[((static_cast<size_t>(b) * t.h + y) * t.w + x) * t.c + ch];
}

DTensor NetExec::gather(const float* images_nchw, const int* idx_dev, int n, int c, int h, int w) {
    DTensor t = alloc(n, c, h, w);
    launch_gather_nhwc(images_nchw, idx_dev, n, c, h, w, t.p, st_);
    return t;
}

DTensor NetExec::upload_ints(const std::vector<int>& v) {
    DTensor t = alloc(1, 1, 1, static_cast<int>(std::max<size_t>(v.size(), 1)));
    if (!v.empty())
        PBKD_CUDA(cudaMemcpyAsync(t.p, v.data(), v.size() * sizeof(int), cudaMemcpyHostToDevice, st_));
    PBKD_CUDA(cudaStreamSynchronize(st_));
    return t;
}

DTensor NetExec::take_samples(const DTensor& src, const int* pos, int n) {
    DTensor t = alloc(n, src.c, src.h, src.w);
    const long long row = static_cast<long long>(src.c) * src.h * src.w;
    k_take_samples<<<grid_for(n * row), 256, 0, st_>>>(src.p, pos, t.p, n, row);
    PBKD_LAUNCH_CHECK();
    return t;
}

DTensor NetExec::slice_samples(const DTensor& src, int first, int n) {
    DTensor t = alloc(n, src.c, src.h, src.w);
    const long long row = static_cast<long long>(src.c) * src.h * src.w;
    PBKD_CUDA(cudaMemcpyAsync(t.p, src.p + first * row, n * row * sizeof(float), cudaMemcpyDeviceToDevice, st_));
    return t;
}

void NetExec::put_samples(DTensor& dst, int first, const DTensor& src) {
    const long long row = static_cast<long long>(dst.c) * dst.h * dst.w;
    PBKD_CUDA(cudaMemcpyAsync(dst.p + first * row, src.p, src.size() * sizeof(float), cudaMemcpyDeviceToDevice, st_));
}

DevBlock NetExec::make_block(const pbkd::Block& b, const float* src, bool src_on_device) {
    DevBlock d;
    long long off = 0;
    std::vector<float> host;
    for (const pbkd::LayerParams& lp : b.layers) {
        DevBlock::Layer l;
        l.kind = lp.kind;
        l.cin = lp.in_channels;
        l.cout = lp.out_channels;
        l.k = lp.kernel;
        l.stride = lp.stride;
        l.pad = lp.padding;
        auto take = [&](const pbkd::Tensor& t) {
            const long long at = off;
            host.insert(host.end(), t.data.begin(), t.data.end());
            off += static_cast<long long>(t.data.size());
            return at;
        };
        switch (lp.kind) {  // for_each_block_array order
            case LayerKind::Conv3x3:
            case LayerKind::Conv1x1:
            case LayerKind::Conv7x7:
            case LayerKind::DepthwiseConv3x3:
            case LayerKind::PointwiseConv:
                l.wn = static_cast<long long>(lp.weight.data.size());
                l.w = take(lp.weight);
                break;
            case LayerKind::Dense:
                l.wn = static_cast<long long>(lp.weight.data.size());
                l.w = take(lp.weight);
                if (!lp.bias.data.empty()) l.b = take(lp.bias);
                break;
            case LayerKind::BatchNorm:
                l.gamma = take(lp.gamma);
                l.beta = take(lp.beta);
                l.mm = take(lp.moving_mean);
                l.mv = take(lp.moving_var);
                break;
            case LayerKind::Add:
                if (!lp.weight.data.empty()) {
                    l.wn = static_cast<long long>(lp.weight.data.size());
                    l.w = take(lp.weight);
                    l.k = 1;
                    l.pad = 0;
                }
                break;
            default:
                break;
        }
        d.layers.push_back(std::move(l));
    }
    d.n = off;
    d.arrays = alloc(1, 1, 1, static_cast<int>(std::max<long long>(off, 1)));
    d.grads = alloc(1, 1, 1, static_cast<int>(std::max<long long>(off, 1)), true);
    d.vel = alloc(1, 1, 1, static_cast<int>(std::max<long long>(off, 1)), true);
    if (off) {
        const float* from = src ? src : host.data();
        PBKD_CUDA(cudaMemcpyAsync(d.arrays.p, from, static_cast<size_t>(off) * sizeof(float),
                                  src && src_on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st_));
        PBKD_CUDA(cudaStreamSynchronize(st_));
    }
    return d;
}

void NetExec::load_arrays(DevBlock& d, const float* host) {
    if (d.n) PBKD_CUDA(cudaMemcpyAsync(d.arrays.p, host, d.n * sizeof(float), cudaMemcpyHostToDevice, st_));
    PBKD_CUDA(cudaStreamSynchronize(st_));
    d.derived_ok = false;
}
void NetExec::arrays_to_host(const DevBlock& d, float* host) {
    if (d.n) PBKD_CUDA(cudaMemcpyAsync(host, d.arrays.p, d.n * sizeof(float), cudaMemcpyDeviceToHost, st_));
    PBKD_CUDA(cudaStreamSynchronize(st_));
}
void NetExec::grads_to_host(const DevBlock& d, float* host) {
    if (d.n) PBKD_CUDA(cudaMemcpyAsync(host, d.grads.p, d.n * sizeof(float), cudaMemcpyDeviceToHost, st_));
    PBKD_CUDA(cudaStreamSynchronize(st_));
}

// conv weights [cout][cin][kk] -> [cout][kk][cin] + tf32 planes; dw -> [9][c]
void NetExec::prepare(DevBlock& b) {
    if (b.derived_ok) return;
    for (DevBlock::Layer& l : b.layers) {
        const bool conv = l.kind == LayerKind::Conv3x3 || l.kind == LayerKind::Conv1x1 ||
                          l.kind == LayerKind::Conv7x7 || (l.kind == LayerKind::Add && l.w >= 0);
        if (conv) {
            const int kk = l.k * l.k;
            if (!l.wk) {
                l.wk = alloc(1, 1, 1, static_cast<int>(l.wn));
                l.whi = alloc(1, 1, 1, static_cast<int>(l.wn));
                l.wlo = alloc(1, 1, 1, static_cast<int>(l.wn));
            }
            launch_conv_weight_prep(b.at(l.w), l.cout, l.cin, kk, kk * l.cin, l.wk.p, l.whi.p, l.wlo.p, st_);
        } else if (l.kind == LayerKind::PointwiseConv) {
            if (!l.wk) l.wk = alloc(1, 1, 1, static_cast<int>(l.wn));
            if (l.stride != 1) {  // strided 1x1: the implicit-im2col conv ([cout][1][cin] = [cout][cin])
                if (!l.whi) l.whi = alloc(1, 1, 1, static_cast<int>(l.wn)), l.wlo = alloc(1, 1, 1, static_cast<int>(l.wn));
                launch_conv_weight_prep(b.at(l.w), l.cout, l.cin, 1, l.cin, l.wk.p, l.whi.p, l.wlo.p, st_);
            } else {
                PBKD_CUDA(cudaMemcpyAsync(l.wk.p, b.at(l.w), l.wn * sizeof(float), cudaMemcpyDeviceToDevice, st_));
            }
        } else if (l.kind == LayerKind::DepthwiseConv3x3) {
            if (!l.wk) l.wk = alloc(1, 1, 9, l.cin);
            k_dw_relayout<<<grid_for(9LL * l.cin), 256, 0, st_>>>(b.at(l.w), l.wk.p, l.cin);
            PBKD_LAUNCH_CHECK();
        }
    }
    b.derived_ok = true;
}

void NetExec::gemm(int M, int N, int K, const float* A, long long lda, bool akm, const float* B, long long ldb,
                   bool bkm, float* C, long long ldc, bool accumulate) {
    GemmOp o{};
    o.M = M, o.N = N, o.K = K;
    o.A = A, o.lda = lda, o.a_kmajor = akm ? 1 : 0;
    o.B = B, o.ldb = ldb, o.b_kmajor = bkm ? 1 : 0;
    o.ldc = ldc;
    // long reductions (weight gradients over rows) run split-K into partials
    o.ksplit = K > 4096 ? std::max(1, std::min(64, ceil_div(K, 2048))) : 1;
    o.epi = o.ksplit > 1 ? 2 : 0;
    DTensor part;
    DTensor tmp;
    if (o.epi == 2) {
        part = alloc(1, 1, o.ksplit, static_cast<int>(static_cast<long long>(M) * ldc));
        o.C = part.p;
    } else if (accumulate) {
        tmp = alloc(1, 1, M, static_cast<int>(ldc));
        o.C = tmp.p;
    } else {
        o.C = C;
    }
    gemm_finalize(o);
    if (o.epi == 2 && o.ksplit > part.h) throw std::logic_error("netexec: split-K partial buffer too small");
    DTensor desc = alloc(1, 1, 1, static_cast<int>((sizeof(GemmOp) + 3) / 4));
    PBKD_CUDA(cudaMemcpyAsync(desc.p, &o, sizeof(GemmOp), cudaMemcpyHostToDevice, st_));
    // (a pageable H2D copy has staged its source when it returns: o may die)
    launch_gemm_bn(reinterpret_cast<const GemmOp*>(desc.p), 1, ctas_gemm(o), gemm_bn_class(o), st_);
    const long long width = static_cast<long long>(M) * ldc;
    if (o.epi == 2) {
        k_sum_parts<<<grid_for(width), 256, 0, st_>>>(part.p, o.ksplit, width, C, accumulate ? 1 : 0);
        PBKD_LAUNCH_CHECK();
    } else if (accumulate) {
        k_axpy<<<grid_for(width), 256, 0, st_>>>(C, tmp.p, width);
        PBKD_LAUNCH_CHECK();
    }
}

std::pair<DTensor, DTensor> NetExec::pw_bn_stats(const DTensor& x, const float* w, int cin, int cout, float* y,
                                                  float* mm, float* mv) {
    GemmOp o{};
    o.M = static_cast<int>(x.rows()), o.N = cout, o.K = cin;
    o.A = x.p, o.lda = cin, o.a_kmajor = 1;
    o.B = w, o.ldb = cin, o.b_kmajor = 1;
    o.C = y, o.ldc = cout;
    o.ksplit = 1;
    o.epi = 1;
    const int tiles = ceil_div(o.M, 128);
    DTensor p0 = alloc(1, 1, tiles, cout), p1 = alloc(1, 1, tiles, cout);
    o.part0 = p0.p, o.part1 = p1.p;
    gemm_finalize(o);
    if (o.tiles_m != tiles) throw std::logic_error("netexec: unexpected GEMM M tiling");
    DTensor desc = alloc(1, 1, 1, static_cast<int>((sizeof(GemmOp) + 3) / 4));
    PBKD_CUDA(cudaMemcpyAsync(desc.p, &o, sizeof(GemmOp), cudaMemcpyHostToDevice, st_));
    launch_gemm_bn(reinterpret_cast<const GemmOp*>(desc.p), 1, ctas_gemm(o), gemm_bn_class(o), st_);
    DTensor mean = alloc(1, 1, 1, cout), inv = alloc(1, 1, 1, cout);
    BnStatOp b{};
    b.part_sum = p0.p, b.part_sq = p1.p, b.tiles = tiles, b.c = cout, b.m = o.M;
    b.mean = mean.p, b.inv = inv.p, b.mm = mm, b.mv = mv, b.update_moving = 1;
    DTensor bdesc = alloc(1, 1, 1, static_cast<int>((sizeof(BnStatOp) + 3) / 4));
    PBKD_CUDA(cudaMemcpyAsync(bdesc.p, &b, sizeof(BnStatOp), cudaMemcpyHostToDevice, st_));
    launch_bn_stat(reinterpret_cast<const BnStatOp*>(bdesc.p), 1, ctas_cols(cout), st_);
    return {mean, inv};
}

DTensor NetExec::conv_fwd(DevBlock::Layer& l, const DTensor& x) {
    const int ho = (x.h + 2 * l.pad - l.k) / l.stride + 1, wo = (x.w + 2 * l.pad - l.k) / l.stride + 1;
    DTensor y = alloc(x.n, l.cout, ho, wo);
    GemmOp o{};
    o.conv = 1;
    o.ih = x.h, o.iw = x.w, o.ic = l.cin, o.ksz = l.k, o.cstride = l.stride, o.cpad = l.pad;
    o.oh = ho, o.ow = wo;
    o.M = x.n * ho * wo, o.N = l.cout, o.K = l.k * l.k * l.cin;
    o.A = x.p;
    o.B = l.wk.p, o.b_hi = l.whi.p, o.b_lo = l.wlo.p, o.ldb = o.K, o.b_kmajor = 1;
    o.C = y.p, o.ldc = l.cout;
    o.ksplit = 1;
    gemm_finalize(o);
    DTensor desc = alloc(1, 1, 1, static_cast<int>((sizeof(GemmOp) + 3) / 4));
    PBKD_CUDA(cudaMemcpyAsync(desc.p, &o, sizeof(GemmOp), cudaMemcpyHostToDevice, st_));
    launch_gemm_bn(reinterpret_cast<const GemmOp*>(desc.p), 1, ctas_gemm(o), gemm_bn_class(o), st_);
    return y;
}

// ops.hpp:77-108 through explicit im2col: wgrad = gy^T . cols, dgrad =
// col2im(gy . W)
void NetExec::conv_bwd(DevBlock& b, DevBlock::Layer& l, const DTensor& x, const DTensor& gy, DTensor* gx,
                       bool wgrad) {
    const int kk = l.k * l.k;
    const int K9 = kk * l.cin;
    const long long M = gy.rows();
    if (wgrad) {
        DTensor cols = alloc(1, 1, static_cast<int>(M), K9);
        k_im2col<<<grid_for(M * K9), 256, 0, st_>>>(x.p, cols.p, x.n, x.h, x.w, x.c, l.k, l.stride, l.pad, gy.h,
                                                     gy.w);
        PBKD_LAUNCH_CHECK();
        DTensor gkt = alloc(1, 1, l.cout, K9);
        gemm(l.cout, K9, static_cast<int>(M), gy.p, l.cout, false, cols.p, K9, false, gkt.p, K9, false);
        k_conv_wgrad_relayout<<<grid_for(static_cast<long long>(l.cout) * K9), 256, 0, st_>>>(
            gkt.p, b.grad_at(l.w), l.cout, l.cin, kk);
        PBKD_LAUNCH_CHECK();
    }
    if (gx) {
        DTensor dcols = alloc(1, 1, static_cast<int>(M), K9);
        gemm(static_cast<int>(M), K9, l.cout, gy.p, l.cout, true, l.wk.p, K9, false, dcols.p, K9, false);
        *gx = alloc(x.n, x.c, x.h, x.w);
        k_col2im<<<grid_for(x.size()), 256, 0, st_>>>(dcols.p, gx->p, x.n, x.h, x.w, x.c, l.k, l.stride, l.pad, gy.h,
                                                      gy.w, 0);
        PBKD_LAUNCH_CHECK();
    }
}

DTensor NetExec::forward(DevBlock& b, const DTensor& x, bool train, BlockCacheDev* cache) {
    prepare(b);
    if (cache) {
        cache->train = train;
        cache->layers.assign(b.layers.size(), LayerCacheDev{});
    }
    DTensor cur = x;
    std::pair<DTensor, DTensor> stats;  // (mean, inv) handed from a pointwise GEMM to its batch norm
    for (size_t i = 0; i < b.layers.size(); ++i) {
        DevBlock::Layer& l = b.layers[i];
        if (cache) cache->layers[i].input = cur;
        DTensor next;
        switch (l.kind) {
            case LayerKind::Conv3x3:
            case LayerKind::Conv1x1:
            case LayerKind::Conv7x7:
                if (cur.c != l.cin) throw pbkd::ShapeError("conv: input channels do not match the layer");
                next = conv_fwd(l, cur);
                break;
            case LayerKind::DepthwiseConv3x3: {
                if (cur.c != l.cin) throw pbkd::ShapeError("depthwise: input channels do not match the layer");
                const int ho = (cur.h + 2 * l.pad - 3) / l.stride + 1, wo = (cur.w + 2 * l.pad - 3) / l.stride + 1;
                next = alloc(cur.n, cur.c, ho, wo);
                k_dw_fwd<<<grid_for(next.size()), 256, 0, st_>>>(cur.p, l.wk.p, next.p, cur.n, cur.h, cur.w, cur.c,
                                                                 ho, wo, l.stride, l.pad);
                PBKD_LAUNCH_CHECK();
                break;
            }
            case LayerKind::PointwiseConv: {
                if (cur.c != l.cin) throw pbkd::ShapeError("pointwise: input channels do not match the layer");
                if (l.stride != 1) {  // strided 1x1: the implicit-im2col conv
                    DevBlock::Layer tmp = l;
                    tmp.k = 1, tmp.pad = 0;
                    next = conv_fwd(tmp, cur);
                } else if (train && i + 1 < b.layers.size() && b.layers[i + 1].kind == LayerKind::BatchNorm) {
                    // pointwise + train-mode BN: the engine's GEMM epilogue
                    // partials and bn_stat_kernel (same statistics bits as
                    // the grouped student step)
                    const DevBlock::Layer& bn = b.layers[i + 1];
                    next = alloc(cur.n, l.cout, cur.h, cur.w);
                    stats = pw_bn_stats(cur, l.wk.p, l.cin, l.cout, next.p, b.at(bn.mm), b.at(bn.mv));
                } else {
                    next = alloc(cur.n, l.cout, cur.h, cur.w);
                    gemm(static_cast<int>(cur.rows()), l.cout, l.cin, cur.p, l.cin, true, l.wk.p, l.cin, true,
                         next.p, l.cout, false);
                }
                break;
            }
            case LayerKind::BatchNorm: {
                if (cur.c != l.cin) throw pbkd::ShapeError("batchnorm: channel count does not match");
                next = alloc(cur.n, cur.c, cur.h, cur.w);
                const long long tot = cur.size();
                if (train) {
                    DTensor mean, inv;
                    if (stats.first) {  // from the pointwise GEMM epilogue
                        mean = stats.first, inv = stats.second;
                        stats = {};
                    } else {
                        const int parts = parts_for(cur.rows());
                        DTensor p0 = alloc(1, 1, parts, cur.c), p1 = alloc(1, 1, parts, cur.c);
                        mean = alloc(1, 1, 1, cur.c), inv = alloc(1, 1, 1, cur.c);
                        k_col_part<0><<<dim3(ceil_div(cur.c, 128), parts), 128, 0, st_>>>(
                            cur.p, nullptr, static_cast<int>(cur.rows()), cur.c, parts, p0.p, p1.p);
                        k_bn_stats<<<ceil_div(cur.c, 128), 128, 0, st_>>>(p0.p, p1.p, parts, cur.c, cur.rows(), mean.p,
                                                                          inv.p, b.at(l.mm), b.at(l.mv));
                    }
                    DTensor xh;
                    if (cache) xh = alloc(cur.n, cur.c, cur.h, cur.w);
                    k_bn_apply<<<grid_for(tot), 256, 0, st_>>>(cur.p, next.p, xh ? xh.p : nullptr, tot, cur.c, mean.p,
                                                               inv.p, b.at(l.gamma), b.at(l.beta));
                    PBKD_LAUNCH_CHECK();
                    if (cache) {
                        cache->layers[i].xhat = xh;
                        cache->layers[i].inv = inv;
                    }
                } else {
                    DTensor sc = alloc(1, 1, 1, cur.c), sh = alloc(1, 1, 1, cur.c);
                    launch_bn_infer_prep(b.at(l.gamma), b.at(l.beta), b.at(l.mm), b.at(l.mv), cur.c, sc.p, sh.p, st_);
                    k_affine<<<grid_for(tot), 256, 0, st_>>>(cur.p, next.p, tot, cur.c, sc.p, sh.p);
                    PBKD_LAUNCH_CHECK();
                }
                break;
            }
            case LayerKind::ReLU:
                next = alloc(cur.n, cur.c, cur.h, cur.w);
                k_relu<<<grid_for(cur.size()), 256, 0, st_>>>(cur.p, next.p, cur.size());
                PBKD_LAUNCH_CHECK();
                break;
            case LayerKind::MaxPool3x3:
                next = alloc(cur.n, cur.c, (cur.h - 1) / 2 + 1, (cur.w - 1) / 2 + 1);
                launch_maxpool3x3(cur.p, next.p, nullptr, nullptr, cur.n, cur.h, cur.w, cur.c, st_);
                break;
            case LayerKind::GlobalAvgPool:
                next = alloc(cur.n, cur.c, 1, 1);
                k_gap<<<grid_for(static_cast<long long>(cur.n) * cur.c), 256, 0, st_>>>(cur.p, next.p, cur.n,
                                                                                        cur.h * cur.w, cur.c);
                PBKD_LAUNCH_CHECK();
                break;
            case LayerKind::Dense:
                if (cur.h != 1 || cur.w != 1)
                    throw pbkd::ShapeError("dense: expects 1x1 spatial input (apply global_avg_pool first)");
                if (cur.c != l.cin) throw pbkd::ShapeError("dense: input features do not match the kernel");
                next = alloc(cur.n, l.cout, 1, 1);
                k_dense<<<grid_for(static_cast<long long>(cur.n) * l.cout), 256, 0, st_>>>(
                    cur.p, b.at(l.w), l.b >= 0 ? b.at(l.b) : nullptr, next.p, cur.n, l.cin, l.cout);
                PBKD_LAUNCH_CHECK();
                break;
            case LayerKind::Add: {
                DTensor skip = x;  // the block input (model.cpp:540-546)
                if (l.w >= 0) skip = conv_fwd(l, x);
                if (skip.n != cur.n || skip.c != cur.c || skip.h != cur.h || skip.w != cur.w)
                    throw pbkd::ShapeError("add: skip path shape does not match the main path");
                next = alloc(cur.n, cur.c, cur.h, cur.w);
                k_add<<<grid_for(cur.size()), 256, 0, st_>>>(cur.p, skip.p, next.p, cur.size());
                PBKD_LAUNCH_CHECK();
                break;
            }
        }
        cur = std::move(next);
    }
    return cur;
}

DTensor NetExec::backward(DevBlock& b, const BlockCacheDev& cache, const DTensor& gy, bool need_gx, bool param_grads) {
    if (cache.layers.size() != b.layers.size()) throw std::logic_error("block_backward: cache does not match block");
    if (!cache.train && param_grads)
        throw std::logic_error("block_backward: parameter gradients require a train-mode cache");
    prepare(b);
    DTensor g = gy;
    DTensor skip_grad;
    for (int i = static_cast<int>(b.layers.size()) - 1; i >= 0; --i) {
        DevBlock::Layer& l = b.layers[static_cast<size_t>(i)];
        const DTensor& x = cache.layers[static_cast<size_t>(i)].input;
        const bool want_gx = i > 0 || need_gx;
        DTensor gx;
        switch (l.kind) {
            case LayerKind::Conv3x3:
            case LayerKind::Conv1x1:
            case LayerKind::Conv7x7:
                conv_bwd(b, l, x, g, want_gx ? &gx : nullptr, param_grads);
                break;
            case LayerKind::DepthwiseConv3x3: {
                if (param_grads) {
                    const int parts = parts_for(g.rows());
                    DTensor part = alloc(1, parts, 9, l.cin);
                    k_dw_wgrad_part<<<dim3(ceil_div(9LL * l.cin, 128), parts), 128, 0, st_>>>(
                        g.p, x.p, part.p, x.n, x.h, x.w, x.c, g.h, g.w, l.stride, l.pad, parts);
                    k_dw_wgrad_fin<<<ceil_div(9LL * l.cin, 128), 128, 0, st_>>>(part.p, parts, l.cin, b.grad_at(l.w));
                    PBKD_LAUNCH_CHECK();
                }
                if (want_gx) {
                    gx = alloc(x.n, x.c, x.h, x.w);
                    k_dw_dgrad<<<grid_for(x.size()), 256, 0, st_>>>(g.p, l.wk.p, gx.p, x.n, x.h, x.w, x.c, g.h, g.w,
                                                                    l.stride, l.pad);
                    PBKD_LAUNCH_CHECK();
                }
                break;
            }
            case LayerKind::PointwiseConv: {
                if (l.stride != 1) {
                    DevBlock::Layer tmp = l;
                    tmp.k = 1, tmp.pad = 0;
                    conv_bwd(b, tmp, x, g, want_gx ? &gx : nullptr, param_grads);
                    break;
                }
                const int M = static_cast<int>(x.rows());
                if (param_grads)  // gw[o][j] += sum_m gy[m][o] x[m][j]
                    gemm(l.cout, l.cin, M, g.p, l.cout, false, x.p, l.cin, false, b.grad_at(l.w), l.cin, true);
                if (want_gx) {  // gx[m][j] = sum_o gy[m][o] w[o][j]
                    gx = alloc(x.n, x.c, x.h, x.w);
                    gemm(M, l.cin, l.cout, g.p, l.cout, true, l.wk.p, l.cin, false, gx.p, l.cin, false);
                }
                break;
            }
            case LayerKind::BatchNorm: {
                const long long tot = g.size();
                if (want_gx) gx = alloc(x.n, x.c, x.h, x.w, true);
                if (cache.train) {
                    const LayerCacheDev& lc = cache.layers[static_cast<size_t>(i)];
                    const int parts = parts_for(g.rows());
                    DTensor p0 = alloc(1, 1, parts, g.c), p1 = alloc(1, 1, parts, g.c);
                    DTensor sg = alloc(1, 1, 1, g.c), sgx = alloc(1, 1, 1, g.c);
                    k_col_part<1><<<dim3(ceil_div(g.c, 128), parts), 128, 0, st_>>>(
                        g.p, lc.xhat.p, static_cast<int>(g.rows()), g.c, parts, p0.p, p1.p);
                    k_bn_bwd_sums<<<ceil_div(g.c, 128), 128, 0, st_>>>(
                        p0.p, p1.p, parts, g.c, sg.p, sgx.p, param_grads ? b.grad_at(l.gamma) : nullptr,
                        param_grads ? b.grad_at(l.beta) : nullptr);
                    if (want_gx) {
                        const float inv_m = 1.0f / static_cast<float>(g.rows());
                        k_bn_bwd_apply<<<grid_for(tot), 256, 0, st_>>>(g.p, lc.xhat.p, gx.p, tot, g.c, b.at(l.gamma),
                                                                       lc.inv.p, sg.p, sgx.p, inv_m);
                    }
                    PBKD_LAUNCH_CHECK();
                } else if (want_gx) {
                    k_bn_infer_bwd<<<grid_for(tot), 256, 0, st_>>>(g.p, b.at(l.gamma), b.at(l.mv), gx.p, tot, g.c);
                    PBKD_LAUNCH_CHECK();
                }
                break;
            }
            case LayerKind::ReLU:
                if (want_gx) {
                    gx = alloc(x.n, x.c, x.h, x.w);
                    k_relu_bwd<<<grid_for(x.size()), 256, 0, st_>>>(x.p, g.p, gx.p, x.size());
                    PBKD_LAUNCH_CHECK();
                }
                break;
            case LayerKind::MaxPool3x3:
                if (want_gx) {
                    gx = alloc(x.n, x.c, x.h, x.w, true);
                    launch_maxpool3x3_bwd(x.p, g.p, gx.p, x.n, x.h, x.w, x.c, st_);
                }
                break;
            case LayerKind::GlobalAvgPool:
                if (want_gx) {
                    gx = alloc(x.n, x.c, x.h, x.w, true);
                    k_gap_bwd<<<grid_for(x.size()), 256, 0, st_>>>(g.p, gx.p, x.n, x.h * x.w, x.c);
                    PBKD_LAUNCH_CHECK();
                }
                break;
            case LayerKind::Dense:
                if (param_grads) {
                    k_dense_wgrad<<<grid_for(static_cast<long long>(l.cout) * l.cin), 256, 0, st_>>>(
                        g.p, x.p, b.grad_at(l.w), l.b >= 0 ? b.grad_at(l.b) : nullptr, x.n, l.cin, l.cout);
                    PBKD_LAUNCH_CHECK();
                }
                if (want_gx) {
                    gx = alloc(x.n, x.c, 1, 1, true);
                    k_dense_dgrad<<<grid_for(static_cast<long long>(x.n) * l.cin), 256, 0, st_>>>(
                        g.p, b.at(l.w), gx.p, x.n, l.cin, l.cout);
                    PBKD_LAUNCH_CHECK();
                }
                break;
            case LayerKind::Add: {
                if (i == 0) throw std::logic_error("block_backward: Add cannot be the first layer");
                const DTensor& bin = cache.layers[0].input;
                if (l.w < 0) {
                    if (need_gx) {
                        if (!skip_grad) skip_grad = alloc(bin.n, bin.c, bin.h, bin.w, true);
                        axpy(skip_grad, g);
                    }
                } else if (param_grads || need_gx) {
                    DTensor sg;
                    conv_bwd(b, l, bin, g, need_gx ? &sg : nullptr, param_grads);
                    if (need_gx) {
                        if (!skip_grad) skip_grad = alloc(bin.n, bin.c, bin.h, bin.w, true);
                        axpy(skip_grad, sg);
                    }
                }
                gx = g;  // the sum passes the gradient to the main path
                break;
            }
        }
        g = want_gx ? gx : DTensor{};
    }
    if (need_gx && skip_grad) {
        DTensor out = alloc(g.n, g.c, g.h, g.w);
        k_add<<<grid_for(g.size()), 256, 0, st_>>>(g.p, skip_grad.p, out.p, g.size());
        PBKD_LAUNCH_CHECK();
        g = out;
    }
    return g;
}

void NetExec::axpy(DTensor& y, const DTensor& x) {
    k_axpy<<<grid_for(y.size()), 256, 0, st_>>>(y.p, x.p, y.size());
    PBKD_LAUNCH_CHECK();
}

float NetExec::mse(const DTensor& s, const DTensor& t) {
    if (s.size() != t.size()) throw pbkd::ShapeError("mse_local_loss: shape mismatch");
    DTensor d = alloc(1, 1, 1, 2);
    double* sum = reinterpret_cast<double*>(d.p);
    launch_mse_segments(s.p, t.p, s.size(), s.size(), 1, sum, st_);
    double h = 0.0;
    PBKD_CUDA(cudaMemcpyAsync(&h, sum, sizeof(double), cudaMemcpyDeviceToHost, st_));
    PBKD_CUDA(cudaStreamSynchronize(st_));
    return static_cast<float>(h / static_cast<double>(s.size()));
}

float NetExec::mse_step(const DTensor& s, const DTensor& t) {
    if (s.size() != t.size()) throw pbkd::ShapeError("mse_local_loss: shape mismatch");
    const long long rows = s.rows();
    const int ctas = rows_part_ctas(rows, s.c), per = rows_part_per(rows, ctas);
    DTensor part = alloc(1, 1, 1, ctas + 1);
    k_loss_parts<<<ctas, 256, 0, st_>>>(s.p, t.p, static_cast<int>(rows), s.c, per, part.p);
    k_loss_final<<<1, 32, 0, st_>>>(part.p, ctas, static_cast<double>(s.size()), part.p + ctas);
    PBKD_LAUNCH_CHECK();
    float h = 0.0f;
    PBKD_CUDA(cudaMemcpyAsync(&h, part.p + ctas, sizeof(float), cudaMemcpyDeviceToHost, st_));
    PBKD_CUDA(cudaStreamSynchronize(st_));
    return h;
}

void NetExec::mse_bwd(const DTensor& s, const DTensor& t, float scale, DTensor& g) {
    const float k = scale * 2.0f / static_cast<float>(s.size());  // ops.hpp:536
    k_mse_bwd<<<grid_for(s.size()), 256, 0, st_>>>(s.p, t.p, g.p, s.size(), k);
    PBKD_LAUNCH_CHECK();
}

double NetExec::softmax_ce(const DTensor& logits, const int* labels, DTensor* probs) {
    const int n = logits.n, k = logits.c;
    DTensor loss = alloc(1, 1, 1, n);
    if (probs) *probs = alloc(n, k, 1, 1);
    k_softmax_ce<<<grid_for(n), 256, 0, st_>>>(logits.p, labels, probs ? probs->p : nullptr, loss.p, n, k);
    PBKD_LAUNCH_CHECK();
    std::vector<float> h(static_cast<size_t>(n));
    PBKD_CUDA(cudaMemcpyAsync(h.data(), loss.p, h.size() * sizeof(float), cudaMemcpyDeviceToHost, st_));
    PBKD_CUDA(cudaStreamSynchronize(st_));
    float total = 0.0f;  // ops.hpp:497-500: float total, / n
    for (float v : h) total += v;
    return total / static_cast<float>(n);
}

void NetExec::softmax_ce_bwd(const DTensor& probs, const int* labels, float scale, DTensor& g) {
    const float inv_n = scale / static_cast<float>(probs.n);
    k_softmax_ce_bwd<<<grid_for(probs.size()), 256, 0, st_>>>(probs.p, labels, g.p, probs.n, probs.c, inv_n);
    PBKD_LAUNCH_CHECK();
}

long long NetExec::count_correct(const DTensor& logits, const int* labels) {
    DTensor d = alloc(1, 1, 1, 1, true);
    int* c = reinterpret_cast<int*>(d.p);
    k_argmax_correct<<<grid_for(logits.n), 256, 0, st_>>>(logits.p, labels, logits.n, logits.c, c);
    PBKD_LAUNCH_CHECK();
    int h = 0;
    PBKD_CUDA(cudaMemcpyAsync(&h, c, sizeof(int), cudaMemcpyDeviceToHost, st_));
    PBKD_CUDA(cudaStreamSynchronize(st_));
    return h;
}

void NetExec::zero_grads(DevBlock& b) {
    if (b.n) PBKD_CUDA(cudaMemsetAsync(b.grads.p, 0, b.n * sizeof(float), st_));
}

void NetExec::sgd(DevBlock& b, float lr, float momentum) {
    if (!(lr > 0.0f)) throw std::invalid_argument("sgd_step: lr must be > 0");
    if (momentum < 0.0f || momentum >= 1.0f) throw std::invalid_argument("sgd_step: momentum must be in [0,1)");
    auto step = [&](long long off, long long n) {
        if (off < 0 || n <= 0) return;
        k_sgd<<<grid_for(n), 256, 0, st_>>>(b.at(off), b.grad_at(off), b.vel.p + off, n, lr, momentum);
        PBKD_LAUNCH_CHECK();
    };
    for (const DevBlock::Layer& l : b.layers) {  // collect_block_trainable: weight, bias, gamma, beta
        step(l.w, l.wn);
        if (l.b >= 0) step(l.b, l.cout);
        if (l.kind == LayerKind::BatchNorm) {
            step(l.gamma, l.cin);
            step(l.beta, l.cin);
        }
    }
    b.derived_ok = false;
}

void NetExec::sync() { PBKD_CUDA(cudaStreamSynchronize(st_)); }

}  // namespace pbkd_gpu
