// ops.cu -- grouped student-step kernels and small helpers (sm_100a).
//
// Exactness notes: elementwise paths (depthwise
// forward, depthwise input-gradient gather, ReLU, batch-norm apply/backward
// apply, MSE gradient, SGD) use the _rn intrinsics in the reference's
// evaluation order and agree bit for bit given identical inputs.  Reductions
// (batch-norm statistics, MSE sum, weight gradients, GEMM K) use fixed-shape
// trees: deterministic run to run, equal to the reference within fp32
// tolerance.
#include <algorithm>

#include "ops.cuh"

namespace pbkd_gpu {

// ---------------------------------------------------------------- partition
int rows_part_ctas(long long rows, int c) {
    const long long elems = rows * static_cast<long long>(c);
    long long ctas = (elems + 4095) / 4096;
    ctas = std::max<long long>(1, std::min<long long>(ctas, 1024));
    ctas = std::min<long long>(ctas, rows);
    const int per = rows_part_per(rows, static_cast<int>(ctas));
    return ceil_div(rows, per);
}
int rows_part_per(long long rows, int ctas) { return ceil_div(rows, ctas); }
int ctas_elem(long long total) { return std::max(1, ceil_div(total, 256LL * 4)); }

template <class Op>
__device__ __forceinline__ const Op& op_of(const Op* ops, int nd, int& local) {
    const int t = op_index(ops, nd, static_cast<int>(blockIdx.x));
    local = static_cast<int>(blockIdx.x) - ops[t].cta_begin;
    return ops[t];
}

__device__ __forceinline__ bool is_failed(const int* f) { return f != nullptr && *f != 0; }

// channel-group geometry shared by the row-partitioned kernels
struct Geo {
    int V, G, RP;  // vector width, channel groups, rows processed in parallel
};
__device__ __forceinline__ Geo geo_of(int c) {
    Geo g;
    g.V = (c % 4 == 0) ? 4 : 1;
    g.G = c / g.V;
    g.RP = max(1, kThreads / g.G);
    return g;
}

__device__ __forceinline__ void load_v(const float* p, int V, float* out) {
    if (V == 4) {
        const float4 q = *reinterpret_cast<const float4*>(p);
        out[0] = q.x, out[1] = q.y, out[2] = q.z, out[3] = q.w;
    } else {
        out[0] = p[0];
    }
}
__device__ __forceinline__ void store_v(float* p, int V, const float* v) {
    if (V == 4)
        *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
    else
        p[0] = v[0];
}

// Reduce per-thread V-vectors over the RP row lanes in fixed order and
// write the CTA's partial row (length c) to out.
__device__ void cta_reduce_rows(float* red, const float* v, const Geo& g, int rr, int gg,
                                bool lane_ok, int c, float* out) {
    if (lane_ok)
        for (int q = 0; q < g.V; ++q) red[rr * c + gg * g.V + q] = v[q];
    __syncthreads();
    for (int ch = threadIdx.x; ch < c; ch += blockDim.x) {
        float s = 0.0f;
        for (int r = 0; r < g.RP; ++r) s += red[r * c + ch];
        out[ch] = s;
    }
    __syncthreads();
}

// ---------------------------------------------------------- depthwise fwd
int ctas_dw_fwd(const DwFwdOp& o) {
    const int V = (o.c % 4 == 0) ? 4 : 1;
    return std::max(1, ceil_div(static_cast<long long>(o.n) * o.ho * o.wo * (o.c / V), kThreads));
}

__global__ void __launch_bounds__(kThreads) dw_fwd_kernel(const DwFwdOp* __restrict__ ops, int nd) {
    int local;
    const DwFwdOp& o = op_of(ops, nd, local);
    if (is_failed(o.failed)) return;
    const int V = (o.c % 4 == 0) ? 4 : 1;
    const int G = o.c / V;
    const long long idx = static_cast<long long>(local) * kThreads + threadIdx.x;
    const long long total = static_cast<long long>(o.n) * o.ho * o.wo * G;
    if (idx >= total) return;
    const int g = static_cast<int>(idx % G);
    const long long r = idx / G;
    const int ox = static_cast<int>(r % o.wo);
    const int oy = static_cast<int>((r / o.wo) % o.ho);
    const int n = static_cast<int>(r / (static_cast<long long>(o.wo) * o.ho));
    const int c0 = g * V;
    float pa[4], pb[4], pc[4], pd[4];
    if (o.pro != 0) {
        load_v(o.pa + c0, V, pa);
        load_v(o.pb + c0, V, pb);
        if (o.pro == 1) {
            load_v(o.pc + c0, V, pc);
            load_v(o.pd + c0, V, pd);
        }
    }
    float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    for (int ky = 0; ky < 3; ++ky) {
        const int iy = oy * o.stride - o.pad + ky;
        if (iy < 0 || iy >= o.h) continue;
        for (int kx = 0; kx < 3; ++kx) {
            const int ix = ox * o.stride - o.pad + kx;
            if (ix < 0 || ix >= o.wd) continue;
            float xv[4], wv[4];
            load_v(o.x + ((static_cast<long long>(n) * o.h + iy) * o.wd + ix) * o.c + c0, V, xv);
            load_v(o.w + (ky * 3 + kx) * o.c + c0, V, wv);
            for (int q = 0; q < V; ++q) {
                float v = xv[q];
                if (o.pro == 1) v = relu(bn_train_apply(v, pa[q], pb[q], pc[q], pd[q]));
                else if (o.pro == 2) v = relu(bn_infer_apply(v, pa[q], pb[q]));
                acc[q] = add(acc[q], mul(v, wv[q]));
            }
        }
    }
    store_v(o.y + r * o.c + c0, V, acc);
}

void launch_dw_fwd(const DwFwdOp* d, int nd, int ctas, cudaStream_t st) {
    dw_fwd_kernel<<<ctas, kThreads, 0, st>>>(d, nd);
    PBKD_LAUNCH_CHECK();
}

// ------------------------------------------- depthwise bwd (unit > 0, s=1)
__global__ void __launch_bounds__(kThreads) dw_bwd_kernel(const DwBwdOp* __restrict__ ops, int nd) {
    extern __shared__ float red[];
    int local;
    const DwBwdOp& o = op_of(ops, nd, local);
    if (is_failed(o.failed)) return;
    const Geo g = geo_of(o.c);
    const int rr = threadIdx.x / g.G, gg = threadIdx.x % g.G;
    const bool lane_ok = rr < g.RP;
    const long long rows = static_cast<long long>(o.n) * o.h * o.wd;
    const long long r0 = static_cast<long long>(local) * o.rows_per;
    const long long r1 = min(rows, r0 + o.rows_per);
    const int c0 = gg * g.V;
    float mean[4], inv[4], gam[4], bet[4], wk[9][4];
    float gk[9][4], sg[4], sgx[4];
    if (lane_ok) {
        load_v(o.mean + c0, g.V, mean);
        load_v(o.inv + c0, g.V, inv);
        load_v(o.gamma + c0, g.V, gam);
        load_v(o.beta + c0, g.V, bet);
        for (int t = 0; t < 9; ++t) load_v(o.w + t * o.c + c0, g.V, wk[t]);
    }
    for (int t = 0; t < 9; ++t)
        for (int q = 0; q < 4; ++q) gk[t][q] = 0.0f;
    for (int q = 0; q < 4; ++q) sg[q] = sgx[q] = 0.0f;
    if (lane_ok) {
        for (long long r = r0 + rr; r < r1; r += g.RP) {
            const int x = static_cast<int>(r % o.wd);
            const int y = static_cast<int>((r / o.wd) % o.h);
            const long long nbase = (r / (static_cast<long long>(o.wd) * o.h)) * o.h;
            // (a) input gradient: outputs touching (y,x) in ascending (oy,ox)
            //     order, tap (1-dy, 1-dx) (ops.hpp:156-174, skip g == 0)
            float gx[4] = {0.0f, 0.0f, 0.0f, 0.0f};
            float gyc[4];
            load_v(o.gy + r * o.c + c0, g.V, gyc);
            for (int dy = -1; dy <= 1; ++dy) {
                const int oy = y + dy;
                if (oy < 0 || oy >= o.h) continue;
                for (int dx = -1; dx <= 1; ++dx) {
                    const int ox = x + dx;
                    if (ox < 0 || ox >= o.wd) continue;
                    float gv[4];
                    load_v(o.gy + ((nbase + oy) * o.wd + ox) * o.c + c0, g.V, gv);
                    const int tap = (1 - dy) * 3 + (1 - dx);
                    for (int q = 0; q < g.V; ++q)
                        if (gv[q] != 0.0f) gx[q] = add(gx[q], mul(gv[q], wk[tap][q]));
                }
            }
            // (b) weight-gradient partials: this output times its 9 inputs,
            //     inputs rebuilt as relu(bn(p_prev))
            for (int ky = 0; ky < 3; ++ky) {
                const int iy = y - 1 + ky;
                if (iy < 0 || iy >= o.h) continue;
                for (int kx = 0; kx < 3; ++kx) {
                    const int ix = x - 1 + kx;
                    if (ix < 0 || ix >= o.wd) continue;
                    float pv[4];
                    load_v(o.xp + ((nbase + iy) * o.wd + ix) * o.c + c0, g.V, pv);
                    for (int q = 0; q < g.V; ++q) {
                        const float xin = relu(bn_train_apply(pv[q], mean[q], inv[q], gam[q], bet[q]));
                        if (gyc[q] != 0.0f) gk[ky * 3 + kx][q] += gyc[q] * xin;
                    }
                }
            }
            // (c) previous unit's ReLU mask and batch-norm partial sums
            float pc[4], outv[4];
            load_v(o.xp + r * o.c + c0, g.V, pc);
            for (int q = 0; q < g.V; ++q) {
                const float xh = mul(sub(pc[q], mean[q]), inv[q]);
                const float yv = add(mul(gam[q], xh), bet[q]);
                const float gm = yv > 0.0f ? add(0.0f, gx[q]) : 0.0f;
                outv[q] = gm;
                sg[q] += gm;
                sgx[q] += gm * xh;
            }
            store_v(o.gyprev + r * o.c + c0, g.V, outv);
        }
    }
    for (int t = 0; t < 9; ++t)
        cta_reduce_rows(red, gk[t], g, rr, gg, lane_ok, o.c,
                        o.part_gk + (static_cast<long long>(local) * 9 + t) * o.c);
    cta_reduce_rows(red, sg, g, rr, gg, lane_ok, o.c, o.part_sg + static_cast<long long>(local) * o.c);
    cta_reduce_rows(red, sgx, g, rr, gg, lane_ok, o.c, o.part_sgx + static_cast<long long>(local) * o.c);
}

static size_t red_smem(int cmax) { return static_cast<size_t>(kThreads) * 4 * sizeof(float) + cmax * 0; }

void launch_dw_bwd(const DwBwdOp* d, int nd, int ctas, cudaStream_t st) {
    // RP*c <= kThreads*V <= 1024 floats
    dw_bwd_kernel<<<ctas, kThreads, red_smem(0), st>>>(d, nd);
    PBKD_LAUNCH_CHECK();
}

// ------------------------------------------- depthwise weight grad (unit 0)
__global__ void __launch_bounds__(kThreads) dw_gk_kernel(const DwGkOp* __restrict__ ops, int nd) {
    extern __shared__ float red[];
    int local;
    const DwGkOp& o = op_of(ops, nd, local);
    if (is_failed(o.failed)) return;
    const Geo g = geo_of(o.c);
    const int rr = threadIdx.x / g.G, gg = threadIdx.x % g.G;
    const bool lane_ok = rr < g.RP;
    const long long rows = static_cast<long long>(o.n) * o.ho * o.wo;
    const long long r0 = static_cast<long long>(local) * o.rows_per;
    const long long r1 = min(rows, r0 + o.rows_per);
    const int c0 = gg * g.V;
    float gk[9][4];
    for (int t = 0; t < 9; ++t)
        for (int q = 0; q < 4; ++q) gk[t][q] = 0.0f;
    if (lane_ok) {
        for (long long r = r0 + rr; r < r1; r += g.RP) {
            const int ox = static_cast<int>(r % o.wo);
            const int oy = static_cast<int>((r / o.wo) % o.ho);
            const long long n = r / (static_cast<long long>(o.wo) * o.ho);
            float gv[4];
            load_v(o.gy + r * o.c + c0, g.V, gv);
            for (int ky = 0; ky < 3; ++ky) {
                const int iy = oy * o.stride - o.pad + ky;
                if (iy < 0 || iy >= o.h) continue;
                for (int kx = 0; kx < 3; ++kx) {
                    const int ix = ox * o.stride - o.pad + kx;
                    if (ix < 0 || ix >= o.wd) continue;
                    float xv[4];
                    load_v(o.x + ((n * o.h + iy) * o.wd + ix) * o.c + c0, g.V, xv);
                    for (int q = 0; q < g.V; ++q)
                        if (gv[q] != 0.0f) gk[ky * 3 + kx][q] += gv[q] * xv[q];
                }
            }
        }
    }
    for (int t = 0; t < 9; ++t)
        cta_reduce_rows(red, gk[t], g, rr, gg, lane_ok, o.c,
                        o.part_gk + (static_cast<long long>(local) * 9 + t) * o.c);
}

void launch_dw_gk(const DwGkOp* d, int nd, int ctas, cudaStream_t st) {
    dw_gk_kernel<<<ctas, kThreads, red_smem(0), st>>>(d, nd);
    PBKD_LAUNCH_CHECK();
}

// --------------------------------------------------------- fixed-order sums
__global__ void __launch_bounds__(kThreads) reduce_kernel(const ReduceOp* __restrict__ ops, int nd) {
    int local;
    const ReduceOp& o = op_of(ops, nd, local);
    if (is_failed(o.failed)) return;
    const int i = local * kThreads + threadIdx.x;
    if (i >= o.width) return;
    float s = 0.0f;
    for (int p = 0; p < o.parts; ++p) s += o.part[static_cast<long long>(p) * o.width + i];
    o.out[i] = s;
}

void launch_reduce(const ReduceOp* d, int nd, int ctas, cudaStream_t st) {
    reduce_kernel<<<ctas, kThreads, 0, st>>>(d, nd);
    PBKD_LAUNCH_CHECK();
}

// ------------------------------------------------------------ BN statistics
// Column sums of [parts][c] partials: a CTA owns 32 channels, 8 lanes stride
// over the parts, lanes combine in fixed order (deterministic, latency-hidden).
constexpr int kColLanes = kThreads / 32;
int ctas_cols(int c) { return ceil_div(c, 32); }

__device__ __forceinline__ float col_sum(const float* __restrict__ part, int parts, int c, int ch,
                                         float (*red)[32]) {
    const int lane = threadIdx.x / 32, col = threadIdx.x % 32;
    float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    if (ch < c) {
        int p = lane;
        for (; p + 3 * kColLanes < parts; p += 4 * kColLanes)
#pragma unroll
            for (int u = 0; u < 4; ++u) acc[u] += part[static_cast<long long>(p + u * kColLanes) * c + ch];
        for (; p < parts; p += kColLanes) acc[0] += part[static_cast<long long>(p) * c + ch];
    }
    red[lane][col] = (acc[0] + acc[1]) + (acc[2] + acc[3]);
    __syncthreads();
    float s = 0.0f;
    for (int l = 0; l < kColLanes; ++l) s += red[l][col];
    __syncthreads();
    return s;
}

__global__ void __launch_bounds__(kThreads) bn_stat_kernel(const BnStatOp* __restrict__ ops, int nd) {
    __shared__ float red[kColLanes][32];
    int local;
    const BnStatOp& o = op_of(ops, nd, local);
    if (is_failed(o.failed)) return;
    const int ch = local * 32 + threadIdx.x % 32;
    const float sum = col_sum(o.part_sum, o.tiles, o.c, ch, red);
    const float sq = col_sum(o.part_sq, o.tiles, o.c, ch, red);
    if (threadIdx.x >= 32 || ch >= o.c) return;
    const float fm = static_cast<float>(o.m);
    const float mean = __fdiv_rn(sum, fm);
    float var = sub(__fdiv_rn(sq, fm), mul(mean, mean));
    if (var < 0.0f) var = 0.0f;
    const float inv = __fdiv_rn(1.0f, __fsqrt_rn(add(var, 1e-5f)));
    o.mean[ch] = mean;
    o.inv[ch] = inv;
    if (o.update_moving) {
        const float mom = 0.9f, one_m = sub(1.0f, mom);
        o.mm[ch] = add(mul(mom, o.mm[ch]), mul(one_m, mean));
        o.mv[ch] = add(mul(mom, o.mv[ch]), mul(one_m, var));
    }
}

void launch_bn_stat(const BnStatOp* d, int nd, int ctas, cudaStream_t st) {
    bn_stat_kernel<<<ctas, kThreads, 0, st>>>(d, nd);
    PBKD_LAUNCH_CHECK();
}

// ------------------------------------------------------------- loss + BN
__global__ void __launch_bounds__(kThreads) loss_kernel(const LossOp* __restrict__ ops, int nd) {
    extern __shared__ float red[];
    __shared__ float lred[kThreads];
    int local;
    const LossOp& o = op_of(ops, nd, local);
    if (is_failed(o.failed)) return;
    const Geo g = geo_of(o.c);
    const int rr = threadIdx.x / g.G, gg = threadIdx.x % g.G;
    const bool lane_ok = rr < g.RP;
    const long long r0 = static_cast<long long>(local) * o.rows_per;
    const long long r1 = min(static_cast<long long>(o.rows), r0 + o.rows_per);
    const int c0 = gg * g.V;
    float sg[4] = {0, 0, 0, 0}, sgx[4] = {0, 0, 0, 0};
    float lsum = 0.0f;
    if (lane_ok) {
        float mean[4], inv[4], gam[4], bet[4];
        load_v(o.mean + c0, g.V, mean);
        load_v(o.inv + c0, g.V, inv);
        load_v(o.gamma + c0, g.V, gam);
        load_v(o.beta + c0, g.V, bet);
        for (long long r = r0 + rr; r < r1; r += g.RP) {
            float pv[4], tv[4];
            load_v(o.p + r * o.c + c0, g.V, pv);
            load_v(o.t + r * o.c + c0, g.V, tv);
            for (int q = 0; q < g.V; ++q) {
                const float xh = mul(sub(pv[q], mean[q]), inv[q]);
                const float y = add(mul(gam[q], xh), bet[q]);
                const float d = sub(relu(y), tv[q]);
                lsum += d * d;
                const float gy = y > 0.0f ? add(0.0f, mul(o.kmse, d)) : 0.0f;
                sg[q] += gy;
                sgx[q] += gy * xh;
            }
        }
    }
    cta_reduce_rows(red, sg, g, rr, gg, lane_ok, o.c, o.part_sg + static_cast<long long>(local) * o.c);
    cta_reduce_rows(red, sgx, g, rr, gg, lane_ok, o.c, o.part_sgx + static_cast<long long>(local) * o.c);
    lred[threadIdx.x] = lsum;
    __syncthreads();
    if (threadIdx.x == 0) {
        float s = 0.0f;
        for (int i = 0; i < kThreads; ++i) s += lred[i];
        o.part_loss[local] = s;
    }
}

void launch_loss(const LossOp* d, int nd, int ctas, cudaStream_t st) {
    loss_kernel<<<ctas, kThreads, red_smem(0), st>>>(d, nd);
    PBKD_LAUNCH_CHECK();
}

__global__ void __launch_bounds__(kThreads) bn_bwd_fin_kernel(const BnBwdFinOp* __restrict__ ops, int nd) {
    __shared__ float red[kColLanes][32];
    int local;
    const BnBwdFinOp& o = op_of(ops, nd, local);
    if (is_failed(o.failed)) return;
    if (o.loss_out && local == 0 && threadIdx.x < 32) {  // one warp, fixed-order tree
        double s = 0.0;
        for (int p = threadIdx.x; p < o.ctas; p += 32) s += static_cast<double>(o.part_loss[p]);
        for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off);
        if (threadIdx.x == 0) {
            const float loss = static_cast<float>(s / o.count);
            *o.loss_out = loss;
            if (!isfinite(loss)) *o.failed = 1;
        }
    }
    const int ch = local * 32 + threadIdx.x % 32;
    const float a = col_sum(o.part_sg, o.ctas, o.c, ch, red);
    const float b = col_sum(o.part_sgx, o.ctas, o.c, ch, red);
    if (threadIdx.x >= 32 || ch >= o.c) return;
    o.sg[ch] = a;
    o.sgx[ch] = b;
    o.gbeta[ch] = a;
    o.ggamma[ch] = b;
}

void launch_bn_bwd_fin(const BnBwdFinOp* d, int nd, int ctas, cudaStream_t st) {
    bn_bwd_fin_kernel<<<ctas, kThreads, 0, st>>>(d, nd);
    PBKD_LAUNCH_CHECK();
}

__global__ void __launch_bounds__(kThreads) bn_bwd_apply_kernel(const BnBwdApplyOp* __restrict__ ops, int nd) {
    int local;
    const BnBwdApplyOp& o = op_of(ops, nd, local);
    if (is_failed(o.failed)) return;
    const long long base = (static_cast<long long>(local) * kThreads + threadIdx.x) * 4;
    for (int q = 0; q < 4; ++q) {
        const long long i = base + q;
        if (i >= o.total) return;
        const int ch = static_cast<int>(i % o.c);
        const float xh = mul(sub(o.p[i], o.mean[ch]), o.inv[ch]);
        float gy;
        if (o.t) {
            const float y = add(mul(o.gamma[ch], xh), o.beta[ch]);
            const float d = sub(relu(y), o.t[i]);
            gy = y > 0.0f ? add(0.0f, mul(o.kmse, d)) : 0.0f;
        } else {
            gy = o.gin[i];
        }
        const float kk = mul(o.gamma[ch], o.inv[ch]);
        const float inner = sub(sub(gy, mul(o.inv_m, o.sg[ch])), mul(mul(xh, o.inv_m), o.sgx[ch]));
        o.gout[i] = add(0.0f, mul(kk, inner));
    }
}

void launch_bn_bwd_apply(const BnBwdApplyOp* d, int nd, int ctas, cudaStream_t st) {
    bn_bwd_apply_kernel<<<ctas, kThreads, 0, st>>>(d, nd);
    PBKD_LAUNCH_CHECK();
}

// -------------------------------------------------------------------- SGD
__global__ void __launch_bounds__(kThreads) sgd_kernel(const SgdOp* __restrict__ ops, int nd) {
    int local;
    const SgdOp& o = op_of(ops, nd, local);
    if (is_failed(o.failed)) return;
    const long long base = (static_cast<long long>(local) * kThreads + threadIdx.x) * 4;
    for (int q = 0; q < 4; ++q) {
        const long long i = base + q;
        if (i >= o.n) return;
        const float v = add(mul(o.mom, o.v[i]), o.g[i]);
        o.v[i] = v;
        o.w[i] = sub(o.w[i], mul(o.lr, v));
    }
}

void launch_sgd(const SgdOp* d, int nd, int ctas, cudaStream_t st) {
    sgd_kernel<<<ctas, kThreads, 0, st>>>(d, nd);
    PBKD_LAUNCH_CHECK();
}

// ---------------------------------------------------------------- scatter
__global__ void __launch_bounds__(kThreads) scatter_kernel(const ScatterOp* __restrict__ ops, int nd) {
    int local;
    const ScatterOp& o = op_of(ops, nd, local);
    const bool v4 = (o.width % 4) == 0;
    const int wv = v4 ? o.width / 4 : o.width;
    const long long total = static_cast<long long>(o.rows) * wv;
    for (long long i = static_cast<long long>(local) * kThreads + threadIdx.x; i < total;
         i += static_cast<long long>(kThreads) * 64) {
        const long long r = i / wv, j = i - r * wv;
        const long long dr = o.pos[r];
        if (v4)
            reinterpret_cast<float4*>(o.dst + dr * o.width)[j] =
                reinterpret_cast<const float4*>(o.src + r * o.width)[j];
        else
            o.dst[dr * o.width + j] = o.src[r * o.width + j];
    }
}

void launch_scatter(const ScatterOp* d, int nd, int ctas, cudaStream_t st) {
    scatter_kernel<<<ctas, kThreads, 0, st>>>(d, nd);
    PBKD_LAUNCH_CHECK();
}

// ---------------------------------------------------------- non-grouped ---
__global__ void gather_nhwc_kernel(const float* __restrict__ img, const int* __restrict__ idx, int n,
                                   int c, int h, int w, float* __restrict__ out) {
    const long long total = static_cast<long long>(n) * c * h * w;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int ch = static_cast<int>(i % c);
        const long long pix = i / c;
        const int x = static_cast<int>(pix % w);
        const int y = static_cast<int>((pix / w) % h);
        const long long s = pix / (static_cast<long long>(w) * h);
        const long long src = idx ? idx[s] : s;
        out[i] = img[((src * c + ch) * h + y) * w + x];
    }
}

void launch_gather_nhwc(const float* images, const int* idx, int n, int c, int h, int w, float* out,
                        cudaStream_t st) {
    const long long total = static_cast<long long>(n) * c * h * w;
    const int blocks = static_cast<int>(std::min<long long>(4096, (total + 255) / 256));
    gather_nhwc_kernel<<<std::max(1, blocks), 256, 0, st>>>(images, idx, n, c, h, w, out);
    PBKD_LAUNCH_CHECK();
}

__global__ void bn_infer_prep_kernel(const float* gamma, const float* beta, const float* mm,
                                     const float* mv, int c, float* scale, float* shift) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= c) return;
    const float inv = __fdiv_rn(1.0f, __fsqrt_rn(add(mv[j], 1e-5f)));
    const float sc = mul(gamma[j], inv);
    scale[j] = sc;
    shift[j] = sub(beta[j], mul(mm[j], sc));
}

void launch_bn_infer_prep(const float* gamma, const float* beta, const float* mm, const float* mv,
                          int c, float* scale, float* shift, cudaStream_t st) {
    bn_infer_prep_kernel<<<ceil_div(c, 256), 256, 0, st>>>(gamma, beta, mm, mv, c, scale, shift);
    PBKD_LAUNCH_CHECK();
}

__global__ void bn_infer_relu_kernel(const float* x, float* y, long long total, int c,
                                     const float* scale, const float* shift) {
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int ch = static_cast<int>(i % c);
        y[i] = relu(bn_infer_apply(x[i], scale[ch], shift[ch]));
    }
}

void launch_bn_infer_relu(const float* x, float* y, long long total, int c, const float* scale,
                          const float* shift, cudaStream_t st) {
    const int blocks = static_cast<int>(std::min<long long>(4096, (total + 255) / 256));
    bn_infer_relu_kernel<<<std::max(1, blocks), 256, 0, st>>>(x, y, total, c, scale, shift);
    PBKD_LAUNCH_CHECK();
}

// one CTA per segment: fixed-order double sum of (s-t)^2
__global__ void mse_segments_kernel(const float* s, const float* t, long long seg, long long total,
                                    double* out) {
    __shared__ double red[256];
    const long long b = static_cast<long long>(blockIdx.x) * seg;
    const long long e = min(total, b + seg);
    double acc = 0.0;
    for (long long i = b + threadIdx.x; i < e; i += blockDim.x) {
        const float d = s[i] - t[i];
        acc += static_cast<double>(d * d);
    }
    red[threadIdx.x] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = 0.0;
        for (int i = 0; i < 256; ++i) a += red[i];
        out[blockIdx.x] = a;
    }
}

void launch_mse_segments(const float* s, const float* t, long long seg, long long total, int nseg,
                         double* out, cudaStream_t st) {
    mse_segments_kernel<<<nseg, 256, 0, st>>>(s, t, seg, total, out);
    PBKD_LAUNCH_CHECK();
}

// One CTA per sample.  GAP and dense keep the reference's serial order per
// output (ops.hpp:395-442); argmax keeps the first maximum (distill.cpp:42-52).
__global__ void classifier_kernel(const float* __restrict__ x, int hw, int c, const int* kinds,
                                  int nlayers, const float* dw, const float* db, int nout,
                                  const int* labels, int* correct) {
    extern __shared__ float vec[];  // 2 * max(c, nout) floats
    const int n = blockIdx.x;
    float* cur = vec;
    float* nxt = vec + max(c, nout);
    int width = c;
    bool pooled = false;
    const float* wp = dw;
    const float* bp = db;
    for (int l = 0; l < nlayers; ++l) {
        const int kind = kinds[2 * l];
        const int outw = kinds[2 * l + 1];
        if (kind == 0) {  // global average pool
            for (int ch = threadIdx.x; ch < c; ch += blockDim.x) {
                float s = 0.0f;
                for (int i = 0; i < hw; ++i) s = add(s, x[(static_cast<long long>(n) * hw + i) * c + ch]);
                cur[ch] = __fdiv_rn(s, static_cast<float>(hw));
            }
            pooled = true;
        } else if (kind == 1) {  // relu
            for (int ch = threadIdx.x; ch < width; ch += blockDim.x) cur[ch] = relu(cur[ch]);
        } else {  // dense [outw][width] + bias[outw]
            for (int o = threadIdx.x; o < outw; o += blockDim.x) {
                float acc = bp[o];
                for (int j = 0; j < width; ++j) acc = add(acc, mul(wp[o * width + j], cur[j]));
                nxt[o] = acc;
            }
            __syncthreads();
            float* tmp = cur;
            cur = nxt;
            nxt = tmp;
            wp += static_cast<long long>(outw) * width;
            bp += outw;
            width = outw;
        }
        __syncthreads();
    }
    (void)pooled;
    if (threadIdx.x == 0) {
        int best = 0;
        float bv = cur[0];
        for (int j = 1; j < width; ++j)
            if (cur[j] > bv) {
                bv = cur[j];
                best = j;
            }
        if (best == labels[n]) atomicAdd(correct, 1);
    }
}

void launch_classifier_count(const float* x, int n, int hw, int c, const int* kinds, int nlayers,
                             const float* dw, const float* db, int nout, const int* labels,
                             int* correct, cudaStream_t st) {
    const size_t smem = 2 * sizeof(float) * std::max(c, nout) + 64;
    classifier_kernel<<<n, 128, smem, st>>>(x, hw, c, kinds, nlayers, dw, db, nout, labels, correct);
    PBKD_LAUNCH_CHECK();
}

}  // namespace pbkd_gpu
