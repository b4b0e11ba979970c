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
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "dw_tile.cuh"
#include "ops.cuh"
#include "tc.cuh"

namespace pbkd_gpu {

bool pdl_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("PBKD_PDL");
        return !(e && e[0] == '0');
    }();
    return on;
}

// ------------------------------------------------------------ CTA tracer
// Diagnosis only (build with NVEXTRA=-DPBKD_GEMM_TRACE_BUILD, run with
// PBKD_CTA_TRACE=<kernel name>): globaltimer stamps per CTA at 4 points,
// summarised per launch on stderr.
#ifdef PBKD_GEMM_TRACE_BUILD
__device__ unsigned long long* g_cta_trace = nullptr;
__device__ __forceinline__ void cta_mark(int ev) {
    unsigned long long* tr = g_cta_trace;
    if (threadIdx.x == 0 && tr != nullptr) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        tr[blockIdx.x * 4 + ev] = t;
    }
}
template <class Launch>
void traced(const char* name, int ctas, cudaStream_t st, Launch launch) {
    static const char* want = std::getenv("PBKD_CTA_TRACE");
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    PBKD_CUDA(cudaStreamIsCapturing(st, &cap));
    if (!want || std::strcmp(want, name) != 0 || cap != cudaStreamCaptureStatusNone) {
        launch();
        return;
    }
    unsigned long long* buf = nullptr;
    PBKD_CUDA(cudaMalloc(&buf, static_cast<size_t>(ctas) * 4 * 8));
    PBKD_CUDA(cudaMemsetAsync(buf, 0, static_cast<size_t>(ctas) * 4 * 8, st));
    PBKD_CUDA(cudaMemcpyToSymbolAsync(g_cta_trace, &buf, sizeof(buf), 0, cudaMemcpyHostToDevice, st));
    launch();
    unsigned long long* none = nullptr;
    PBKD_CUDA(cudaMemcpyToSymbolAsync(g_cta_trace, &none, sizeof(none), 0, cudaMemcpyHostToDevice, st));
    std::vector<unsigned long long> h(static_cast<size_t>(ctas) * 4);
    PBKD_CUDA(cudaMemcpyAsync(h.data(), buf, h.size() * 8, cudaMemcpyDeviceToHost, st));
    PBKD_CUDA(cudaStreamSynchronize(st));
    PBKD_CUDA(cudaFree(buf));
    unsigned long long t0 = ~0ull, t1 = 0;
    for (int b = 0; b < ctas; ++b)
        if (h[b * 4]) t0 = std::min(t0, h[b * 4]), t1 = std::max(t1, h[b * 4 + 3]);
    std::vector<double> ph[3];
    for (int b = 0; b < ctas; ++b) {
        if (!h[b * 4] || !h[b * 4 + 1] || !h[b * 4 + 2] || !h[b * 4 + 3]) continue;
        for (int k = 0; k < 3; ++k) ph[k].push_back((h[b * 4 + k + 1] - h[b * 4 + k]) * 1e-3);
    }
    auto med = [](std::vector<double> v) {
        if (v.empty()) return 0.0;
        std::nth_element(v.begin(), v.begin() + v.size() / 2, v.end());
        return v[v.size() / 2];
    };
    auto mx = [](const std::vector<double>& v) { return v.empty() ? 0.0 : *std::max_element(v.begin(), v.end()); };
    static int no = 0;
    std::fprintf(stderr, "[cta-trace] %s #%d ctas=%d span %.2f us | setup med %.2f max %.2f | stage med %.2f max %.2f | compute med %.2f max %.2f\n",
                 name, no++, ctas, (t1 - t0) * 1e-3, med(ph[0]), mx(ph[0]), med(ph[1]), mx(ph[1]), med(ph[2]), mx(ph[2]));
    // start-time histogram (waves)
    std::vector<double> st0;
    for (int b = 0; b < ctas; ++b)
        if (h[b * 4]) st0.push_back((h[b * 4] - t0) * 1e-3);
    std::sort(st0.begin(), st0.end());
    std::fprintf(stderr, "[cta-trace]   starts: p10 %.2f p50 %.2f p90 %.2f max %.2f\n", st0[st0.size() / 10], st0[st0.size() / 2],
                 st0[st0.size() * 9 / 10], st0.back());
}
#else
__device__ __forceinline__ void cta_mark(int) {}
template <class Launch>
void traced(const char*, int, cudaStream_t, Launch launch) {
    launch();
}
#endif

// ---------------------------------------------------------------- partition
// Row partition of the loss / BN-backward partial sums: ~16K elements per CTA
// (per-CTA fixed costs amortised; fewer partial rows for the final sums).
int rows_part_ctas(long long rows, int c) {
    const long long elems = rows * static_cast<long long>(c);
    static const long long per_cta = [] {
        const char* e = std::getenv("PBKD_ROWS_PER_CTA");
        return e ? std::max(256LL, std::atoll(e)) : 16384LL;
    }();
    long long ctas = (elems + per_cta - 1) / per_cta;
    ctas = std::max<long long>(1, std::min<long long>(ctas, 1024));
    ctas = std::min<long long>(ctas, rows);
    const int per = rows_part_per(rows, static_cast<int>(ctas));
    return ceil_div(rows, per);
}
int rows_part_per(long long rows, int ctas) { return ceil_div(rows, ctas); }

template <class Op>
__device__ __forceinline__ const Op& op_of(const Op* ops, int nd, int& local) {
    const int t = op_index(ops, nd, static_cast<int>(blockIdx.x));
    local = static_cast<int>(blockIdx.x) - ops[t].cta_begin;
    return ops[t];
}

__device__ __forceinline__ bool is_failed(const int* f) { return f != nullptr && *f != 0; }

// element i of a batch stored as a gather: sample i / srow is sample
// rows[i / srow] of the source (srow elements per sample; a step's batch
// has < 2^31 elements, so the division is 32-bit)
__device__ __forceinline__ long long row_remap(const int* rows, long long srow, long long i) {
    const unsigned smp = static_cast<unsigned>(i) / static_cast<unsigned>(srow);
    return static_cast<long long>(__ldg(rows + smp)) * srow + (i - static_cast<long long>(smp) * srow);
}

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

// ------------------------------------------------------- depthwise tiling
// A CTA stages ni images x tr rows x tw cols x 32 channels of its input(s) in
// shared memory ([pixel][32], zero halo), then thread (channel = tid % 32,
// pixel lane = tid / 32) walks the tile's output pixels.  Warps read 32
// consecutive words (conflict-free); global loads/stores are 128-byte rows.
// Shared-memory budget per staged array (PBKD_DW_TILE_KB, default 48).
static int dw_tile_bytes() {
    static const int b = [] {
        const char* e = std::getenv("PBKD_DW_TILE_KB");
        return std::max(24, std::min(96, e ? std::atoi(e) : 48)) * 1024;
    }();
    return b;
}

// per-array budget of the two-array kernels (dw backward, dw weight grad)
static int dw_tile_bytes2() {
    static const int b = [] {
        const char* e = std::getenv("PBKD_DW_TILE2_KB");
        return std::max(12, std::min(96, e ? std::atoi(e) : 48)) * 1024;
    }();
    return b;
}

DwTile dw_tile(int n, int ho, int wo, int c, int stride, int arrays) {
    DwTile t{};
    static const int target = [] {  // output pixels per CTA (PBKD_DW_TARGET)
        const char* e = std::getenv("PBKD_DW_TARGET");
        return e ? std::max(32, std::atoi(e)) : 256;
    }();
    if (ho * wo >= target) {
        t.ni = 1;
        t.th = std::max(1, std::min(ho, target / wo));
    } else {
        t.th = ho;
        t.ni = std::max(1, std::min(n, target / (ho * wo)));
    }
    auto fp = [&](const DwTile& q) {
        return static_cast<long long>(q.ni) * ((q.th - 1) * stride + 3) * ((wo - 1) * stride + 3) * kDwC * 4;
    };
    while (fp(t) > (arrays >= 2 ? dw_tile_bytes2() : dw_tile_bytes()) && (t.ni > 1 || t.th > 1)) {
        if (t.ni > 1) t.ni = (t.ni + 1) / 2;
        else t.th = (t.th + 1) / 2;
    }
    t.tr = (t.th - 1) * stride + 3;
    t.tw = (wo - 1) * stride + 3;
    t.tiles_y = ceil_div(ho, t.th);
    t.tiles = ceil_div(n, t.ni) * t.tiles_y;
    t.cslices = ceil_div(c, kDwC);
    // x segments per output row so that the 16 packed row workers all have
    // work on tiles with few rows (wide images)
    t.xsh = 0;
    while ((t.ni * t.th << t.xsh) < 16 && (2 << t.xsh) <= wo) ++t.xsh;
    return t;
}
static size_t dw_smem(const DwTile& t) { return static_cast<size_t>(t.ni) * t.tr * t.tw * kDwC * sizeof(float); }

// Tensor maps of the staged tiles (TMA path) are built here, so the tensor
// pointers must be final before finalize.
void dw_fwd_finalize(DwFwdOp& o) {
    o.tile = dw_tile(o.n, o.ho, o.wo, o.c, o.stride, 1);
    const DwTile& t = o.tile;
    const int nsrc = o.rows ? o.nsrc : o.n;  // gather: single-image boxes over all source images
    o.tma = encode_nhwc_box(&o.map_x, o.x, nsrc, o.h, o.wd, o.c, kDwC, t.tw, t.tr, o.rows ? 1 : t.ni) ? 1 : 0;
}
void dw_bwd_finalize(DwBwdOp& o) {
    o.tile = dw_tile(o.n, o.h, o.wd, o.c, 1, 2);
    o.ctas = o.tile.tiles;
    o.rows_per = 0;
    const DwTile& t = o.tile;
    o.tma = encode_nhwc_box(&o.map_g, o.gy, o.n, o.h, o.wd, o.c, kDwC, t.tw, t.tr, t.ni) &&
                    encode_nhwc_box(&o.map_x, o.xp, o.n, o.h, o.wd, o.c, kDwC, t.tw, t.tr, t.ni)
                ? 1
                : 0;
}
void dw_gk_finalize(DwGkOp& o) {
    o.tile = dw_tile(o.n, o.ho, o.wo, o.c, o.stride, 2);
    o.ctas = o.tile.tiles;
    o.rows_per = 0;
    const DwTile& t = o.tile;
    const int nsrc = o.rows ? o.nsrc : o.n;
    o.tma = encode_nhwc_box(&o.map_x, o.x, nsrc, o.h, o.wd, o.c, kDwC, t.tw, t.tr, o.rows ? 1 : t.ni) &&
                    encode_nhwc_box(&o.map_g, o.gy, o.n, o.ho, o.wo, o.c, kDwC, o.wo, t.th, t.ni)
                ? 1
                : 0;
}
int ctas_dw_fwd(const DwFwdOp& o) { return o.tile.tiles * o.tile.cslices; }
int ctas_dw_bwd(const DwBwdOp& o) { return o.tile.tiles * o.tile.cslices; }
int ctas_dw_gk(const DwGkOp& o) { return o.tile.tiles * o.tile.cslices; }

// Stage a [ni][tr][tw][32] tile of an NHWC tensor (n, h, w, c), origin
// (n0, iy0, ix0, c0) with cp.async (all loads in flight at once; zero fill
// for out-of-range pixels / channels, the reference's padding).  16-byte
// copies when the 32-channel slice is whole and aligned, else 4-byte.
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, int bytes) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async4(uint32_t dst, const void* src, int bytes) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(dst), "l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
}

// Staged rows: R = i*tr + rr (image i of the tile, input row rr); a warp
// takes whole rows, lanes walk the row's 16-byte chunks (col*8 + q), so the
// only index math per chunk is a shift and a mask.
__device__ __forceinline__ void dw_stage(float* dst, const float* __restrict__ src, const DwTile& t, int n, int h,
                                         int w, int c, int n0, int iy0, int ix0, int c0, const int* gather = nullptr) {
    const uint32_t sd = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int rows = t.ni * t.tr;
    const bool vec = (c % 4 == 0) && (c0 + kDwC <= c);
    for (int R = warp; R < rows; R += kThreads / 32) {
        const int i = R / t.tr, rr = R - i * t.tr;
        const int nn = n0 + i, iy = iy0 + rr;
        const bool row_in = nn < n && iy >= 0 && iy < h;
        const long long img = gather != nullptr && nn < n ? __ldg(gather + nn) : nn;
        const float* rowp = src + (img * h + iy) * w * c;
        const uint32_t drow = sd + R * t.tw * kDwC * 4;
        if (vec) {
            for (int it = lane; it < t.tw * 8; it += 32) {
                const int col = it >> 3, q = it & 7, ix = ix0 + col;
                const bool in = row_in && ix >= 0 && ix < w;
                cp_async16(drow + it * 16, in ? rowp + static_cast<long long>(ix) * c + c0 + q * 4 : src, in ? 16 : 0);
            }
        } else {
            const bool cin = c0 + lane < c;
            for (int col = 0; col < t.tw; ++col) {
                const int ix = ix0 + col;
                const bool in = row_in && cin && ix >= 0 && ix < w;
                cp_async4(drow + (col * kDwC + lane) * 4, in ? rowp + static_cast<long long>(ix) * c + c0 + lane : src,
                          in ? 4 : 0);
            }
        }
    }
    cp_async_wait_all();
}

// In-place prologue f on the staged in-range pixels (padding stays 0); the
// caller synchronises before and after.  Warp = staged row, lane = channel.
// Rows are walked without divisions (tile row counts are small).
template <class F>
__device__ __forceinline__ void dw_map(float* buf, const DwTile& t, int n, int h, int w, int n0, int iy0, int ix0,
                                       F f) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    int i = 0, rr = warp;
    while (rr >= t.tr) rr -= t.tr, ++i;
    const int cb = max(0, -ix0), ce = min(t.tw, w - ix0);
    for (; i < t.ni;) {
        const int iy = iy0 + rr;
        if (n0 + i < n && iy >= 0 && iy < h) {
            float* row = buf + (i * t.tr + rr) * t.tw * kDwC + lane;
            for (int col = cb; col < ce; ++col) row[col * kDwC] = f(row[col * kDwC], lane);
        }
        rr += kThreads / 32;
        while (rr >= t.tr) rr -= t.tr, ++i;
    }
}

// Grouped-launch descriptor copied once into shared memory (16-byte words):
// one global-load latency per CTA, then every field read is a shared-memory
// broadcast.  Thread 0 also initialises the CTA's staging barrier.
template <class Op>
__device__ __forceinline__ int op_to_shared(const Op* __restrict__ ops, int nd, Op* sh, uint64_t* bar, int& local) {
    static_assert(sizeof(Op) % 16 == 0, "descriptor copied in 16-byte words");
    const int t = op_index(ops, nd, static_cast<int>(blockIdx.x));
    const uint4* src = reinterpret_cast<const uint4*>(ops + t);
    uint4* dst = reinterpret_cast<uint4*>(sh);
    for (int i = threadIdx.x; i < static_cast<int>(sizeof(Op) / 16); i += blockDim.x) dst[i] = __ldg(src + i);
    if (threadIdx.x == 0) {
        tc::mbar_init(bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    local = static_cast<int>(blockIdx.x) - sh->cta_begin;
    return t;
}

// Depthwise forward of one tile staged by cp.async (channel counts TMA cannot
// address): warp = output row, lane = channel.  Called by the whole CTA.
__device__ __forceinline__ void dw_fwd_plain(const DwFwdOp& o, const DwPos& q, float* xs) {
    const DwTile t = o.tile;
    const int n = o.n, h = o.h, w = o.wd, C = o.c, ho = o.ho, wo = o.wo, s = o.stride, pad = o.pad, pro = o.pro;
    const int iy0 = q.y0 * s - pad;
    const int ch = threadIdx.x & 31, warp = threadIdx.x >> 5, c = q.c0 + ch;
    const bool cok = c < C;
    float wk[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) wk[k] = cok ? o.w[k * C + c] : 0.0f;
    float* const yh = o.y_hi;
    float* const yl = o.y_lo;
    float* const yf = o.y;
    {
        float pa = 0, pb = 0, pc = 0, pd = 0;
        if (pro != 0 && cok) {
            pa = o.pa[c], pb = o.pb[c];
            if (pro == 1) pc = o.pc[c], pd = o.pd[c];
        }
        dw_stage(xs, o.x, t, n, h, w, C, q.n0, iy0, -pad, q.c0, o.rows);
        __syncthreads();
        if (pro == 1) {
            dw_map(xs, t, n, h, w, q.n0, iy0, -pad, [&](float v, int) { return relu(bn_train_apply(v, pa, pb, pc, pd)); });
            __syncthreads();
        } else if (pro == 2) {
            dw_map(xs, t, n, h, w, q.n0, iy0, -pad, [&](float v, int) { return relu(bn_infer_apply(v, pa, pb)); });
            __syncthreads();
        }
    }
    const int rs = t.tw * kDwC;
    if (!cok) return;
    int i = 0, oy = warp;
    while (oy >= t.th) oy -= t.th, ++i;
    for (; i < t.ni;) {
        const int nn = q.n0 + i, yy = q.y0 + oy;
        if (nn < n && yy < ho) {
            const float* base = xs + ((i * t.tr + oy * s) * t.tw) * kDwC + ch;
            long long off = ((static_cast<long long>(nn) * ho + yy) * wo) * C + c;
            float win[3][3];  // stride 1: 3x3 register window slid along x
            if (s == 1) {
#pragma unroll
                for (int r = 0; r < 3; ++r) win[r][1] = base[r * rs], win[r][2] = base[r * rs + kDwC];
            }
#pragma unroll 2
            for (int ox = 0; ox < wo; ++ox, off += C) {
                if (s == 1) {
#pragma unroll
                    for (int r = 0; r < 3; ++r)
                        win[r][0] = win[r][1], win[r][1] = win[r][2], win[r][2] = base[r * rs + (ox + 2) * kDwC];
                } else {
                    const float* b = base + ox * s * kDwC;
#pragma unroll
                    for (int r = 0; r < 3; ++r)
#pragma unroll
                        for (int cc = 0; cc < 3; ++cc) win[r][cc] = b[r * rs + cc * kDwC];
                }
                float acc = 0.0f;  // 9-term serial sum in (ky, kx) order (ops.hpp:131-140)
#pragma unroll
                for (int ky = 0; ky < 3; ++ky)
#pragma unroll
                    for (int kx = 0; kx < 3; ++kx) acc = add(acc, mul(win[ky][kx], wk[ky * 3 + kx]));
                if (yh) {  // tf32 planes for the pointwise GEMMs (3xTF32 operand split)
                    const float hv = __uint_as_float(tc_split_hi(acc));
                    yh[off] = hv;
                    yl[off] = __uint_as_float(tc_split_lo(acc, hv));
                    if (o.y_both) yf[off] = acc;
                } else {
                    yf[off] = acc;
                }
            }
        }
        oy += kThreads / 32;
        while (oy >= t.th) oy -= t.th, ++i;
    }
}


// ---------------------------------------------------------- depthwise fwd
// The x tile arrives by one 4-D TMA box (zero-filled halo / channel tail) or,
// for channel counts TMA cannot address, by cp.async.  Warp = output row
// (image i, row oy) of the tile, lane = channel; stride 1 slides a 3x3
// register window along x (3 shared loads per output).
__global__ void __launch_bounds__(kThreads) dw_fwd_kernel(const DwFwdOp* __restrict__ ops, int nd) {
    pdl_trigger();
    cta_mark(0);
    extern __shared__ __align__(128) float xs[];
    __shared__ DwFwdOp osh;
    __shared__ uint64_t bar;
    int local;
    const int oi = op_to_shared(ops, nd, &osh, &bar, local);
    pdl_wait();  // descriptor copy above overlaps the predecessor's tail
    cta_mark(1);
    const DwFwdOp& o = osh;
    if (is_failed(o.failed)) return;
    const DwTile t = o.tile;
    const DwPos q = dw_pos(t, local);
    const int n = o.n, h = o.h, w = o.wd, C = o.c, ho = o.ho, wo = o.wo, s = o.stride, pad = o.pad, pro = o.pro;
    const int iy0 = q.y0 * s - pad;
    const bool tma = o.tma != 0;
    if (tma && threadIdx.x < 32) {
        if (o.rows == nullptr) {
            if (threadIdx.x == 0) {
                tc::mbar_arrive_expect_tx(&bar, static_cast<uint32_t>(t.ni * t.tr * t.tw * kDwC * 4));
                tc::tma_load_4d(xs, &ops[oi].map_x, &bar, q.c0, -pad, iy0, q.n0);
            }
        } else {  // gather: one single-image box per batch image, lanes in parallel
            const int cnt = min(t.ni, n - q.n0), img_f = t.tr * t.tw * kDwC;
            if (threadIdx.x == 0) tc::mbar_arrive_expect_tx(&bar, static_cast<uint32_t>(cnt * img_f * 4));
            __syncwarp();
            for (int i = threadIdx.x; i < cnt; i += 32)
                tc::tma_load_4d(xs + i * img_f, &ops[oi].map_x, &bar, q.c0, -pad, iy0, __ldg(o.rows + q.n0 + i));
        }
    }
    if (tma) {
        dw_fwd_tile(o, q, xs, [&] { tc::mbar_wait(&bar, 0); cta_mark(2); });
    } else {
        dw_fwd_plain(o, q, xs);
    }
    cta_mark(3);
}

// Persistent variant: 2 CTAs per SM, each walks tiles b, b + G, ... with two
// staging buffers, so tile j+1's TMA box (and its descriptor copy) is in
// flight while tile j is mapped and computed.  Same per-tile code as
// dw_fwd_kernel: identical bits.
constexpr int kDwPersistPerSm = 2;
constexpr int kDwMaxOps = 64;

// warp 0: stage tile q of op o (TMA path) into xs, completion on bar
__device__ __forceinline__ void dw_fwd_issue(const DwFwdOp& o, const CUtensorMap* map, const DwPos& q, float* xs,
                                             uint64_t* bar) {
    const DwTile& t = o.tile;
    const int iy0 = q.y0 * o.stride - o.pad;
    if (o.rows == nullptr) {
        if (threadIdx.x == 0) {
            tc::mbar_arrive_expect_tx(bar, static_cast<uint32_t>(t.ni * t.tr * t.tw * kDwC * 4));
            tc::tma_load_4d(xs, map, bar, q.c0, -o.pad, iy0, q.n0);
        }
    } else {
        const int cnt = min(t.ni, o.n - q.n0), img_f = t.tr * t.tw * kDwC;
        if (threadIdx.x == 0) tc::mbar_arrive_expect_tx(bar, static_cast<uint32_t>(cnt * img_f * 4));
        __syncwarp();
        for (int i = threadIdx.x; i < cnt; i += 32) tc::tma_load_4d(xs + i * img_f, map, bar, q.c0, -o.pad, iy0, __ldg(o.rows + q.n0 + i));
    }
}

__global__ void __launch_bounds__(kThreads, kDwPersistPerSm) dw_fwd_persist_kernel(const DwFwdOp* __restrict__ ops,
                                                                                 int nd, int total, int buf_floats) {
    pdl_trigger();
    extern __shared__ __align__(128) float xbuf[];
    __shared__ __align__(16) DwFwdOp osh[2];
    __shared__ uint64_t bar[2];
    __shared__ int begins[kDwMaxOps];
    __shared__ int opi[2];
    const int G = static_cast<int>(gridDim.x), b = static_cast<int>(blockIdx.x);
    for (int i = threadIdx.x; i < nd; i += blockDim.x) begins[i] = ops[i].cta_begin;
    if (threadIdx.x == 0) {
        tc::mbar_init(&bar[0], 1);
        tc::mbar_init(&bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const int nt = b < total ? (total - 1 - b) / G + 1 : 0;
    // descriptor of tile j into slot j & 1 (all threads); returns the tile's local index
    auto load_desc = [&](int j) {
        const int t = b + j * G;
        int lo = 0, hi = nd - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (begins[mid] <= t) lo = mid;
            else hi = mid - 1;
        }
        const uint4* src = reinterpret_cast<const uint4*>(ops + lo);
        uint4* dst = reinterpret_cast<uint4*>(&osh[j & 1]);
        for (int i = threadIdx.x; i < static_cast<int>(sizeof(DwFwdOp) / 16); i += blockDim.x) dst[i] = __ldg(src + i);
        if (threadIdx.x == 0) opi[j & 1] = lo;
        return t - begins[lo];
    };
    auto stage = [&](int j, int local) {  // warp 0, after the descriptor is visible
        const DwFwdOp& o = osh[j & 1];
        if (threadIdx.x < 32 && o.tma && !is_failed(o.failed)) {
            tc::fence_async_smem();  // generic writes of this buffer's previous tile precede the TMA
            dw_fwd_issue(o, &ops[opi[j & 1]].map_x, dw_pos(o.tile, local), xbuf + (j & 1) * buf_floats, &bar[j & 1]);
        }
    };
    if (nt == 0) return;
    int local = load_desc(0);
    __syncthreads();
    pdl_wait();  // descriptors above overlap the predecessor's tail
    stage(0, local);
    uint32_t phase[2] = {0u, 0u};
    for (int j = 0; j < nt; ++j) {
        const int slot = j & 1;
        int next = 0;
        if (j + 1 < nt) next = load_desc(j + 1);
        __syncthreads();
        if (j + 1 < nt) stage(j + 1, next);
        const DwFwdOp& o = osh[slot];
        if (!is_failed(o.failed)) {
            const DwPos q = dw_pos(o.tile, local);
            float* xs = xbuf + slot * buf_floats;
            if (o.tma) {
                const uint32_t ph = phase[slot];
                dw_fwd_tile(o, q, xs, [&] { tc::mbar_wait(&bar[slot], ph); });
                phase[slot] ^= 1u;
            } else {
                dw_fwd_plain(o, q, xs);
            }
        }
        __syncthreads();  // buffer and descriptor slot free for tile j + 2
        local = next;
    }
}

void launch_dw_fwd(const DwFwdOp* d, int nd, int ctas, cudaStream_t st) {
    // PBKD_DW_PERSIST=1: the persistent double-buffered variant -- measured
    // 6% slower per launch (2 CTAs / 16 warps per SM hide the window's FFMA2
    // and shared-memory latencies worse than 3 one-tile CTAs), so off
    static const bool persist = [] {
        const char* e = std::getenv("PBKD_DW_PERSIST");
        return e && e[0] == '1';
    }();
    if (persist && nd <= kDwMaxOps) {
        static bool pattr = false;
        const int bytes = 2 * dw_tile_bytes();
        if (!pattr) {
            PBKD_CUDA(cudaFuncSetAttribute(dw_fwd_persist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
            pattr = true;
        }
        static int sms = [] {
            int dev = 0, v = 0;
            PBKD_CUDA(cudaGetDevice(&dev));
            PBKD_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev));
            return std::max(1, v);
        }();
        const int grid = std::max(1, std::min(ctas, kDwPersistPerSm * sms));
        traced("dw_fwd", grid, st, [&] {
            launch_k(dw_fwd_persist_kernel, dim3(grid), dim3(kThreads), static_cast<size_t>(bytes), st, d, nd, ctas,
                     dw_tile_bytes() / 4);
        });
        PBKD_LAUNCH_CHECK();
        return;
    }
    static bool attr = false;
    if (!attr) {  // 48 KB dynamic + the static descriptor copy exceed the default
        PBKD_CUDA(cudaFuncSetAttribute(dw_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, dw_tile_bytes()));
        attr = true;
    }
    traced("dw_fwd", ctas, st, [&] { launch_k(dw_fwd_kernel, dim3(ctas), dim3(kThreads), dw_tile_bytes(), st, d, nd); });
    PBKD_LAUNCH_CHECK();
}

// CTA-level fixed-order sum of per-thread values over the row workers.
// Scalar layout: thread (row worker = warp, channel = lane) holds v[k].
// Packed layout: thread (row worker = 2*warp + lane/16, channels 2p, 2p+1
// with p = lane%16) holds v2[k].  Thread ch < 32 gets out[k] for channel ch.
template <int NV>
__device__ __forceinline__ void dw_lane_sum(float* red, const float* v, float* out) {
    const int ch = threadIdx.x % kDwC, lane = threadIdx.x / kDwC;
#pragma unroll
    for (int k = 0; k < NV; ++k) red[(lane * NV + k) * kDwC + ch] = v[k];
    __syncthreads();
    if (lane == 0) {
#pragma unroll
        for (int k = 0; k < NV; ++k) {
            float acc = 0.0f;
            for (int l = 0; l < kDwLanes; ++l) acc += red[(l * NV + k) * kDwC + ch];
            out[k] = acc;
        }
    }
}
// ------------------------------------------- depthwise bwd (unit > 0, s=1)
// gy (dw output gradient) and the previous unit's activation relu(bn(p)) are
// staged with halos; per pixel: the input gradient gathered in ascending
// (oy, ox) order with zero terms skipped (ops.hpp:156-174), the weight-
// gradient terms, the previous ReLU mask and batch-norm partial sums.
__global__ void __launch_bounds__(kThreads) dw_bwd_kernel(const DwBwdOp* __restrict__ ops, int nd) {
    pdl_trigger();
    cta_mark(0);
    extern __shared__ __align__(128) float sm[];
    __shared__ DwBwdOp osh;
    __shared__ uint64_t bar;
    int local;
    const int oi = op_to_shared(ops, nd, &osh, &bar, local);
    pdl_wait();  // descriptor copy above overlaps the predecessor's tail
    cta_mark(1);
    const DwBwdOp& o = osh;
    if (is_failed(o.failed)) return;
    const DwTile t = o.tile;
    const DwPos q = dw_pos(t, local);
    const int n = o.n, h = o.h, w = o.wd, C = o.c;
    const int tile_elems = t.ni * t.tr * t.tw * kDwC;
    float* gs = sm;
    float* xs = sm + tile_elems;
    const bool tma = o.tma != 0;
    if (tma && threadIdx.x == 0) {
        tc::mbar_arrive_expect_tx(&bar, static_cast<uint32_t>(2 * tile_elems * 4));
        tc::tma_load_4d(gs, &ops[oi].map_g, &bar, q.c0, -1, q.y0 - 1, q.n0);
        tc::tma_load_4d(xs, &ops[oi].map_x, &bar, q.c0, -1, q.y0 - 1, q.n0);
    }
    const int ch = threadIdx.x % kDwC, c = q.c0 + ch;
    const bool cok = c < C;
    float mean = 0, inv = 0, gam = 0, bet = 0;
    if (cok) mean = o.mean[c], inv = o.inv[c], gam = o.gamma[c], bet = o.beta[c];
    float wk[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) wk[k] = cok ? o.w[k * C + c] : 0.0f;
    const float* const xp = o.xp;
    float* const gyprev = o.gyprev;
    // TMA path: pass A reads the raw p centre from the staged tile, then xs
    // is mapped to relu(bn(p)) (the dw layer's input) for pass B.  Scalar
    // path: xs is mapped first and the raw centre is re-read from global.
    if (tma) {
        tc::mbar_wait(&bar, 0);
        cta_mark(2);
    } else {
        dw_stage(gs, o.gy, t, n, h, w, C, q.n0, q.y0 - 1, -1, q.c0);
        dw_stage(xs, xp, t, n, h, w, C, q.n0, q.y0 - 1, -1, q.c0);
        __syncthreads();
        dw_map(xs, t, n, h, w, q.n0, q.y0 - 1, -1, [&](float v, int) { return relu(bn_train_apply(v, mean, inv, gam, bet)); });
    }
    __syncthreads();

    if (tma) {
        dw_bwd_tile(o, q, gs, xs, [] {});
        cta_mark(3);
        return;
    }
    float acc[11];  // gk[9], sg, sgx
#pragma unroll
    for (int k = 0; k < 11; ++k) acc[k] = 0.0f;
    if (cok) {
        const int warp = threadIdx.x >> 5, rs = t.tw * kDwC;
        int i = 0, y = warp;
        while (y >= t.th) y -= t.th, ++i;
        for (; i < t.ni;) {
            const int nn = q.n0 + i, yy = q.y0 + y;
            if (nn < n && yy < h) {
                long long gi = ((static_cast<long long>(nn) * h + yy) * w) * C + c;
                // 3x3 register windows over tile rows y..y+2 (= image rows yy-1..yy+1),
                // columns x..x+2 (= image columns x-1..x+1), slid along x
                const float* g0 = gs + ((i * t.tr + y) * t.tw) * kDwC + ch;
                const float* x0 = xs + ((i * t.tr + y) * t.tw) * kDwC + ch;
                float gw[3][3], xw[3][3];
#pragma unroll
                for (int r = 0; r < 3; ++r)
#pragma unroll
                    for (int cc = 0; cc < 2; ++cc) {
                        gw[r][cc + 1] = g0[r * rs + cc * kDwC];
                        xw[r][cc + 1] = x0[r * rs + cc * kDwC];
                    }
#pragma unroll 4
                for (int x = 0; x < w; ++x, gi += C) {
#pragma unroll
                    for (int r = 0; r < 3; ++r) {
                        gw[r][0] = gw[r][1], gw[r][1] = gw[r][2], gw[r][2] = g0[r * rs + (x + 2) * kDwC];
                        xw[r][0] = xw[r][1], xw[r][1] = xw[r][2], xw[r][2] = x0[r * rs + (x + 2) * kDwC];
                    }
                    // input gradient: outputs (oy, ox) = (yy+dy, x+dx) ascending, tap
                    // (1-dy, 1-dx), zero terms skipped (ops.hpp:156-174)
                    float gx = 0.0f;
#pragma unroll
                    for (int r = 0; r < 3; ++r)
#pragma unroll
                        for (int cc = 0; cc < 3; ++cc) {
                            const float gv = gw[r][cc];
                            if (gv != 0.0f) gx = add(gx, mul(gv, wk[(2 - r) * 3 + (2 - cc)]));
                        }
                    const float gyc = gw[1][1];
                    if (gyc != 0.0f) {
#pragma unroll
                        for (int r = 0; r < 3; ++r)
#pragma unroll
                            for (int cc = 0; cc < 3; ++cc) acc[r * 3 + cc] += gyc * xw[r][cc];
                    }
                    const float xh = mul(sub(__ldg(xp + gi), mean), inv);
                    const float yv = add(mul(gam, xh), bet);
                    const float gm = yv > 0.0f ? add(0.0f, gx) : 0.0f;
                    gyprev[gi] = gm;
                    acc[9] += gm;
                    acc[10] += gm * xh;
                }
            }
            y += kThreads / 32;
            while (y >= t.th) y -= t.th, ++i;
        }
    }
    __syncthreads();  // staging buffers are reused for the reduction
    float out[11];
    dw_lane_sum<11>(sm, acc, out);
    if (threadIdx.x < kDwC && cok) {
        for (int k = 0; k < 9; ++k) o.part_gk[(static_cast<long long>(q.tile) * 9 + k) * C + c] = out[k];
        o.part_sg[static_cast<long long>(q.tile) * C + c] = out[9];
        o.part_sgx[static_cast<long long>(q.tile) * C + c] = out[10];
    }
    cta_mark(3);
}

void launch_dw_bwd(const DwBwdOp* d, int nd, int ctas, cudaStream_t st) {
    static bool attr = false;
    if (!attr) {
        PBKD_CUDA(cudaFuncSetAttribute(dw_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * dw_tile_bytes2()));
        attr = true;
    }
    traced("dw_bwd", ctas, st, [&] { launch_k(dw_bwd_kernel, dim3(ctas), dim3(kThreads), 2 * dw_tile_bytes2(), st, d, nd); });
    PBKD_LAUNCH_CHECK();
}

// ------------------------------------------- depthwise weight grad (unit 0)
// model.cpp:570 skips the input gradient of the block's first layer.  With
// TMA both the input tile (halo) and the output-gradient tile are staged.
__global__ void __launch_bounds__(kThreads) dw_gk_kernel(const DwGkOp* __restrict__ ops, int nd) {
    pdl_trigger();
    cta_mark(0);
    extern __shared__ __align__(128) float sm[];
    __shared__ DwGkOp osh;
    __shared__ uint64_t bar;
    int local;
    const int oi = op_to_shared(ops, nd, &osh, &bar, local);
    pdl_wait();  // descriptor copy above overlaps the predecessor's tail
    cta_mark(1);
    const DwGkOp& o = osh;
    if (is_failed(o.failed)) return;
    const DwTile t = o.tile;
    const DwPos q = dw_pos(t, local);
    const int n = o.n, h = o.h, w = o.wd, C = o.c, ho = o.ho, wo = o.wo, s = o.stride, pad = o.pad;
    const int tile_elems = t.ni * t.tr * t.tw * kDwC;
    float* xs = sm;
    float* gs = sm + tile_elems;  // [ni][th][wo][32] (TMA path)
    const bool tma = o.tma != 0;
    if (tma && threadIdx.x < 32) {
        if (o.rows == nullptr) {
            if (threadIdx.x == 0) {
                tc::mbar_arrive_expect_tx(&bar, static_cast<uint32_t>((tile_elems + t.ni * t.th * wo * kDwC) * 4));
                tc::tma_load_4d(xs, &ops[oi].map_x, &bar, q.c0, -pad, q.y0 * s - pad, q.n0);
                tc::tma_load_4d(gs, &ops[oi].map_g, &bar, q.c0, 0, q.y0, q.n0);
            }
        } else {  // x gathered image by image (lanes in parallel), gy as one box
            const int cnt = min(t.ni, n - q.n0), img_f = t.tr * t.tw * kDwC;
            if (threadIdx.x == 0) {
                tc::mbar_arrive_expect_tx(&bar, static_cast<uint32_t>((cnt * img_f + t.ni * t.th * wo * kDwC) * 4));
                tc::tma_load_4d(gs, &ops[oi].map_g, &bar, q.c0, 0, q.y0, q.n0);
            }
            __syncwarp();
            for (int i = threadIdx.x; i < cnt; i += 32)
                tc::tma_load_4d(xs + i * img_f, &ops[oi].map_x, &bar, q.c0, -pad, q.y0 * s - pad, __ldg(o.rows + q.n0 + i));
        }
    }
    const int ch = threadIdx.x % kDwC, c = q.c0 + ch;
    const bool cok = c < C;
    const float* const gy = o.gy;
    if (tma) {
        tc::mbar_wait(&bar, 0);
        cta_mark(2);
    } else {
        dw_stage(xs, o.x, t, n, h, w, C, q.n0, q.y0 * s - pad, -pad, q.c0, o.rows);
        __syncthreads();
    }
    if (tma) {
        dw_gk_tile(o, q, xs, gs, sm, [] {});
        cta_mark(3);
        return;
    }
    float acc[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) acc[k] = 0.0f;
    if (cok) {
        const int warp = threadIdx.x >> 5;
        int i = 0, oy = warp;
        while (oy >= t.th) oy -= t.th, ++i;
        for (; i < t.ni;) {
            const int nn = q.n0 + i, yy = q.y0 + oy;
            if (nn < n && yy < ho) {
                const float* gyr = gy + ((static_cast<long long>(nn) * ho + yy) * wo) * C + c;
                const float* gsr = gs + ((i * t.th + oy) * wo) * kDwC + ch;
                const float* base = xs + ((i * t.tr + oy * s) * t.tw) * kDwC + ch;
#pragma unroll 2
                for (int ox = 0; ox < wo; ++ox) {
                    const float gv = tma ? gsr[ox * kDwC] : __ldg(gyr + static_cast<long long>(ox) * C);
                    if (gv == 0.0f) continue;
                    const float* b = base + ox * s * kDwC;
#pragma unroll
                    for (int ky = 0; ky < 3; ++ky)
#pragma unroll
                        for (int kx = 0; kx < 3; ++kx) acc[ky * 3 + kx] += gv * b[(ky * t.tw + kx) * kDwC];
                }
            }
            oy += kThreads / 32;
            while (oy >= t.th) oy -= t.th, ++i;
        }
    }
    __syncthreads();
    float out[9];
    dw_lane_sum<9>(sm, acc, out);
    if (threadIdx.x < kDwC && cok)
        for (int k = 0; k < 9; ++k) o.part_gk[(static_cast<long long>(q.tile) * 9 + k) * C + c] = out[k];
    cta_mark(3);
}

void launch_dw_gk(const DwGkOp* d, int nd, int ctas, cudaStream_t st) {
    static bool attr = false;
    if (!attr) {
        PBKD_CUDA(cudaFuncSetAttribute(dw_gk_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * dw_tile_bytes2()));
        attr = true;
    }
    traced("dw_gk", ctas, st, [&] { launch_k(dw_gk_kernel, dim3(ctas), dim3(kThreads), 2 * dw_tile_bytes2(), st, d, nd); });
    PBKD_LAUNCH_CHECK();
}

static size_t red_smem(int) { return static_cast<size_t>(kThreads) * 4 * sizeof(float); }

// ------------------------------------------------------------ BN statistics
// Column sums of [parts][c] partials: a CTA owns 32 channels, 8 lanes stride
// over the parts, lanes combine in fixed order (deterministic, latency-hidden).
constexpr int kColLanes = kThreads / 32;
int ctas_cols(int c) { return ceil_div(c, 32); }

// Column sums of two [parts][c] partial arrays at once (a CTA owns 32
// columns; its 8 warps stride over the parts with 8 loads of each array in
// flight per round, then combine in fixed order): one dependent round trip
// per 64 parts instead of one per 32 parts and array.
__device__ __forceinline__ void col_sum2(const float* __restrict__ pa, const float* __restrict__ pb, int parts, int c,
                                         int ch, float (*red)[2][32], float& sa, float& sb) {
    const int lane = threadIdx.x / 32, col = threadIdx.x % 32;
    float a[4] = {0.0f, 0.0f, 0.0f, 0.0f}, b[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    if (ch < c) {
        int p = lane;
        for (; p + 7 * kColLanes < parts; p += 8 * kColLanes) {
            float va[8], vb[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const long long off = static_cast<long long>(p + u * kColLanes) * c + ch;
                va[u] = __ldg(pa + off);
                vb[u] = __ldg(pb + off);
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) a[u & 3] += va[u], b[u & 3] += vb[u];
        }
        for (; p < parts; p += kColLanes) {
            const long long off = static_cast<long long>(p) * c + ch;
            a[0] += __ldg(pa + off);
            b[0] += __ldg(pb + off);
        }
    }
    red[lane][0][col] = (a[0] + a[1]) + (a[2] + a[3]);
    red[lane][1][col] = (b[0] + b[1]) + (b[2] + b[3]);
    __syncthreads();
    sa = sb = 0.0f;
    for (int l = 0; l < kColLanes; ++l) sa += red[l][0][col], sb += red[l][1][col];
    __syncthreads();
}

__global__ void __launch_bounds__(kThreads) bn_stat_kernel(const BnStatOp* __restrict__ ops, int nd) {
    pdl_trigger();
    __shared__ float red[kColLanes][2][32];
    int local;
    const BnStatOp o = op_of(ops, nd, local);  // copy: no reloads after stores
    pdl_wait();  // the static descriptor read above overlaps the predecessor's tail
    if (is_failed(o.failed)) return;
    const int ch = local * 32 + threadIdx.x % 32;
    float sum, sq;
    col_sum2(o.part_sum, o.part_sq, o.tiles, o.c, ch, red, sum, sq);
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

// --------------------------------------------------------- fixed-order sums
// out[i] = sum over parts of part[p][i]: a CTA owns 32 columns; its 8 warps
// stride over the parts (4 independent accumulators each), then the 8 warp
// sums combine in fixed order -- the order depends only on `parts`, and the
// dependent-load chain is parts/32 deep instead of parts.
int ctas_reduce(const ReduceOp& o) { return std::max(1, ceil_div(o.width, 32)); }

__global__ void __launch_bounds__(kThreads) reduce_kernel(const ReduceOp* __restrict__ ops, int nd) {
    pdl_trigger();
    __shared__ float red[kThreads / 32][32];
    int local;
    const ReduceOp o = op_of(ops, nd, local);  // copy: no reloads after stores
    pdl_wait();  // the static descriptor read above overlaps the predecessor's tail
    if (is_failed(o.failed)) return;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const int col = local * 32 + lane;
    float a0 = 0.0f, a1 = 0.0f, a2 = 0.0f, a3 = 0.0f;
    if (col < o.width) {
        const float* __restrict__ p = o.part + col;
        const long long wd = o.width;
        int q = w;
        for (; q + 24 < o.parts; q += 32) {
            a0 += __ldg(p + q * wd);
            a1 += __ldg(p + (q + 8) * wd);
            a2 += __ldg(p + (q + 16) * wd);
            a3 += __ldg(p + (q + 24) * wd);
        }
        for (; q < o.parts; q += 8) a0 += __ldg(p + q * wd);
    }
    red[w][lane] = (a0 + a1) + (a2 + a3);
    __syncthreads();
    if (w == 0 && col < o.width) {
        float sacc = 0.0f;
#pragma unroll
        for (int i = 0; i < kThreads / 32; ++i) sacc += red[i][lane];
        o.out[col] = sacc;
        if (o.out2) o.out2[col] = sacc;
    }
}

void launch_reduce(const ReduceOp* d, int nd, int ctas, cudaStream_t st) {
    launch_k(reduce_kernel, dim3(ctas), dim3(kThreads), 0, st, d, nd);
    PBKD_LAUNCH_CHECK();
}

void launch_bn_stat(const BnStatOp* d, int nd, int ctas, cudaStream_t st) {
    launch_k(bn_stat_kernel, dim3(ctas), dim3(kThreads), 0, st, d, nd);
    PBKD_LAUNCH_CHECK();
}

// ------------------------------------------------------------- loss + BN
// One channel pass of the loss kernel: thread (rr, gg) owns V channels of
// [cb, cb+cw) and rows rr, rr+RP, ... of the CTA's row range.
__device__ __forceinline__ void loss_pass(const LossOp& o, int local, int cb, int cw, int V, float* red, float& lsum) {
    Geo g;
    g.V = V, g.G = cw / V, g.RP = max(1, kThreads / g.G);
    const int rr = threadIdx.x / g.G, gg = threadIdx.x % g.G;
    const bool lane_ok = rr < g.RP;
    const long long r0 = static_cast<long long>(local) * o.rows_per;
    const long long r1 = min(static_cast<long long>(o.rows), r0 + o.rows_per);
    const int c0 = cb + gg * g.V;
    float sg[4] = {0, 0, 0, 0}, sgx[4] = {0, 0, 0, 0};
    if (lane_ok) {
        float mean[4], inv[4], gam[4], bet[4];
        load_v(o.mean + c0, g.V, mean);
        load_v(o.inv + c0, g.V, inv);
        load_v(o.gamma + c0, g.V, gam);
        load_v(o.beta + c0, g.V, bet);
        auto body = [&](long long r, const float* tp) {
            float pv[4], tv[4];
            load_v(o.p + r * o.c + c0, g.V, pv);
            load_v(tp, g.V, tv);
            for (int q = 0; q < g.V; ++q) {
                const float xh = mul(sub(pv[q], mean[q]), inv[q]);
                const float y = add(mul(gam[q], xh), bet[q]);
                const float d = sub(relu(y), tv[q]);
                lsum += d * d;
                const float gy = y > 0.0f ? add(0.0f, mul(o.kmse, d)) : 0.0f;
                sg[q] += gy;
                sgx[q] += gy * xh;
            }
        };
        if (o.trows == nullptr) {
#pragma unroll 4
            for (long long r = r0 + rr; r < r1; r += g.RP) body(r, o.t + r * o.c + c0);
        } else {  // targets gathered through the epoch order
#pragma unroll 4
            for (long long r = r0 + rr; r < r1; r += g.RP) body(r, o.t + row_remap(o.trows, o.srow, r * o.c + c0));
        }
    }
    cta_reduce_rows(red, sg, g, rr, gg, lane_ok, cw, o.part_sg + static_cast<long long>(local) * o.c + cb);
    cta_reduce_rows(red, sgx, g, rr, gg, lane_ok, cw, o.part_sgx + static_cast<long long>(local) * o.c + cb);
}

__global__ void __launch_bounds__(kThreads) loss_kernel(const LossOp* __restrict__ ops, int nd) {
    pdl_trigger();
    extern __shared__ float red[];
    __shared__ float lred[kThreads];
    int local;
    const LossOp o = op_of(ops, nd, local);  // copy: no reloads after stores
    pdl_wait();  // the static descriptor read above overlaps the predecessor's tail
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
        auto body = [&](long long r, const float* tp) {
            float pv[4], tv[4];
            load_v(o.p + r * o.c + c0, g.V, pv);
            load_v(tp, g.V, tv);
            for (int q = 0; q < g.V; ++q) {
                const float xh = mul(sub(pv[q], mean[q]), inv[q]);
                const float y = add(mul(gam[q], xh), bet[q]);
                const float d = sub(relu(y), tv[q]);
                lsum += d * d;
                const float gy = y > 0.0f ? add(0.0f, mul(o.kmse, d)) : 0.0f;
                sg[q] += gy;
                sgx[q] += gy * xh;
            }
        };
        if (o.trows == nullptr) {
#pragma unroll 4
            for (long long r = r0 + rr; r < r1; r += g.RP) body(r, o.t + r * o.c + c0);
        } else {  // targets gathered through the epoch order
#pragma unroll 4
            for (long long r = r0 + rr; r < r1; r += g.RP) body(r, o.t + row_remap(o.trows, o.srow, r * o.c + c0));
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

__global__ void __launch_bounds__(kThreads) loss_wide_kernel(const LossOp* __restrict__ ops, int nd) {
    pdl_trigger();
    extern __shared__ float red[];
    __shared__ float lred[kThreads];
    int local;
    const LossOp o = op_of(ops, nd, local);  // copy: no reloads after stores
    pdl_wait();  // the static descriptor read above overlaps the predecessor's tail
    if (is_failed(o.failed)) return;
    const int V = (o.c % 4 == 0) ? 4 : 1;
    float lsum = 0.0f;
    // channel passes of kThreads*V (the 2048-channel ResNet-50 stage); same
    // per-thread order as loss_kernel when there is one pass
    for (int cb = 0; cb < o.c; cb += kThreads * V) loss_pass(o, local, cb, min(kThreads * V, o.c - cb), V, red, lsum);
    lred[threadIdx.x] = lsum;
    __syncthreads();
    if (threadIdx.x == 0) {
        float s = 0.0f;
        for (int i = 0; i < kThreads; ++i) s += lred[i];
        o.part_loss[local] = s;
    }
}

void launch_loss(const LossOp* d, int nd, int ctas, cudaStream_t st) {
    launch_k(loss_kernel, dim3(ctas), dim3(kThreads), red_smem(0), st, d, nd);
    PBKD_LAUNCH_CHECK();
}

void launch_loss_wide(const LossOp* d, int nd, int ctas, cudaStream_t st) {
    launch_k(loss_wide_kernel, dim3(ctas), dim3(kThreads), red_smem(0), st, d, nd);
    PBKD_LAUNCH_CHECK();
}

__global__ void __launch_bounds__(kThreads) bn_bwd_fin_kernel(const BnBwdFinOp* __restrict__ ops, int nd) {
    pdl_trigger();
    __shared__ float red[kColLanes][2][32];
    int local;
    const BnBwdFinOp o = op_of(ops, nd, local);  // copy: no reloads after stores
    pdl_wait();  // the static descriptor read above overlaps the predecessor's tail
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
    float a, b;
    col_sum2(o.part_sg, o.part_sgx, o.ctas, o.c, ch, red, a, b);
    if (threadIdx.x >= 32 || ch >= o.c) return;
    o.sg[ch] = a;
    o.sgx[ch] = b;
    o.gbeta[ch] = a;
    o.ggamma[ch] = b;
}

void launch_bn_bwd_fin(const BnBwdFinOp* d, int nd, int ctas, cudaStream_t st) {
    launch_k(bn_bwd_fin_kernel, dim3(ctas), dim3(kThreads), 0, st, d, nd);
    PBKD_LAUNCH_CHECK();
}

// Each thread owns 4 consecutive elements (one channel quad when c % 4 == 0,
// per-channel parameters as float4); every load is issued before any store.
struct BnBwdPar {
    float mean, inv, gamma, beta, sg, sgx;
};
__device__ __forceinline__ float bn_bwd_one(const BnBwdApplyOp& o, const BnBwdPar& q, float p, float tg) {
    const float xh = mul(sub(p, q.mean), q.inv);
    float gy;
    if (o.t) {
        const float y = add(mul(q.gamma, xh), q.beta);
        const float d = sub(relu(y), tg);
        gy = y > 0.0f ? add(0.0f, mul(o.kmse, d)) : 0.0f;
    } else {
        gy = tg;
    }
    const float kk = mul(q.gamma, q.inv);
    const float inner = sub(sub(gy, mul(o.inv_m, q.sg)), mul(mul(xh, o.inv_m), q.sgx));
    return add(0.0f, mul(kk, inner));
}
__device__ __forceinline__ BnBwdPar bn_bwd_par(const BnBwdApplyOp& o, int ch) {
    return {o.mean[ch], o.inv[ch], o.gamma[ch], o.beta[ch], o.sg[ch], o.sgx[ch]};
}

__device__ __forceinline__ float4 bn_bwd_quad(const BnBwdApplyOp& o, int ch, float4 p, float4 g) {
    const float4 mn = __ldg(reinterpret_cast<const float4*>(o.mean + ch));
    const float4 iv = __ldg(reinterpret_cast<const float4*>(o.inv + ch));
    const float4 gm = __ldg(reinterpret_cast<const float4*>(o.gamma + ch));
    const float4 bt = __ldg(reinterpret_cast<const float4*>(o.beta + ch));
    const float4 s1 = __ldg(reinterpret_cast<const float4*>(o.sg + ch));
    const float4 s2 = __ldg(reinterpret_cast<const float4*>(o.sgx + ch));
    float4 r;
    r.x = bn_bwd_one(o, {mn.x, iv.x, gm.x, bt.x, s1.x, s2.x}, p.x, g.x);
    r.y = bn_bwd_one(o, {mn.y, iv.y, gm.y, bt.y, s1.y, s2.y}, p.y, g.y);
    r.z = bn_bwd_one(o, {mn.z, iv.z, gm.z, bt.z, s1.z, s2.z}, p.z, g.z);
    r.w = bn_bwd_one(o, {mn.w, iv.w, gm.w, bt.w, s1.w, s2.w}, p.w, g.w);
    return r;
}
__device__ __forceinline__ void split_store4(float* hi, float* lo, long long i, float4 r) {
    float4 h, l;
    h.x = __uint_as_float(tc_split_hi(r.x)), l.x = __uint_as_float(tc_split_lo(r.x, h.x));
    h.y = __uint_as_float(tc_split_hi(r.y)), l.y = __uint_as_float(tc_split_lo(r.y, h.y));
    h.z = __uint_as_float(tc_split_hi(r.z)), l.z = __uint_as_float(tc_split_lo(r.z, h.z));
    h.w = __uint_as_float(tc_split_hi(r.w)), l.w = __uint_as_float(tc_split_lo(r.w, h.w));
    *reinterpret_cast<float4*>(hi + i) = h;
    *reinterpret_cast<float4*>(lo + i) = l;
}

// kElemQuads float4 quads per thread (strided by the CTA: coalesced), all
// loads issued before any store
constexpr int kElemQuads = 4;
int ctas_elem(long long total) { return std::max(1, ceil_div(total, 4LL * kThreads * kElemQuads)); }
constexpr int kSgdQuads = 1;  // SGD: more CTAs beat deeper per-thread batches (measured)
int ctas_sgd(long long n) { return std::max(1, ceil_div(n, 4LL * kThreads * kSgdQuads)); }

__global__ void __launch_bounds__(kThreads) bn_bwd_apply_kernel(const BnBwdApplyOp* __restrict__ ops, int nd) {
    pdl_trigger();
    int local;
    const BnBwdApplyOp o = op_of(ops, nd, local);  // copy: no reloads after stores
    pdl_wait();  // the static descriptor read above overlaps the predecessor's tail
    if (is_failed(o.failed)) return;
    const float* tg = o.t ? o.t : o.gin;
    const long long cta0 = static_cast<long long>(local) * kThreads * kElemQuads * 4;
    if ((o.c & 3) == 0 && (4 * kThreads * kElemQuads) % o.c == 0 && cta0 + 4LL * kThreads * kElemQuads <= o.total) {
        // c divides the CTA's element span: all of this thread's quads are the
        // same four channels, so the per-channel parameters and the products
        // gamma*inv, inv_m*sg (bn_bwd_one) are loaded / formed once
        const int ch = (threadIdx.x * 4) % o.c;
        const float4 mn = __ldg(reinterpret_cast<const float4*>(o.mean + ch));
        const float4 iv = __ldg(reinterpret_cast<const float4*>(o.inv + ch));
        const float4 gm = __ldg(reinterpret_cast<const float4*>(o.gamma + ch));
        const float4 bt = __ldg(reinterpret_cast<const float4*>(o.beta + ch));
        const float4 s1 = __ldg(reinterpret_cast<const float4*>(o.sg + ch));
        const float4 s2 = __ldg(reinterpret_cast<const float4*>(o.sgx + ch));
        const float mnv[4] = {mn.x, mn.y, mn.z, mn.w}, ivv[4] = {iv.x, iv.y, iv.z, iv.w};
        const float gmv[4] = {gm.x, gm.y, gm.z, gm.w}, btv[4] = {bt.x, bt.y, bt.z, bt.w};
        const float s2v[4] = {s2.x, s2.y, s2.z, s2.w};
        float kk[4], a1[4];
        const float s1v[4] = {s1.x, s1.y, s1.z, s1.w};
#pragma unroll
        for (int q = 0; q < 4; ++q) kk[q] = mul(gmv[q], ivv[q]), a1[q] = mul(o.inv_m, s1v[q]);
        float4 p[kElemQuads], g[kElemQuads];
#pragma unroll
        for (int j = 0; j < kElemQuads; ++j) {
            const long long i = cta0 + (static_cast<long long>(j) * kThreads + threadIdx.x) * 4;
            p[j] = __ldg(reinterpret_cast<const float4*>(o.p + i));
            g[j] = __ldg(reinterpret_cast<const float4*>(tg + (o.trows ? row_remap(o.trows, o.srow, i) : i)));
        }
#pragma unroll
        for (int j = 0; j < kElemQuads; ++j) {
            const long long i = cta0 + (static_cast<long long>(j) * kThreads + threadIdx.x) * 4;
            const float pv[4] = {p[j].x, p[j].y, p[j].z, p[j].w}, gv[4] = {g[j].x, g[j].y, g[j].z, g[j].w};
            float rv[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {  // bn_bwd_one with the hoisted products
                const float xh = mul(sub(pv[q], mnv[q]), ivv[q]);
                float gy;
                if (o.t) {
                    const float y = add(mul(gmv[q], xh), btv[q]);
                    const float d = sub(relu(y), gv[q]);
                    gy = y > 0.0f ? add(0.0f, mul(o.kmse, d)) : 0.0f;
                } else {
                    gy = gv[q];
                }
                const float inner = sub(sub(gy, a1[q]), mul(mul(xh, o.inv_m), s2v[q]));
                rv[q] = add(0.0f, mul(kk[q], inner));
            }
            const float4 r = make_float4(rv[0], rv[1], rv[2], rv[3]);
            if (o.gout_hi) split_store4(o.gout_hi, o.gout_lo, i, r);
            else *reinterpret_cast<float4*>(o.gout + i) = r;
        }
        return;
    }
    if ((o.c & 3) == 0 && cta0 + 4LL * kThreads * kElemQuads <= o.total) {
        float4 p[kElemQuads], g[kElemQuads];
#pragma unroll
        for (int j = 0; j < kElemQuads; ++j) {
            const long long i = cta0 + (static_cast<long long>(j) * kThreads + threadIdx.x) * 4;
            p[j] = __ldg(reinterpret_cast<const float4*>(o.p + i));
            g[j] = __ldg(reinterpret_cast<const float4*>(tg + (o.trows ? row_remap(o.trows, o.srow, i) : i)));
        }
#pragma unroll
        for (int j = 0; j < kElemQuads; ++j) {
            const long long i = cta0 + (static_cast<long long>(j) * kThreads + threadIdx.x) * 4;
            const float4 r = bn_bwd_quad(o, static_cast<int>(i % o.c), p[j], g[j]);
            if (o.gout_hi) split_store4(o.gout_hi, o.gout_lo, i, r);
            else *reinterpret_cast<float4*>(o.gout + i) = r;
        }
        return;
    }
    for (int j = 0; j < kElemQuads; ++j) {  // tail / odd channel counts
        const long long base = cta0 + (static_cast<long long>(j) * kThreads + threadIdx.x) * 4;
        if (base >= o.total) break;
        float pv[4], gv[4], rv[4];
        const int cnt = static_cast<int>(min(4LL, o.total - base));
        for (int q = 0; q < cnt; ++q) pv[q] = o.p[base + q], gv[q] = tg[o.trows ? row_remap(o.trows, o.srow, base + q) : base + q];
        for (int q = 0; q < cnt; ++q) rv[q] = bn_bwd_one(o, bn_bwd_par(o, static_cast<int>((base + q) % o.c)), pv[q], gv[q]);
        for (int q = 0; q < cnt; ++q) {
            if (o.gout_hi) {
                const float hv = __uint_as_float(tc_split_hi(rv[q]));
                o.gout_hi[base + q] = hv;
                o.gout_lo[base + q] = __uint_as_float(tc_split_lo(rv[q], hv));
            } else {
                o.gout[base + q] = rv[q];
            }
        }
    }
}

void launch_bn_bwd_apply(const BnBwdApplyOp* d, int nd, int ctas, cudaStream_t st) {
    launch_k(bn_bwd_apply_kernel, dim3(ctas), dim3(kThreads), 0, st, d, nd);
    PBKD_LAUNCH_CHECK();
}

// -------------------------------------------------------------------- SGD
__device__ __forceinline__ void sgd_quad(const SgdOp& o, long long i, float4 v, float4 g, float4 w) {
    // v = m*v + g; w = w - lr*v   (ops.hpp:554-557, two roundings each)
    float4 nv, nw;
    nv.x = add(mul(o.mom, v.x), g.x), nv.y = add(mul(o.mom, v.y), g.y);
    nv.z = add(mul(o.mom, v.z), g.z), nv.w = add(mul(o.mom, v.w), g.w);
    nw.x = sub(w.x, mul(o.lr, nv.x)), nw.y = sub(w.y, mul(o.lr, nv.y));
    nw.z = sub(w.z, mul(o.lr, nv.z)), nw.w = sub(w.w, mul(o.lr, nv.w));
    *reinterpret_cast<float4*>(o.v + i) = nv;
    *reinterpret_cast<float4*>(o.w + i) = nw;
    if (o.w_hi) split_store4(o.w_hi, o.w_lo, i, nw);
}

__global__ void __launch_bounds__(kThreads) sgd_kernel(const SgdOp* __restrict__ ops, int nd) {
    pdl_trigger();
    int local;
    const SgdOp o = op_of(ops, nd, local);  // copy: no reloads after stores
    pdl_wait();  // the static descriptor read above overlaps the predecessor's tail
    if (is_failed(o.failed)) return;
    const long long cta0 = static_cast<long long>(local) * kThreads * kSgdQuads * 4;
    if (cta0 + 4LL * kThreads * kSgdQuads <= o.n) {  // flat buffers: 16-byte aligned, n % 4 == 0
        float4 v[kSgdQuads], g[kSgdQuads], w[kSgdQuads];
#pragma unroll
        for (int j = 0; j < kSgdQuads; ++j) {
            const long long i = cta0 + (static_cast<long long>(j) * kThreads + threadIdx.x) * 4;
            v[j] = *reinterpret_cast<const float4*>(o.v + i);
            g[j] = __ldg(reinterpret_cast<const float4*>(o.g + i));
            w[j] = *reinterpret_cast<const float4*>(o.w + i);
        }
#pragma unroll
        for (int j = 0; j < kSgdQuads; ++j)
            sgd_quad(o, cta0 + (static_cast<long long>(j) * kThreads + threadIdx.x) * 4, v[j], g[j], w[j]);
        return;
    }
    for (int j = 0; j < kSgdQuads; ++j) {
        const long long base = cta0 + (static_cast<long long>(j) * kThreads + threadIdx.x) * 4;
        for (long long i = base; i < min(o.n, base + 4); ++i) {
            const float vv = add(mul(o.mom, o.v[i]), o.g[i]);
            o.v[i] = vv;
            const float ww = sub(o.w[i], mul(o.lr, vv));
            o.w[i] = ww;
            if (o.w_hi) {
                const float hv = __uint_as_float(tc_split_hi(ww));
                o.w_hi[i] = hv;
                o.w_lo[i] = __uint_as_float(tc_split_lo(ww, hv));
            }
        }
    }
}

void launch_sgd(const SgdOp* d, int nd, int ctas, cudaStream_t st) {
    launch_k(sgd_kernel, dim3(ctas), dim3(kThreads), 0, st, d, nd);
    PBKD_LAUNCH_CHECK();
}

// ---------------------------------------------------------------- scatter
__global__ void __launch_bounds__(kThreads) scatter_kernel(const ScatterOp* __restrict__ ops, int nd) {
    pdl_trigger();
    int local;
    const ScatterOp o = op_of(ops, nd, local);  // copy: no reloads after stores
    pdl_wait();  // the static descriptor read above overlaps the predecessor's tail
    const long long step = static_cast<long long>(kThreads) * kScatterCtas;
    if (o.cd > 0) {  // channel-padded destination rows
        const long long total = static_cast<long long>(o.rows) * o.width;
        const long long wd = static_cast<long long>(o.width / o.cs) * o.cd;
        for (long long i = static_cast<long long>(local) * kThreads + threadIdx.x; i < total; i += step) {
            const long long r = i / o.width, j = i - r * o.width;
            const long long px = j / o.cs, ch = j - px * o.cs;
            o.dst[static_cast<long long>(__ldg(o.pos + r)) * wd + px * o.cd + ch] = __ldg(o.src + i);
        }
        return;
    }
    if ((o.width % 4) == 0) {
        const int wv = o.width / 4;
        const long long total = static_cast<long long>(o.rows) * wv;
        const float4* src = reinterpret_cast<const float4*>(o.src);
        float4* dst = reinterpret_cast<float4*>(o.dst);
        for (long long i = static_cast<long long>(local) * kThreads + threadIdx.x; i < total; i += 4 * step) {
            float4 v[4];
            long long d[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {  // all loads first
                const long long ii = i + u * step;
                if (ii < total) {
                    const long long r = ii / wv;
                    d[u] = static_cast<long long>(__ldg(o.pos + r)) * wv + (ii - r * wv);
                    v[u] = __ldg(src + ii);
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (i + u * step < total) dst[d[u]] = v[u];
        }
        return;
    }
    const long long total = static_cast<long long>(o.rows) * o.width;
    for (long long i = static_cast<long long>(local) * kThreads + threadIdx.x; i < total; i += step) {
        const long long r = i / o.width, j = i - r * o.width;
        o.dst[static_cast<long long>(o.pos[r]) * o.width + j] = o.src[i];
    }
}

void launch_scatter(const ScatterOp* d, int nd, int ctas, cudaStream_t st) {
    launch_k(scatter_kernel, dim3(ctas), dim3(kThreads), 0, st, d, nd);
    PBKD_LAUNCH_CHECK();
}

// ---------------------------------------------------------- non-grouped ---
// tf32 hi / lo planes of x (RNE split, as the GEMM converters do it)
__global__ void tf32_split_kernel(const float* __restrict__ x, long long n, float* __restrict__ hi,
                                  float* __restrict__ lo) {
    pdl_enter();
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const float v = x[i];
        const float h = __uint_as_float(tc_split_hi(v));
        hi[i] = h;
        lo[i] = __uint_as_float(tc_split_lo(v, h));
    }
}

// Teacher conv weights [cout][cin][kk] (model.cpp layout) -> implicit-GEMM
// layout [cout][kk][cin] (K index = tap * cin + j) plus its tf32 planes.
// [cout][cin][kk] -> [cout][kk][cin] rows of pitch kp >= kk * cin (the pad
// stays as the caller zeroed it), with the tf32 planes
__global__ void conv_weight_prep_kernel(const float* __restrict__ raw, int cout, int cin, int kk, int kp,
                                        float* __restrict__ w, float* __restrict__ hi, float* __restrict__ lo) {
    pdl_enter();
    const long long n = static_cast<long long>(cout) * cin * kk;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int j = static_cast<int>(i % cin);
        const long long r = i / cin;
        const int t = static_cast<int>(r % kk);
        const long long o = r / kk;
        const float v = raw[(o * cin + j) * kk + t];
        const float h = __uint_as_float(tc_split_hi(v));
        const long long d = o * kp + static_cast<long long>(t) * cin + j;
        w[d] = v;
        hi[d] = h;
        lo[d] = __uint_as_float(tc_split_lo(v, h));
    }
}

void launch_conv_weight_prep(const float* raw, int cout, int cin, int kk, int kp, float* w, float* hi, float* lo,
                             cudaStream_t st) {
    const long long n = static_cast<long long>(cout) * cin * kk;
    const int blocks = static_cast<int>(std::min<long long>(4096, (n + 255) / 256));
    launch_k(conv_weight_prep_kernel, dim3(std::max(1, blocks)), dim3(256), 0, st, raw, cout, cin, kk, kp, w, hi, lo);
    PBKD_LAUNCH_CHECK();
}

void launch_tf32_split(const float* x, long long n, float* hi, float* lo, cudaStream_t st) {
    const int blocks = static_cast<int>(std::min<long long>(4096, (n + 255) / 256));
    launch_k(tf32_split_kernel, dim3(std::max(1, blocks)), dim3(256), 0, st, x, n, hi, lo);
    PBKD_LAUNCH_CHECK();
}

__global__ void gather_nhwc_kernel(const float* __restrict__ img, const int* __restrict__ idx, int n,
                                   int c, int h, int w, float* __restrict__ out) {
    pdl_enter();
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
    launch_k(gather_nhwc_kernel, dim3(std::max(1, blocks)), dim3(256), 0, st, images, idx, n, c, h, w, out);
    PBKD_LAUNCH_CHECK();
}

__global__ void bn_infer_prep_kernel(const float* gamma, const float* beta, const float* mm,
                                     const float* mv, int c, float* scale, float* shift) {
    pdl_enter();
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= c) return;
    const float inv = __fdiv_rn(1.0f, __fsqrt_rn(add(mv[j], 1e-5f)));
    const float sc = mul(gamma[j], inv);
    scale[j] = sc;
    shift[j] = sub(beta[j], mul(mm[j], sc));
}

void launch_bn_infer_prep(const float* gamma, const float* beta, const float* mm, const float* mv,
                          int c, float* scale, float* shift, cudaStream_t st) {
    launch_k(bn_infer_prep_kernel, dim3(ceil_div(c, 256)), dim3(256), 0, st, gamma, beta, mm, mv, c, scale, shift);
    PBKD_LAUNCH_CHECK();
}

__global__ void bn_infer_relu_kernel(const float* x, float* y, long long total, int c,
                                     const float* scale, const float* shift) {
    pdl_enter();
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int ch = static_cast<int>(i % c);
        y[i] = relu(bn_infer_apply(x[i], scale[ch], shift[ch]));
    }
}

void launch_bn_infer_relu(const float* x, float* y, long long total, int c, const float* scale,
                          const float* shift, cudaStream_t st) {
    const int blocks = static_cast<int>(std::min<long long>(4096, (total + 255) / 256));
    launch_k(bn_infer_relu_kernel, dim3(std::max(1, blocks)), dim3(256), 0, st, x, y, total, c, scale, shift);
    PBKD_LAUNCH_CHECK();
}

// ------------------------------------------------------------- max pool
__global__ void maxpool3x3_kernel(const float* __restrict__ x, float* __restrict__ y, float* y_hi, float* y_lo,
                                  int n, int h, int w, int c, int ho, int wo) {
    pdl_enter();
    const long long total = static_cast<long long>(n) * ho * wo * c;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int ch = static_cast<int>(i % c);
        long long r = i / c;
        const int ox = static_cast<int>(r % wo);
        r /= wo;
        const int oy = static_cast<int>(r % ho);
        const long long b = r / ho;
        float m = -INFINITY;
        for (int ky = 0; ky < 3; ++ky) {
            const int iy = oy * 2 - 1 + ky;
            if (iy < 0 || iy >= h) continue;
            for (int kx = 0; kx < 3; ++kx) {
                const int ix = ox * 2 - 1 + kx;
                if (ix < 0 || ix >= w) continue;
                m = fmaxf(m, x[((b * h + iy) * w + ix) * c + ch]);
            }
        }
        y[i] = m;
        if (y_hi) {
            const float hv = __uint_as_float(tc_split_hi(m));
            y_hi[i] = hv;
            y_lo[i] = __uint_as_float(tc_split_lo(m, hv));
        }
    }
}

void launch_maxpool3x3(const float* x, float* y, float* y_hi, float* y_lo, int n, int h, int w, int c,
                       cudaStream_t st) {
    const int ho = (h + 2 - 3) / 2 + 1, wo = (w + 2 - 3) / 2 + 1;
    const long long total = static_cast<long long>(n) * ho * wo * c;
    const int blocks = static_cast<int>(std::max<long long>(1, std::min<long long>(148LL * 16, (total + 255) / 256)));
    launch_k(maxpool3x3_kernel, dim3(blocks), dim3(256), 0, st, x, y, y_hi, y_lo, n, h, w, c, ho, wo);
    PBKD_LAUNCH_CHECK();
}

__global__ void maxpool3x3_bwd_kernel(const float* __restrict__ x, const float* __restrict__ gy, float* gx, int n,
                                      int h, int w, int c, int ho, int wo) {
    pdl_enter();
    const long long total = static_cast<long long>(n) * h * w * c;
    for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
         i += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int ch = static_cast<int>(i % c);
        long long r = i / c;
        const int ix = static_cast<int>(r % w);
        r /= w;
        const int iy = static_cast<int>(r % h);
        const long long b = r / h;
        float acc = 0.0f;
        for (int oy = max(0, iy / 2 - 1); oy <= min(ho - 1, (iy + 1) / 2); ++oy)
            for (int ox = max(0, ix / 2 - 1); ox <= min(wo - 1, (ix + 1) / 2); ++ox) {
                int by = -1, bx = -1;  // the window's first maximum
                float m = -INFINITY;
                for (int ky = 0; ky < 3; ++ky) {
                    const int yy = oy * 2 - 1 + ky;
                    if (yy < 0 || yy >= h) continue;
                    for (int kx = 0; kx < 3; ++kx) {
                        const int xx = ox * 2 - 1 + kx;
                        if (xx < 0 || xx >= w) continue;
                        const float v = x[((b * h + yy) * w + xx) * c + ch];
                        if (v > m || by < 0) m = v, by = yy, bx = xx;
                    }
                }
                if (by == iy && bx == ix) acc = __fadd_rn(acc, gy[((b * ho + oy) * wo + ox) * c + ch]);
            }
        gx[i] = __fadd_rn(gx[i], acc);
    }
}

void launch_maxpool3x3_bwd(const float* x, const float* gy, float* gx, int n, int h, int w, int c, cudaStream_t st) {
    const int ho = (h + 2 - 3) / 2 + 1, wo = (w + 2 - 3) / 2 + 1;
    const long long total = static_cast<long long>(n) * h * w * c;
    const int blocks = static_cast<int>(std::max<long long>(1, std::min<long long>(148LL * 16, (total + 255) / 256)));
    launch_k(maxpool3x3_bwd_kernel, dim3(blocks), dim3(256), 0, st, x, gy, gx, n, h, w, c, ho, wo);
    PBKD_LAUNCH_CHECK();
}

// one CTA per segment: fixed-order double sum of (s-t)^2
__global__ void mse_segments_kernel(const float* s, const float* t, long long seg, long long total,
                                    double* out) {
    pdl_enter();
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
    launch_k(mse_segments_kernel, dim3(nseg), dim3(256), 0, st, s, t, seg, total, out);
    PBKD_LAUNCH_CHECK();
}

// One CTA per sample.  GAP and dense keep the reference's serial order per
// output (ops.hpp:395-442); argmax keeps the first maximum (distill.cpp:42-52).
__global__ void classifier_kernel(const float* __restrict__ x, int hw, int c, const int* kinds,
                                  int nlayers, const float* dw, const float* db, int nout,
                                  const int* labels, int* correct) {
    pdl_enter();
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
    launch_k(classifier_kernel, dim3(n), dim3(128), smem, st, x, hw, c, kinds, nlayers, dw, db, nout, labels, correct);
    PBKD_LAUNCH_CHECK();
}

}  // namespace pbkd_gpu
