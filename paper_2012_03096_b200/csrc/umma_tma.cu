// umma_tma.cu -- persistent, warp-specialised tcgen05 GEMM with TMA operand
// loads, for the student pointwise convs (fwd / dgrad / wgrad).
//
//   C[m][n] = sum_k A(m,k) * B(n,k),   fp32 in / fp32 out, 3xTF32 split
//
// Same arithmetic as umma.cu (identical MMA sequence per 32-wide K chunk,
// per-chunk TMEM drain summed in fp32 in chunk order), so both kernels give
// the same bits; this one is built for the HBM-bound pointwise shapes
// (arithmetic intensity <= 125 flop/B) where the register-staged kernel was
// latency-bound.  Warp roles (448 threads):
//
//   warp 0      TMA producer: raw fp32 tiles (A 128x32, B BNx32) into a
//               kR-deep ring, either orientation (K-major or MN-major
//               source), zero fill out of bounds
//   warp 1      TMEM allocator + MMA issuer (one elected lane)
//   warps 2-5   converters: raw fp32 -> tf32 hi / lo in the canonical
//               K-major SWIZZLE_128B layout (transposing MN-major sources),
//               kS-deep operand ring
//   warps 6-13  drain + epilogue: per chunk tcgen05.ld of the chunk's TMEM
//               slot and fp32 add; at the tile end the epilogue (store,
//               batch-norm partials, split-K partials)
//
// Persistent: grid = min(tiles, #SMs); CTA i takes tiles i, i+grid, ... of the
// grouped launch (every task's tiles, cta_begin prefix), all rings continue
// across tiles so the next tile's loads overlap this tile's epilogue.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <vector>

#include "gemm_epi.cuh"
#include "ops.cuh"
#include "tc.cuh"

namespace pbkd_gpu {

using namespace tc;

namespace {

constexpr int kWarpsT = 15;
constexpr int kBWarp = 14;  // loads pre-split B (tf32 hi/lo) straight into the operand ring
constexpr int kThreadsT = kWarpsT * 32;
constexpr int kConvThreads = 128;  // warps 2-5
constexpr int kEpiWarp0 = 6;

// PS: every op of the launch takes both operands pre-split (no raw ring, no
// conversion: deeper operand ring).  cs: C staging for the TMA-store
// epilogue, one column half (BN/2 columns x 128 rows, 128-byte swizzled
// 32-column blocks).
template <int BN, bool PS>
struct Cfg {
    static constexpr int R = PS ? 0 : (BN >= 64 ? 2 : 4);  // raw (TMA) stages
#ifdef PBKD_EXP_STAGES128  // diagnosis build only: operand stages of the 128-wide pre-split kernel
    static constexpr int S = PS ? (BN >= 128 ? PBKD_EXP_STAGES128 : BN >= 64 ? 4 : 5) : (BN >= 128 ? 2 : 3);
#else
    static constexpr int S = PS ? (BN >= 128 ? 3 : BN >= 64 ? 4 : 5) : (BN >= 128 ? 2 : 3);  // operand stages
#endif
    static constexpr int a_raw = kBM * kBK * 4;
    static constexpr int b_raw = BN * kBK * 4;
    static constexpr int raw_stage = a_raw + b_raw;
    static constexpr int a_op = kBM * kRowBytes;
    static constexpr int b_op = BN * kRowBytes;
    static constexpr int op_stage = 2 * a_op + 2 * b_op;
    static constexpr int cs = kBM * 32 * 4;  // one 32-column block
    static constexpr int smem = 1024 + R * raw_stage + S * op_stage + cs;
    static constexpr int A = 4;  // TMEM accumulator slots (one per K chunk in flight)
    static constexpr int tmem_cols = (A * BN <= 128) ? 128 : (A * BN <= 256) ? 256 : 512;
    static constexpr int RB = R > 0 ? R : 1;  // barrier array sizes
};

__device__ __forceinline__ float4 lds128(uint32_t a) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ float lds32(uint32_t a) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts128(uint32_t a, uint32_t x, uint32_t y, uint32_t z, uint32_t w) {
    asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(a), "r"(x), "r"(y), "r"(z), "r"(w) : "memory");
}

struct TileGeo {
    int split, tm, tn, k0, nchunks;
};
struct TileInfo {
    int op;  // -1: skip (the task's failure flag is set)
    TileGeo g;
};
constexpr int kMaxTiles = 64;  // tiles per CTA (host sizes the grid)
constexpr int kMaxOps = 64;    // ops per launch
template <int BN>
__device__ __forceinline__ TileGeo tile_geo(const GemmOp& o, int local) {
    TileGeo g;
    const int tiles_mn = o.tiles_m * o.tiles_n;
    g.split = local / tiles_mn;
    const int rem = local - g.split * tiles_mn;
    g.tm = rem / o.tiles_n;
    g.tn = rem - g.tm * o.tiles_n;
    g.k0 = g.split * o.kchunk;
    const int kend = min(o.K, g.k0 + o.kchunk);
    g.nchunks = max(1, (kend - g.k0 + kBK - 1) / kBK);
    return g;
}

__device__ __forceinline__ bool op_failed(const GemmOp& o) { return o.failed != nullptr && *o.failed != 0; }

// raw tile (rows x 32 fp32) -> hi/lo K-major SW128.  kmajor: raw is
// [rows][32] (128-byte rows); else raw is [32][rows] (MN contiguous).
// Shared-space addresses (u32) so every access is LDS/STS.
__device__ __forceinline__ void split4(const float* x, uint32_t* hv, uint32_t* lv, bool split) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        hv[q] = to_tf32(x[q]);
        lv[q] = split && !isinf(x[q]) ? to_tf32(__fsub_rn(x[q], __uint_as_float(hv[q]))) : 0u;
    }
}
__device__ __forceinline__ void convert_tile(uint32_t raw, uint32_t hi, uint32_t lo, int rows, bool kmajor,
                                             bool split, int ct) {
    const int items = rows * 8;  // (row, 16-byte chunk)
    if (kmajor) {
#pragma unroll 4
        for (int i = ct; i < items; i += kConvThreads) {
            const int r = i >> 3, c = i & 7;
            const float4 x = lds128(raw + r * kRowBytes + c * 16);
            const float xs[4] = {x.x, x.y, x.z, x.w};
            uint32_t hv[4], lv[4];
            split4(xs, hv, lv, split);
            const int off = sw128(r, c);
            sts128(hi + off, hv[0], hv[1], hv[2], hv[3]);
            if (split) sts128(lo + off, lv[0], lv[1], lv[2], lv[3]);
        }
    } else {
#pragma unroll 4
        for (int i = ct; i < items; i += kConvThreads) {
            const int r = i % rows, c = i / rows;
            float xs[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) xs[q] = lds32(raw + ((4 * c + q) * rows + r) * 4);
            uint32_t hv[4], lv[4];
            split4(xs, hv, lv, split);
            const int off = sw128(r, c);
            sts128(hi + off, hv[0], hv[1], hv[2], hv[3]);
            if (split) sts128(lo + off, lv[0], lv[1], lv[2], lv[3]);
        }
    }
}

__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, uint32_t src, int c0, int c1, int c2) {
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(src), "r"(c0), "r"(c1), "r"(c2)
                 : "memory");
}
__device__ __forceinline__ void tma_store_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void tma_store_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void tma_store_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void tma_store_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// Epilogue through shared memory, in 32-column passes: the pass's block of
// the tile (128 rows x 32 columns, 128-byte swizzled: conflict-free
// thread-per-row 16-byte stores) is staged, optionally transformed in place
// (teacher conv: BN affine, skip add, ReLU, tf32 planes of the output),
// written by one TMA store (whole 128-byte lines, tails clipped per split)
// and, for epi 1, reduced into the batch-norm partial sums: warp-level
// butterflies over each 32-row quarter and the quarter order of
// gemm_epilogue, so both epilogues give identical bits.  Loops that need no
// register arrays stay rolled: the kernel's code must fit the instruction
// cache next to the producer / MMA roles.
__device__ __forceinline__ uint32_t cs_addr(uint32_t cs, int r, int col) {  // element (r, col) of a block
    return cs + r * 128 + ((((col >> 2) ^ (r & 7))) << 4) + (col & 3) * 4;
}

template <int BN, int KIND>
__device__ __forceinline__ void staged_epilogue(const GemmOp& op, const float* acc, int tm, int tn, int split, int q,
                                                int h, int lane, int et, float (*red)[4][32], uint32_t cs0,
                                                uint32_t cs1, int& stores, int bnt) {
    constexpr int HB = BN / 2;
    const int warp8 = et >> 5;
    // every descriptor field in registers up front: the global stores below
    // could alias the descriptor, which would force a reload of each field
    // after each store (a dependent L1/L2 round trip per element)
    const int M = op.M, N = op.N, epi = op.epi, relu_on = op.relu;
    const long long ldc = op.ldc;
    const float* __restrict__ scale = op.scale;
    const float* __restrict__ shift = op.shift;
    const float* __restrict__ skip = op.skip;
    float* __restrict__ c_hi = op.c_hi;
    float* __restrict__ c_lo = op.c_lo;
    float* __restrict__ part0 = op.part0;
    float* __restrict__ part1 = op.part1;
    const CUtensorMap* map_c = &op.map_c;
    const int bm = (KIND == kGemmKindConv && op.conv) ? op.bm : kBM;  // rows of this tile
    const int m0 = tm * bm, n0 = tn * bnt;  // bnt: the op's N tile (<= BN)
    const int r = q * 32 + lane;
    const bool xform = KIND == kGemmKindConv && (scale || skip || relu_on || c_hi);
#pragma unroll
    for (int pass = 0; pass < BN / 32; ++pass) {
        if (pass * 32 >= bnt) break;  // tile-uniform
        // staging block of this pass: with a second block (cs1) the passes
        // alternate, so only the store issued two passes ago must have read
        // its block; otherwise the previous pass's store
        const uint32_t cs = (cs1 && (stores & 1)) ? cs1 : cs0;
        if (et == 0 && stores) {
            if (cs1) tma_store_wait_read1();
            else tma_store_wait_read();
        }
        named_bar(1, 256);
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            const int col = pass * 32 + 4 * c;  // tile column (compile time)
            const int hh = col / HB;
            if (h == hh) {
                const int j = col - hh * HB;
                sts128(cs + r * 128 + ((c ^ (r & 7)) << 4), __float_as_uint(acc[j]), __float_as_uint(acc[j + 1]),
                       __float_as_uint(acc[j + 2]), __float_as_uint(acc[j + 3]));
            }
        }
        if (xform) {  // thread = column (lane), rows strided by warp
            named_bar(1, 256);
            const int n = n0 + pass * 32 + lane;
            float sc = 1.0f, sh = 0.0f;
            if (scale && n < N) sc = __ldg(scale + n), sh = __ldg(shift + n);
            for (int rr = warp8; rr < bm; rr += 8) {
                const int row = m0 + rr;
                if (row >= M || n >= N) continue;
                const uint32_t a = cs_addr(cs, rr, lane);
                float x = lds32(a);
                if (scale) x = bn_infer_apply(x, sc, sh);
                if (skip) x = add(x, __ldg(skip + static_cast<long long>(row) * ldc + n));
                if (relu_on) x = relu(x);
                asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(x) : "memory");
                if (c_hi) {
                    const float hv = __uint_as_float(tc_split_hi(x));
                    c_hi[static_cast<long long>(row) * ldc + n] = hv;
                    c_lo[static_cast<long long>(row) * ldc + n] = __uint_as_float(tc_split_lo(x, hv));
                }
            }
        }
        fence_async_smem();
        named_bar(1, 256);
        if (et == 0) {
            tma_store_3d(map_c, cs, n0 + pass * 32, m0, split);  // split 0 unless split-K (epi 2)
            tma_store_commit();
        }
        ++stores;  // every thread: the pass parity picks the staging block
        if (KIND == 1) {
            // thread = (column, row quarter, sum | sum of squares), warp-uniform
            // quarter and kind: the quarter's 32 rows summed serially in the
            // xor-butterfly tree of gemm_epilogue (rows i, i+16 first, then
            // +8, +4, +2, +1: identical bits, no shuffle latency chains)
            const int col = et & 31, qq = (et >> 5) & 3, sqr = et >> 7;
            float v[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                float x[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {  // rows i, i+16, i+8, i+24
                    x[k] = lds32(cs_addr(cs, qq * 32 + i + (k & 1) * 16 + (k >> 1) * 8, col));
                    if (sqr) x[k] = __fmul_rn(x[k], x[k]);
                }
                v[i] = __fadd_rn(__fadd_rn(x[0], x[1]), __fadd_rn(x[2], x[3]));
            }
#pragma unroll
            for (int w = 4; w > 0; w >>= 1)
#pragma unroll
                for (int i = 0; i < w; ++i) v[i] = __fadd_rn(v[i], v[i + w]);
            red[sqr][qq][col] = v[0];
            named_bar(1, 256);
            if (et < 32) {
                const int cg = n0 + pass * 32 + et;
                if (cg < N) {
                    part0[static_cast<long long>(tm) * N + cg] =
                        __fadd_rn(__fadd_rn(red[0][0][et], red[0][1][et]), __fadd_rn(red[0][2][et], red[0][3][et]));
                    part1[static_cast<long long>(tm) * N + cg] =
                        __fadd_rn(__fadd_rn(red[1][0][et], red[1][1][et]), __fadd_rn(red[1][2][et], red[1][3][et]));
                }
            }
        }
    }
}

}  // namespace

template <int BN, bool PS, int KIND>
__global__ void __launch_bounds__(kThreadsT, 1) umma_tma_kernel(const GemmOp* __restrict__ ops, int nd, int total,
                                                                 unsigned long long* __restrict__ trace,
                                                                 const int* __restrict__ perm) {
    using C = Cfg<BN, PS>;
    constexpr bool CONV = KIND == kGemmKindConv;
    constexpr int R = C::R, S = C::S, HB = BN / 2;
    extern __shared__ uint8_t smem_raw[];
    __shared__ uint64_t raw_full[C::RB], raw_empty[C::RB], op_full[S], op_empty[S], acc_full[C::A], acc_empty[C::A];
    __shared__ uint32_t tmem_base_sh;
    __shared__ float red_buf[256];  // [8][32] (gemm_epilogue) or [2][4][32] (staged_epilogue)
    auto red = reinterpret_cast<float(*)[4][32]>(red_buf);
    __shared__ int begins[kMaxOps];
    __shared__ TileInfo tiles_sh[kMaxTiles];

    // Pipeline tracer (build with -DPBKD_GEMM_TRACE_BUILD, run with
    // PBKD_GEMM_TRACE=<launch>): CTA 0 globaltimer stamps per event.
#ifdef PBKD_GEMM_TRACE_BUILD
    const bool tr_on = trace != nullptr && blockIdx.x == 0;
    auto mark = [&](int ev, uint32_t i) {
        if (tr_on && i < 512) {
            unsigned long long t;
            asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
            trace[ev * 512 + i] = t;
        }
    };
#else
    auto mark = [](int, uint32_t) {};
    (void)trace;
#endif
    if (threadIdx.x == 0) mark(5, 0);
#ifdef PBKD_GEMM_TRACE_BUILD
    if (trace != nullptr && threadIdx.x == 0 && blockIdx.x < 1024) {  // per-CTA start
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        trace[10 * 512 + blockIdx.x] = t;
    }
#endif
    const uint32_t sbase = smem_u32(smem_raw);
    const uint32_t pad = (1024u - (sbase & 1023u)) & 1023u;
    uint8_t* raw_ring = smem_raw + pad;  // stays a shared-space pointer
    uint8_t* op_ring = raw_ring + R * C::raw_stage;
    const uint32_t raw_s = sbase + pad, op_s = raw_s + R * C::raw_stage;
    const uint32_t cs_s = op_s + S * C::op_stage;  // epilogue staging (C::cs bytes)
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                     "r"(C::tmem_cols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        for (int i = 0; i < R; ++i) {
            mbar_init(&raw_full[i], 1);
            mbar_init(&raw_empty[i], kConvThreads / 32);
        }
        for (int i = 0; i < S; ++i) {
            mbar_init(&op_full[i], PS ? 1 : kConvThreads / 32 + 1);  // converters + the loader warp
            mbar_init(&op_empty[i], 1);
        }
        for (int i = 0; i < C::A; ++i) {
            mbar_init(&acc_full[i], 1);
            mbar_init(&acc_empty[i], 8);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // decode this CTA's tiles once (all threads in parallel: one global-load
    // latency instead of a dependent chain per tile per role).  The op
    // descriptors are static, so this runs before the programmatic-launch
    // wait (overlapping the predecessor's tail); failure flags and operands
    // are read only after it.
    for (int i = tid; i < nd; i += kThreadsT) begins[i] = ops[i].cta_begin;
    __syncthreads();
    const int ntiles = static_cast<int>(blockIdx.x) < total ? (total - 1 - static_cast<int>(blockIdx.x)) / static_cast<int>(gridDim.x) + 1 : 0;
    for (int j = tid; j < ntiles; j += kThreadsT) {
        int t = static_cast<int>(blockIdx.x) + j * static_cast<int>(gridDim.x);
        if (perm) {  // balanced slot -> tile map (host LPT schedule)
            t = perm[t];
            if (t < 0) {
                tiles_sh[j].op = -1;
                continue;
            }
        }
        int lo = 0, hi = nd - 1;  // last op with begins[op] <= t
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (begins[mid] <= t) lo = mid;
            else hi = mid - 1;
        }
        const GemmOp& o = ops[lo];
        TileInfo ti;
        ti.op = lo;
        ti.g = tile_geo<BN>(o, t - begins[lo]);
        tiles_sh[j] = ti;
        if (j == 0) {  // warm the first tile's tensor maps
            if (o.a_presplit) prefetch_map(&o.map_ah), prefetch_map(&o.map_al);
            else prefetch_map(&o.map_a);
            if (o.b_presplit) prefetch_map(&o.map_bh), prefetch_map(&o.map_bl);
            else prefetch_map(&o.map_b);
        }
    }
    // predecessor results (failure flags, operands) only after this point
    pdl_enter();
    for (int j = tid; j < ntiles; j += kThreadsT)
        if (tiles_sh[j].op >= 0 && op_failed(ops[tiles_sh[j].op])) tiles_sh[j].op = -1;  // task predicated off (diverged)
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base_sh;
    if (threadIdx.x == 0) mark(5, 1);

    if (warp == 0) {
        // ------------------------------------------------------ TMA producer
        if (PS) goto done;  // nothing to convert: no raw loads
        uint32_t it = 0;
        for (int j = 0; j < ntiles; ++j) {
            if (tiles_sh[j].op < 0) continue;  // task predicated off (diverged)
            const GemmOp& o = ops[tiles_sh[j].op];
            const TileGeo g = tiles_sh[j].g;
            const bool conv = CONV && o.conv != 0, akm = o.a_kmajor != 0, bkm = o.b_kmajor != 0;
            const int bm = conv ? o.bm : kBM;
            const int m0 = g.tm * bm, n0 = g.tn * BN;
            int img = 0, y0 = 0;
            if (conv) {  // tiles cover whole output rows / images (gemm_tma_prepare)
                const int hw = o.oh * o.ow;
                img = m0 / hw;
                y0 = (m0 - img * hw) / o.ow * o.cstride - o.cpad;
            }
            if (lane == 0) {
                for (int kc = 0; kc < g.nchunks; ++kc, ++it) {
                    const int r = it % R;
                    mbar_wait(&raw_empty[r], ((it / R) & 1) ^ 1);
                    uint8_t* st = raw_ring + r * C::raw_stage;
                    const uint32_t bytes = (o.a_presplit ? 0 : bm * kBK * 4) + (o.b_presplit ? 0 : C::b_raw);
                    if (bytes == 0) {  // both operands go straight to the operand ring
                        mbar_arrive(&raw_full[r]);
                        continue;
                    }
                    mbar_arrive_expect_tx(&raw_full[r], bytes);
                    const int k = g.k0 + kc * kBK;
                    if (o.a_presplit) {
                        // A goes straight to the operand ring (warp kBWarp)
                    } else if (conv) {  // implicit im2col: tap (ky,kx), channels c0..c0+31
                        const int tap = k / o.ic, c0 = k - tap * o.ic;
                        const int ky = tap / o.ksz, kx = tap - ky * o.ksz;
                        tma_load_4d(st, &o.map_a, &raw_full[r], c0, kx - o.cpad, y0 + ky, img);
                    } else if (akm) {
                        tma_load_2d(st, &o.map_a, &raw_full[r], k, m0);
                    } else {
                        tma_load_2d(st, &o.map_a, &raw_full[r], m0, k);
                    }
                    mark(0, it);
                    if (o.b_presplit) {
                        // B goes straight to the operand ring (warp kBWarp)
                    } else if (bkm) {
                        tma_load_2d(st + C::a_raw, &o.map_b, &raw_full[r], k, n0);
                    } else {
                        tma_load_2d(st + C::a_raw, &o.map_b, &raw_full[r], n0, k);
                    }
                }
            } else {
                it += g.nchunks;
            }
            __syncwarp();
        }
    } else if (warp == 1) {
        // ------------------------------------------------------ MMA issuer
        // whole warp waits (warp-uniform values), one elected lane issues
        uint32_t it = 0;
        for (int j = 0; j < ntiles; ++j) {
            if (tiles_sh[j].op < 0) continue;  // task predicated off (diverged)
            const GemmOp& o = ops[tiles_sh[j].op];
            const TileGeo g = tiles_sh[j].g;
            const int terms = o.tf32x3;
            // pre-split MN-major operands stay MN-major in shared memory
            const bool amn = o.a_presplit && !(CONV && o.conv) && !o.a_kmajor, bmn = o.b_presplit && !o.b_kmajor;
            const uint32_t idesc = instr_desc(PS ? o.bn : BN, amn, bmn);
            for (int kc = 0; kc < g.nchunks; ++kc, ++it) {
                const int s = it % S, a = it % C::A;
                mbar_wait(&op_full[s], (it / S) & 1);
                mbar_wait(&acc_empty[a], ((it / C::A) & 1) ^ 1);
                tc_fence_after();
                const uint32_t ah = op_s + s * C::op_stage, al = ah + C::a_op, bh = al + C::a_op, bl = bh + C::b_op;
                if (elect_one()) {
                    if ((amn || bmn) && terms == 3) {
                        // MN-major (BASE32B): atoms of 32 MN x 4 K (512 B), MN atoms
                        // 4096 B apart (one TMA box each); a k-step of 8 advances 1024 B
                        constexpr uint32_t lbo = 4096, sbo = 512;
                        const uint64_t dah = amn ? smem_desc_mn(ah, lbo, sbo) : smem_desc(ah);
                        const uint64_t dal = amn ? smem_desc_mn(al, lbo, sbo) : smem_desc(al);
                        const uint64_t dbh = bmn ? smem_desc_mn(bh, lbo, sbo) : smem_desc(bh);
                        const uint64_t dbl = bmn ? smem_desc_mn(bl, lbo, sbo) : smem_desc(bl);
                        mma_chunk3d(tmem + a * BN, dah, dal, dbh, dbl, amn ? 64 : 2, bmn ? 64 : 2, idesc);
                    } else {
#ifdef PBKD_EXP_TERMS1  // diagnosis build only: hi*hi alone (wrong results)
                        mma_chunk(tmem + a * BN, ah, al, bh, bl, idesc, 1);
#else
                        mma_chunk(tmem + a * BN, ah, al, bh, bl, idesc, terms);
#endif
                    }
                    mma_commit(&op_empty[s]);
                    mma_commit(&acc_full[a]);
                    mark(2, it);
                }
                __syncwarp();
            }
        }
    } else if (warp == kBWarp) {
        // ------------------------------------------------------ operand loader
        // pre-split (tf32 hi / lo) operands straight into the operand ring:
        // K-major as one 128-byte-swizzled box per plane, MN-major as one
        // {32 MN, 32 K} swizzled box per 32-wide MN atom.  One arrive per chunk
        // on op_full (with the bytes), after the stage is free.
        uint32_t it = 0;
        for (int j = 0; j < ntiles; ++j) {
            if (tiles_sh[j].op < 0) continue;  // task predicated off (diverged)
            const GemmOp& o = ops[tiles_sh[j].op];
            const TileGeo g = tiles_sh[j].g;
            const int bnt = PS ? o.bn : BN;  // a pre-split launch mixes N tiles (gemm_bn_class)
            const int bm = (CONV && o.conv) ? o.bm : kBM;
            const int m0 = g.tm * bm, n0 = g.tn * bnt;
            const bool apre = o.a_presplit != 0, bpre = o.b_presplit != 0;
            const bool akm = (CONV && o.conv != 0) || o.a_kmajor != 0, bkm = o.b_kmajor != 0;
            int img = 0, y0 = 0;
            if (CONV && o.conv) {
                const int hw = o.oh * o.ow;
                img = m0 / hw;
                y0 = (m0 - img * hw) / o.ow * o.cstride - o.cpad;
            }
            if (lane == 0) {
                for (int kc = 0; kc < g.nchunks; ++kc, ++it) {
                    const int s = it % S;
                    mbar_wait(&op_empty[s], ((it / S) & 1) ^ 1);
#ifdef PBKD_EXP_NOLO  // diagnosis build only: hi planes alone (wrong results)
                    const uint32_t bytes = (apre ? bm * kRowBytes : 0) + (bpre ? bnt * kRowBytes : 0);
#else
                    const uint32_t bytes = (apre ? 2 * bm * kRowBytes : 0) + (bpre ? 2 * bnt * kRowBytes : 0);
#endif
                    if (bytes == 0) {
                        mbar_arrive(&op_full[s]);
                        continue;
                    }
                    mbar_arrive_expect_tx(&op_full[s], bytes);
                    mark(0, it);
                    uint8_t* os = op_ring + s * C::op_stage;
                    const int k = g.k0 + kc * kBK;
                    if (apre) {
                        if (CONV && o.conv) {
                            const int tap = k / o.ic, c0 = k - tap * o.ic;
                            const int ky = tap / o.ksz, kx = tap - ky * o.ksz;
                            tma_load_4d(os, &o.map_ah, &op_full[s], c0, kx - o.cpad, y0 + ky, img);
                            tma_load_4d(os + C::a_op, &o.map_al, &op_full[s], c0, kx - o.cpad, y0 + ky, img);
                        } else if (akm) {
                            tma_load_2d(os, &o.map_ah, &op_full[s], k, m0);
                            #ifndef PBKD_EXP_NOLO
                            tma_load_2d(os + C::a_op, &o.map_al, &op_full[s], k, m0);
#endif
                        } else {
#pragma unroll
                            for (int at = 0; at < kBM / 32; ++at) {
                                tma_load_2d(os + at * 4096, &o.map_ah, &op_full[s], m0 + 32 * at, k);
                                #ifndef PBKD_EXP_NOLO
                                tma_load_2d(os + C::a_op + at * 4096, &o.map_al, &op_full[s], m0 + 32 * at, k);
#endif
                            }
                        }
                    }
                    if (bpre) {
                        uint8_t* ob = os + 2 * C::a_op;
                        if (bkm) {
                            tma_load_2d(ob, &o.map_bh, &op_full[s], k, n0);
                            #ifndef PBKD_EXP_NOLO
                            tma_load_2d(ob + C::b_op, &o.map_bl, &op_full[s], k, n0);
#endif
                        } else {
#pragma unroll
                            for (int at = 0; at < BN / 32; ++at) {
                                if (at * 32 >= bnt) break;
                                tma_load_2d(ob + at * 4096, &o.map_bh, &op_full[s], n0 + 32 * at, k);
                                #ifndef PBKD_EXP_NOLO
                                tma_load_2d(ob + C::b_op + at * 4096, &o.map_bl, &op_full[s], n0 + 32 * at, k);
#endif
                            }
                        }
                    }
                }
            } else {
                it += g.nchunks;
            }
            __syncwarp();
        }
    } else if (warp < kEpiWarp0) {
        // ------------------------------------------------------ converters
        if (PS) goto done;
        const int ct = tid - 64;
        uint32_t it = 0;
        for (int j = 0; j < ntiles; ++j) {
            if (tiles_sh[j].op < 0) continue;  // task predicated off (diverged)
            const GemmOp& o = ops[tiles_sh[j].op];
            const TileGeo g = tiles_sh[j].g;
            const bool split3 = o.tf32x3 > 1;
            const bool akm = (CONV && o.conv != 0) || o.a_kmajor != 0, bkm = o.b_kmajor != 0;
            for (int kc = 0; kc < g.nchunks; ++kc, ++it) {
                const int r = it % R, s = it % S;
                mbar_wait(&raw_full[r], (it / R) & 1);
                if (warp == 2 && lane == 0) mark(6, it);
                mbar_wait(&op_empty[s], ((it / S) & 1) ^ 1);
                if (warp == 2 && lane == 0) mark(7, it);
                const uint32_t rs = raw_s + r * C::raw_stage;
                const uint32_t os = op_s + s * C::op_stage;
                if (!o.a_presplit) convert_tile(rs, os, os + C::a_op, kBM, akm, split3, ct);
                if (warp == 2 && lane == 0) mark(8, it);
                if (!o.b_presplit)
                    convert_tile(rs + C::a_raw, os + 2 * C::a_op, os + 2 * C::a_op + C::b_op, BN, bkm, split3, ct);
                if (warp == 2 && lane == 0) mark(9, it);
                fence_async_smem();
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive(&raw_empty[r]);
                    mbar_arrive(&op_full[s]);
                    if (warp == 2) mark(1, it);
                }
            }
        }
    } else {
        // ------------------------------------------------------ drain + epilogue
        const int q = warp & 3, h = (warp - kEpiWarp0) >> 2, et = tid - kEpiWarp0 * 32;
        const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
        int stores = 0;  // TMA store groups in flight (elected thread)
        uint32_t it = 0;
        for (int j = 0; j < ntiles; ++j) {
            if (tiles_sh[j].op < 0) continue;  // task predicated off (diverged)
            const GemmOp& o = ops[tiles_sh[j].op];
            const TileGeo g = tiles_sh[j].g;
            const int bnt = PS ? o.bn : BN;
            const int hcols = min(HB, max(0, bnt - h * HB));  // this half's live columns
            float acc[HB];
#pragma unroll
            for (int j = 0; j < HB; ++j) acc[j] = 0.0f;
            for (int kc = 0; kc < g.nchunks; ++kc, ++it) {
                const int a = it % C::A;
                mbar_wait(&acc_full[a], (it / C::A) & 1);
                tc_fence_after();
                const uint32_t base = tmem + lane_off + a * BN + h * HB;
#pragma unroll
                for (int c0 = 0; c0 < HB; c0 += 16) {
#ifndef PBKD_EXP_NODRAIN  // diagnosis build only: no per-chunk drain (wrong results)
                    if (c0 < hcols) tmem_add16(base + c0, acc + c0);
#endif
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive(&acc_empty[a]);
                    if (warp == kEpiWarp0) mark(3, it);
                }
            }
            staged_epilogue<BN, KIND>(o, acc, g.tm, g.tn, g.split, q, h, lane, et, red, cs_s, 0u, stores, bnt);
            if (warp == kEpiWarp0 && lane == 0) mark(4, j);
        }
    }
    // the thread that issued the TMA stores waits for them before the CTA's
    // shared memory goes away (bulk async-groups are per thread)
    if (tid == kEpiWarp0 * 32) tma_store_wait_all();
    (void)op_ring;
done:
    tc_fence_before();
    __syncthreads();
#ifdef PBKD_GEMM_TRACE_BUILD
    if (trace != nullptr && threadIdx.x == 0 && blockIdx.x < 1024) {  // per-CTA end and chunk count
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        trace[10 * 512 + 1024 + blockIdx.x] = t;
        unsigned long long nc = 0;
        for (int j = 0; j < ntiles; ++j)
            if (tiles_sh[j].op >= 0) nc += tiles_sh[j].g.nchunks;
        trace[10 * 512 + 2048 + blockIdx.x] = nc | (static_cast<unsigned long long>(ntiles) << 32);
    }
#endif
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(C::tmem_cols));
    }
}

// ------------------------------------------------------- A through TMEM
// Variant for ops whose A operand is raw fp32 in global memory (o.a_tmem):
// the loader warp brings the raw A tile (K-major, 128-byte swizzled, or
// MN-major [32 k][128 m]) and the pre-split B planes into a kSt-deep ring;
// converter warps 2-5 (thread = TMEM lane = tile row) split their row into
// tf32 hi / lo and store them into TMEM (tcgen05.st); the MMA warp issues
// the chunk's 12 MMAs with A read from TMEM ("ts" form) and only B from
// shared memory.  Per 32-wide K chunk the SM's shared memory then carries
// 48 KB of TMA writes + 16 KB of converter reads + 48 KB of MMA reads instead
// of 64 + 96 KB (hi/lo planes of both operands): the pre-split kernel is
// shared-memory-bandwidth bound (tools/probes/gemm_probe.cu).  Same MMA
// sequence and per-chunk drain as umma_tma_kernel: identical bits.
namespace {
constexpr int kTsBN = 128;
constexpr int kTsSt = 4;                                     // smem stages
// TMEM: 3 accumulator slots x 128 + 2 A stages x 64 = all 512 columns (the
// third accumulator slot lets the MMA run further ahead of a tile epilogue;
// 3 A stages / 2 slots measured 0.3% slower on the epoch)
constexpr int kTsTm = 2;                                     // TMEM A stages
constexpr int kTsAcc = 3;                                    // TMEM accumulator slots
constexpr int kTsARaw = kBM * kBK * 4;                       // 16 KB raw A
constexpr int kTsBOp = kTsBN * kRowBytes;                    // 16 KB per B plane
constexpr int kTsStage = kTsARaw + 2 * kTsBOp;               // 48 KB
// + epilogue staging: two alternating 16 KB blocks (one for the forward kind,
// whose batch-norm partial buffer leaves no room for a second next to the ring)
#ifdef PBKD_EXP_TS1_ST3  // diagnosis build: forward kind with 3 operand stages and two staging blocks
template <int KIND>
constexpr int ts_stages() { return KIND == 1 ? 3 : kTsSt; }
template <int KIND>
constexpr int ts_staging_blocks() { return 2; }
#else
template <int KIND>
constexpr int ts_stages() { return kTsSt; }
template <int KIND>
constexpr int ts_staging_blocks() { return KIND == 1 ? 1 : 2; }
#endif
template <int KIND>
constexpr int ts_smem() { return 1024 + ts_stages<KIND>() * kTsStage + ts_staging_blocks<KIND>() * kBM * 32 * 4; }
constexpr int kTsAcol0 = kTsAcc * kTsBN;                     // first TMEM column of the A stages
}  // namespace

#ifdef PBKD_GEMM_TRACE_BUILD
__device__ unsigned long long* g_ts_trace = nullptr;  // per-CTA [start | end | chunks, tiles] (tracer build)
__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#endif

// Raw B box of one operand stage -> tf32 hi in place, lo into the lo plane's
// slot (an elementwise pass: the planes keep the box's swizzled layout), by
// the 256 epilogue threads; generic-proxy stores, then the proxy fence the
// MMA's async-proxy reads need.
__device__ __forceinline__ void split_b_stage(uint32_t bh, uint32_t bl, int bn, int et) {
    const int n16 = bn * (kRowBytes / 16);  // 16-byte items: bn 32 / 64 / 128 -> 1 / 2 / 4 per thread
    // one item at a time: the drain's accumulator registers are live here
#pragma unroll 1
    for (int i = et; i < n16; i += 256) {
        const float4 x = lds128(bh + 16 * i);
        const float xs[4] = {x.x, x.y, x.z, x.w};
        uint32_t h4[4], l4[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            h4[q] = tc_split_hi(xs[q]);
            l4[q] = tc_split_lo(xs[q], __uint_as_float(h4[q]));
        }
        sts128(bh + 16 * i, h4[0], h4[1], h4[2], h4[3]);
        sts128(bl + 16 * i, l4[0], l4[1], l4[2], l4[3]);
    }
    fence_async_smem();
}

template <int KIND>
__global__ void __launch_bounds__(kThreadsT, 1) umma_ts_kernel(const GemmOp* __restrict__ ops, int nd, int total,
                                                                const int* __restrict__ perm) {
    constexpr int BN = kTsBN, HB = BN / 2, S = ts_stages<KIND>(), T = kTsTm, AC = kTsAcc;
    extern __shared__ uint8_t smem_raw[];
#ifdef PBKD_GEMM_TRACE_BUILD
    if (threadIdx.x == 0 && g_ts_trace && blockIdx.x < 1024) g_ts_trace[blockIdx.x] = gtimer();
#endif
    __shared__ uint64_t op_full[S], op_empty[S], a_full[T], a_empty[T], acc_full[AC], acc_empty[AC];
    __shared__ uint64_t b_full[S];  // raw B split by the epilogue warps (launches with b_split ops)
    __shared__ uint32_t tmem_base_sh;
    __shared__ float red_buf[256];
    auto red = reinterpret_cast<float(*)[4][32]>(red_buf);
    __shared__ int begins[kMaxOps];
    __shared__ TileInfo tiles_sh[kMaxTiles];
    const uint32_t sbase = smem_u32(smem_raw);
    const uint32_t pad = (1024u - (sbase & 1023u)) & 1023u;
    uint8_t* ring = smem_raw + pad;
    const uint32_t ring_s = sbase + pad;
    const uint32_t cs_s = ring_s + S * kTsStage;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;

    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                     "r"(512));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        for (int i = 0; i < S; ++i) {
            mbar_init(&op_full[i], 1);
            mbar_init(&op_empty[i], 1);
        }
        for (int i = 0; i < T; ++i) {
            mbar_init(&a_full[i], kConvThreads / 32);
            mbar_init(&a_empty[i], 1);
        }
        for (int i = 0; i < AC; ++i) {
            mbar_init(&acc_full[i], 1);
            mbar_init(&acc_empty[i], 8);
        }
        for (int i = 0; i < S; ++i) mbar_init(&b_full[i], 8);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    int any_bsplit = 0;
    for (int i = tid; i < nd; i += kThreadsT) {
        begins[i] = ops[i].cta_begin;
        any_bsplit |= ops[i].b_split;
    }
    // a launch with raw-B ops: the epilogue warps split every stage's B (an
    // op with planes only passes), the MMA waits for that on every chunk
    const int any_b = __syncthreads_or(any_bsplit);  // also the barrier after the setup above (every kind)
    const bool bsp = KIND == 0 && any_b != 0;
    const int ntiles = static_cast<int>(blockIdx.x) < total ? (total - 1 - static_cast<int>(blockIdx.x)) / static_cast<int>(gridDim.x) + 1 : 0;
    for (int j = tid; j < ntiles; j += kThreadsT) {
        int t = static_cast<int>(blockIdx.x) + j * static_cast<int>(gridDim.x);
        if (perm) {  // balanced slot -> tile map (host LPT schedule)
            t = perm[t];
            if (t < 0) {
                tiles_sh[j].op = -1;
                continue;
            }
        }
        int lo = 0, hi = nd - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (begins[mid] <= t) lo = mid;
            else hi = mid - 1;
        }
        const GemmOp& o = ops[lo];
        TileInfo ti;
        ti.op = lo;
        ti.g = tile_geo<BN>(o, t - begins[lo]);
        tiles_sh[j] = ti;
        if (j == 0) prefetch_map(&o.map_a), prefetch_map(&o.map_bh), prefetch_map(&o.map_bl);
    }
    pdl_enter();
    for (int j = tid; j < ntiles; j += kThreadsT)
        if (tiles_sh[j].op >= 0 && op_failed(ops[tiles_sh[j].op])) tiles_sh[j].op = -1;
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base_sh;

    if (warp == kBWarp) {
        // ------------------------------------------------------ loader
        uint32_t it = 0;
        for (int j = 0; j < ntiles; ++j) {
            if (tiles_sh[j].op < 0) continue;
            const GemmOp& o = ops[tiles_sh[j].op];
            const TileGeo g = tiles_sh[j].g;
            const int bnt = o.bn;
            const bool conv = KIND == kGemmKindConv && o.conv != 0;
            const int bm = conv ? o.bm : kBM;
            const int m0 = g.tm * bm, n0 = g.tn * bnt;
            const bool akm = conv || o.a_kmajor != 0, bkm = o.b_kmajor != 0;
            int img = 0, y0 = 0;
            if (conv) {  // tiles of whole output rows / images (gemm_tma_prepare)
                const int hw = o.oh * o.ow;
                img = m0 / hw;
                y0 = (m0 - img * hw) / o.ow * o.cstride - o.cpad;
            }
            if (lane == 0) {
                for (int kc = 0; kc < g.nchunks; ++kc, ++it) {
                    const int s = it % S;
                    mbar_wait(&op_empty[s], ((it / S) & 1) ^ 1);
                    mbar_arrive_expect_tx(&op_full[s], static_cast<uint32_t>((o.a_gather ? 0 : bm * kBK * 4) +
                                                                             (o.b_split ? 1 : 2) * bnt * kRowBytes));
                    uint8_t* st = ring + s * kTsStage;
                    const int k = g.k0 + kc * kBK;
                    if (o.a_gather) {
                        // A gathered by the converter warps (small channel counts)
                    } else if (conv) {  // implicit im2col: tap (ky, kx), channels c0..c0+31 of the raw input
                        const int tap = k / o.ic, c0 = k - tap * o.ic;
                        const int ky = tap / o.ksz, kx = tap - ky * o.ksz;
                        tma_load_4d(st, &o.map_a, &op_full[s], c0, kx - o.cpad, y0 + ky, img);
                    } else if (akm) {
                        tma_load_2d(st, &o.map_a, &op_full[s], k, m0);
                    } else {
                        tma_load_2d(st, &o.map_a, &op_full[s], m0, k);
                    }
                    uint8_t* ob = st + kTsARaw;
                    if (bkm) {
                        tma_load_2d(ob, &o.map_bh, &op_full[s], k, n0);
                        if (!o.b_split) tma_load_2d(ob + kTsBOp, &o.map_bl, &op_full[s], k, n0);
                    } else {
#pragma unroll
                        for (int at = 0; at < BN / 32; ++at) {
                            if (at * 32 >= bnt) break;
                            tma_load_2d(ob + at * 4096, &o.map_bh, &op_full[s], n0 + 32 * at, k);
                            if (!o.b_split) tma_load_2d(ob + kTsBOp + at * 4096, &o.map_bl, &op_full[s], n0 + 32 * at, k);
                        }
                    }
                }
            } else {
                it += g.nchunks;
            }
            __syncwarp();
        }
    } else if (warp >= 2 && warp < kEpiWarp0) {
        // ------------------------------------------------------ converters
        const int row = (warp & 3) * 32 + lane;  // this warp's TMEM lane quarter
        const uint32_t lane_off = static_cast<uint32_t>((warp & 3) * 32) << 16;
        uint32_t it = 0;
        for (int j = 0; j < ntiles; ++j) {
            if (tiles_sh[j].op < 0) continue;
            const GemmOp& o = ops[tiles_sh[j].op];
            const TileGeo g = tiles_sh[j].g;
            const bool akm = (KIND == kGemmKindConv && o.conv != 0) || o.a_kmajor != 0;
            for (int kc = 0; kc < g.nchunks; ++kc, ++it) {
                const int s = it % S, t = it % T;
                mbar_wait(&op_full[s], (it / S) & 1);
                mbar_wait(&a_empty[t], ((it / T) & 1) ^ 1);
                tc_fence_after();
                const uint32_t raw = ring_s + s * kTsStage;
                uint32_t hv[32], lv[32];
                if (o.a_gather) {  // im2col row of output pixel m0 + row, k = k0 .. k0 + 31, from global
                    const int m = g.tm * kBM + row, k0 = g.k0 + kc * kBK;
                    const int hw = o.oh * o.ow;
                    const int img = m / hw, rem = m - img * hw, oy = rem / o.ow, ox = rem - oy * o.ow;
                    int tap = k0 / o.ic, c = k0 - tap * o.ic;
                    int ky = tap / o.ksz, kx = tap - ky * o.ksz;
                    const float* __restrict__ src = o.A;
#pragma unroll
                    for (int q = 0; q < 32; ++q) {
                        const int iy = oy * o.cstride - o.cpad + ky, ix = ox * o.cstride - o.cpad + kx;
                        float x = 0.0f;
                        if (m < o.M && k0 + q < o.K && iy >= 0 && iy < o.ih && ix >= 0 && ix < o.iw)
                            x = __ldg(src + (static_cast<long long>(img * o.ih + iy) * o.iw + ix) * o.ic + c);
                        hv[q] = tc_split_hi(x);
                        lv[q] = tc_split_lo(x, __uint_as_float(hv[q]));
                        if (++c == o.ic) {
                            c = 0;
                            if (++kx == o.ksz) kx = 0, ++ky;
                        }
                    }
                } else if (akm) {  // [128 rows][32 k], 128-byte swizzled rows
#pragma unroll
                    for (int c = 0; c < 8; ++c) {
                        const float4 x = lds128(raw + sw128(row, c));
                        const float xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
                        for (int q = 0; q < 4; ++q) {
                            hv[4 * c + q] = tc_split_hi(xs[q]);
                            lv[4 * c + q] = tc_split_lo(xs[q], __uint_as_float(hv[4 * c + q]));
                        }
                    }
                } else {  // [32 k][128 m]
#pragma unroll
                    for (int k = 0; k < 32; ++k) {
                        const float x = lds32(raw + (k * kBM + row) * 4);
                        hv[k] = tc_split_hi(x);
                        lv[k] = tc_split_lo(x, __uint_as_float(hv[k]));
                    }
                }
                const uint32_t acol = tmem + lane_off + kTsAcol0 + t * 64;
                tmem_st32(acol, hv);
                tmem_st32(acol + 32, lv);
                tmem_st_wait();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&a_full[t]);
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------ MMA issuer
        uint32_t it = 0;
        for (int j = 0; j < ntiles; ++j) {
            if (tiles_sh[j].op < 0) continue;
            const GemmOp& o = ops[tiles_sh[j].op];
            const TileGeo g = tiles_sh[j].g;
            const bool bmn = !o.b_kmajor;
            const uint32_t idesc = instr_desc(o.bn, false, bmn);
            for (int kc = 0; kc < g.nchunks; ++kc, ++it) {
                const int s = it % S, t = it % T, a = it % AC;
                mbar_wait(&op_full[s], (it / S) & 1);
                mbar_wait(&a_full[t], (it / T) & 1);
                if (bsp) mbar_wait(&b_full[s], (it / S) & 1);
                mbar_wait(&acc_empty[a], ((it / AC) & 1) ^ 1);
                tc_fence_after();
                const uint32_t bh = ring_s + s * kTsStage + kTsARaw, bl = bh + kTsBOp;
                const uint32_t ah = tmem + kTsAcol0 + t * 64, al = ah + 32;
                if (elect_one()) {
                    if (bmn) {
                        constexpr uint32_t lbo = 4096, sbo = 512;
                        mma_chunk3_ts(tmem + a * BN, ah, al, smem_desc_mn(bh, lbo, sbo), smem_desc_mn(bl, lbo, sbo), 64,
                                      idesc);
                    } else {
                        mma_chunk3_ts(tmem + a * BN, ah, al, smem_desc(bh), smem_desc(bl), 2, idesc);
                    }
                    mma_commit(&op_empty[s]);
                    mma_commit(&a_empty[t]);
                    mma_commit(&acc_full[a]);
                }
                __syncwarp();
            }
        }
    } else if (warp >= kEpiWarp0 && warp < kEpiWarp0 + 8) {
        // ------------------------------------------------------ drain + epilogue
        const int q = warp & 3, h = (warp - kEpiWarp0) >> 2, et = tid - kEpiWarp0 * 32;
        const uint32_t lane_off = static_cast<uint32_t>(q * 32) << 16;
        int stores = 0;
        uint32_t it = 0;
        // split cursor (bsp launches): the B box of chunk `sit` (tile sj, chunk
        // skc) is split while the drain waits for chunk it; kept kBLead
        // chunks ahead of the drain, so the MMA can run that far ahead
#ifndef PBKD_EXP_BLEAD
        constexpr uint32_t kBLead = 2;
#else
        constexpr uint32_t kBLead = PBKD_EXP_BLEAD;  // diagnosis build
#endif
        int sj = 0, skc = 0;
        uint32_t sit = 0;
        auto split_ahead = [&](uint32_t upto) {  // split chunks sit .. upto-1
            while (sit < upto && sj < ntiles) {
                if (tiles_sh[sj].op < 0 || skc >= tiles_sh[sj].g.nchunks) {
                    ++sj, skc = 0;
                    continue;
                }
                const GemmOp& so = ops[tiles_sh[sj].op];
                const int s = sit % S;
                mbar_wait(&op_full[s], (sit / S) & 1);
                if (so.b_split) {
                    const uint32_t bh = ring_s + s * kTsStage + kTsARaw;
                    split_b_stage(bh, bh + kTsBOp, so.bn, et);
                }
                __syncwarp();
                if (lane == 0) mbar_arrive(&b_full[s]);
                ++skc, ++sit;
            }
        };
        for (int j = 0; j < ntiles; ++j) {
            if (tiles_sh[j].op < 0) continue;
            const GemmOp& o = ops[tiles_sh[j].op];
            const TileGeo g = tiles_sh[j].g;
            const int bnt = o.bn;
            const int hcols = min(HB, max(0, bnt - h * HB));
            float acc[HB];
#pragma unroll
            for (int i = 0; i < HB; ++i) acc[i] = 0.0f;
            for (int kc = 0; kc < g.nchunks; ++kc, ++it) {
                const int a = it % AC;
                if (bsp) split_ahead(it + 1 + kBLead);
                mbar_wait(&acc_full[a], (it / AC) & 1);
                tc_fence_after();
                const uint32_t base = tmem + lane_off + a * BN + h * HB;
#pragma unroll
                for (int c0 = 0; c0 < HB; c0 += 32) {  // hcols is a multiple of 32: one load + wait per 32 columns
                    if (c0 < hcols) tmem_add32(base + c0, acc + c0);
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&acc_empty[a]);
            }
            staged_epilogue<BN, KIND>(o, acc, g.tm, g.tn, g.split, q, h, lane, et, red, cs_s,
                                      ts_staging_blocks<KIND>() > 1 ? cs_s + kBM * 32 * 4 : 0u, stores, bnt);
        }
        if (tid == kEpiWarp0 * 32) tma_store_wait_all();
    }
    tc_fence_before();
    __syncthreads();
#ifdef PBKD_GEMM_TRACE_BUILD
    if (threadIdx.x == 0 && g_ts_trace && blockIdx.x < 1024) {
        g_ts_trace[1024 + blockIdx.x] = gtimer();
        unsigned long long nc = 0, nt = 0;
        for (int j = 0; j < ntiles; ++j)
            if (tiles_sh[j].op >= 0) nc += tiles_sh[j].g.nchunks, ++nt;
        g_ts_trace[2048 + blockIdx.x] = nc | (nt << 32);
    }
#endif
    if (warp == 1) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
    }
}

// ------------------------------------------------------------------- host
namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        PBKD_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (p == nullptr || q != cudaDriverEntryPointSuccess)
            throw CudaError("cuTensorMapEncodeTiled is not available from the driver");
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }();
    return fn;
}

// 2-D fp32 tensor [outer][ld] (inner extent `inner` <= ld), box {bi, bo}.
bool encode(CUtensorMap* m, const float* base, long long inner, long long outer, long long ld, int bi, int bo,
            CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_NONE) {
    if ((reinterpret_cast<uintptr_t>(base) & 15) != 0 || (ld * 4) % 16 != 0 || inner < 1 || outer < 1) return false;
    const cuuint64_t dims[2] = {static_cast<cuuint64_t>(inner), static_cast<cuuint64_t>(outer)};
    const cuuint64_t strides[1] = {static_cast<cuuint64_t>(ld) * 4};
    const cuuint32_t box[2] = {static_cast<cuuint32_t>(bi), static_cast<cuuint32_t>(bo)};
    const cuuint32_t estr[2] = {1, 1};
    const CUresult r = encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box,
                                   estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

int num_sms() {
    static int n = [] {
        int dev = 0, v = 0;
        PBKD_CUDA(cudaGetDevice(&dev));
        PBKD_CUDA(cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev));
        return std::max(1, v);
    }();
    return n;
}

template <int BN, bool PS, int KIND>
void launch_tma_t(const GemmOp* d, int nd, int total, cudaStream_t st, const int* perm) {
    static bool attr = false;
    if (!attr) {
        PBKD_CUDA(cudaFuncSetAttribute(umma_tma_kernel<BN, PS, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       Cfg<BN, PS>::smem));
        attr = true;
    }
    if (nd > kMaxOps) throw CudaError("umma_tma: too many ops in one launch");
    static const int grid_cap = [] {  // diagnosis (tools/gpu_gridcap.sh): cap the persistent grid
        const char* e = std::getenv("PBKD_GEMM_GRID_MAX");
        return e ? std::max(1, std::atoi(e)) : 1 << 30;
    }();
    const int grid = perm ? gemm_tma_grid(total)
                          : std::max({1, std::min({total, num_sms(), grid_cap}), (total + kMaxTiles - 1) / kMaxTiles});
    static const bool trace_on = std::getenv("PBKD_GEMM_TRACE") != nullptr;
    static unsigned long long* trace = nullptr;
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (trace_on) PBKD_CUDA(cudaStreamIsCapturing(st, &cap));
    if (trace_on && cap == cudaStreamCaptureStatusNone && !trace)
        PBKD_CUDA(cudaMalloc(&trace, (10 * 512 + 3 * 1024) * sizeof(unsigned long long)));
    unsigned long long* tr = cap == cudaStreamCaptureStatusNone ? trace : nullptr;
    if (tr) PBKD_CUDA(cudaMemsetAsync(tr, 0, (10 * 512 + 3 * 1024) * sizeof(unsigned long long), st));
    launch_k(umma_tma_kernel<BN, PS, KIND>, dim3(grid), dim3(kThreadsT), static_cast<size_t>(Cfg<BN, PS>::smem), st, d, nd,
             total, tr, perm);
    PBKD_LAUNCH_CHECK();
    static const int trace_from = [] {
        const char* e = std::getenv("PBKD_GEMM_TRACE");
        return e ? std::atoi(e) : 0;
    }();
    static int launch_no = 0;
    if (tr) ++launch_no;
    static const int trace_n = [] {
        const char* e = std::getenv("PBKD_GEMM_TRACE_N");
        return e ? std::atoi(e) : 8;
    }();
    if (tr && launch_no >= trace_from && launch_no < trace_from + trace_n) {  // diagnosis: CTA 0 timeline on stderr
        std::vector<unsigned long long> h(10 * 512 + 3 * 1024);
        PBKD_CUDA(cudaMemcpyAsync(h.data(), trace, h.size() * 8, cudaMemcpyDeviceToHost, st));
        PBKD_CUDA(cudaStreamSynchronize(st));
        const unsigned long long t0 = h[5 * 512];
        auto rel = [&](int ev, int i) { return h[ev * 512 + i] ? static_cast<long long>(h[ev * 512 + i] - t0) : -1LL; };
        std::fprintf(stderr, "[gemm-trace] launch %d BN=%d grid=%d tiles=%d nd=%d setup=%lld ns\n", launch_no, BN, grid,
                     total, nd, rel(5, 1));
        {  // per-CTA: start / end relative to the earliest start, chunks, tiles
            unsigned long long s0 = ~0ull, e1 = 0;
            for (int b = 0; b < grid && b < 1024; ++b) {
                s0 = std::min(s0, h[5120 + b]);
                e1 = std::max(e1, h[5120 + 1024 + b]);
            }
            std::fprintf(stderr, "[gemm-cta] launch %d BN=%d PS=%d grid=%d span %.2f us\n", launch_no, BN, PS ? 1 : 0,
                         grid, (e1 - s0) * 1e-3);
            std::vector<GemmOp> hop(static_cast<size_t>(nd));
            PBKD_CUDA(cudaMemcpy(hop.data(), d, hop.size() * sizeof(GemmOp), cudaMemcpyDeviceToHost));
            for (const GemmOp& o : hop)
                std::fprintf(stderr, "[gemm-cta]   op M=%d N=%d K=%d ksplit=%d tiles=%dx%d epi=%d conv=%d\n", o.M, o.N,
                             o.K, o.ksplit, o.tiles_m, o.tiles_n, o.epi, o.conv);
            for (int b = 0; b < grid && b < 1024; ++b)
                std::fprintf(stderr, "[gemm-cta]   cta %3d start %7.2f end %7.2f chunks %4llu tiles %llu\n", b,
                             (h[5120 + b] - s0) * 1e-3, (h[5120 + 1024 + b] - s0) * 1e-3, h[5120 + 2048 + b] & 0xffffffffull,
                             h[5120 + 2048 + b] >> 32);
        }
        for (int i = 0; i < 512 && h[i]; ++i)
            std::fprintf(stderr, "[gemm-trace]   chunk %3d: tma %8lld raw_full %8lld op_empty %8lld A %8lld B %8lld fence %8lld mma %8lld drain %8lld\n",
                         i, rel(0, i), rel(6, i), rel(7, i), rel(8, i), rel(9, i), rel(1, i), rel(2, i), rel(3, i));
        for (int j = 0; j < 512 && h[4 * 512 + j]; ++j)
            std::fprintf(stderr, "[gemm-trace]   tile %3d epilogue end %8lld\n", j, rel(4, j));
        std::fprintf(stderr, "[gemm-trace]   tile 0 epilogue: staged start %lld passes", rel(9, 0));
        for (int p = 0; p < 4; ++p) std::fprintf(stderr, " %lld", rel(8, p));
        std::fprintf(stderr, "\n");
    }
}

template <int KIND>
void launch_ts_t(const GemmOp* d, int nd, int total, cudaStream_t st, const int* perm) {
    static bool attr = false;
    if (!attr) {
        PBKD_CUDA(cudaFuncSetAttribute(umma_ts_kernel<KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, ts_smem<KIND>()));
        attr = true;
    }
    if (nd > kMaxOps) throw CudaError("umma_ts: too many ops in one launch");
    const int grid = gemm_tma_grid(total);
#ifdef PBKD_GEMM_TRACE_BUILD
    // diagnosis (PBKD_GEMM_TRACE set, uncaptured launches): per-CTA lines in
    // launch_tma_t's [gemm-cta] format (tools/cta_trace_summary.py), launch
    // ids 1000 * kind + n
    static const bool trace_on = std::getenv("PBKD_GEMM_TRACE") != nullptr;
    static unsigned long long* buf = nullptr;
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    if (trace_on) PBKD_CUDA(cudaStreamIsCapturing(st, &cap));
    const bool tr = trace_on && cap == cudaStreamCaptureStatusNone;
    if (tr) {
        if (!buf) PBKD_CUDA(cudaMalloc(&buf, 3 * 1024 * sizeof(unsigned long long)));
        PBKD_CUDA(cudaMemsetAsync(buf, 0, 3 * 1024 * sizeof(unsigned long long), st));
        PBKD_CUDA(cudaMemcpyToSymbolAsync(g_ts_trace, &buf, sizeof(buf), 0, cudaMemcpyHostToDevice, st));
    }
#endif
    launch_k(umma_ts_kernel<KIND>, dim3(grid), dim3(kThreadsT), static_cast<size_t>(ts_smem<KIND>()), st, d, nd, total,
             perm);
    PBKD_LAUNCH_CHECK();
#ifdef PBKD_GEMM_TRACE_BUILD
    if (tr) {
        static int launch_no = 0;
        ++launch_no;
        std::vector<unsigned long long> h(3 * 1024);
        PBKD_CUDA(cudaMemcpyAsync(h.data(), buf, h.size() * 8, cudaMemcpyDeviceToHost, st));
        unsigned long long* none = nullptr;
        PBKD_CUDA(cudaMemcpyToSymbolAsync(g_ts_trace, &none, sizeof(none), 0, cudaMemcpyHostToDevice, st));
        PBKD_CUDA(cudaStreamSynchronize(st));
        unsigned long long s0 = ~0ull, e1 = 0;
        for (int b = 0; b < grid && b < 1024; ++b) s0 = std::min(s0, h[b]), e1 = std::max(e1, h[1024 + b]);
        std::fprintf(stderr, "[gemm-cta] launch %d BN=%d PS=2 grid=%d span %.2f us\n", launch_no + 1000 * KIND, kTsBN, grid,
                     (e1 - s0) * 1e-3);
        std::vector<GemmOp> hop(static_cast<size_t>(nd));
        PBKD_CUDA(cudaMemcpy(hop.data(), d, hop.size() * sizeof(GemmOp), cudaMemcpyDeviceToHost));
        for (const GemmOp& o : hop)
            std::fprintf(stderr, "[gemm-cta]   op M=%d N=%d K=%d ksplit=%d tiles=%dx%d epi=%d conv=%d\n", o.M, o.N, o.K,
                         o.ksplit, o.tiles_m, o.tiles_n, o.epi, o.conv);
        for (int b = 0; b < grid && b < 1024; ++b)
            std::fprintf(stderr, "[gemm-cta]   cta %3d start %7.2f end %7.2f chunks %4llu tiles %llu\n", b, (h[b] - s0) * 1e-3,
                         (h[1024 + b] - s0) * 1e-3, h[2048 + b] & 0xffffffffull, h[2048 + b] >> 32);
    }
#endif
}

}  // namespace

int gemm_tma_grid(int total) {
    static const int grid_cap = [] {  // diagnosis (tools/gpu_gridcap.sh): cap the persistent grid
        const char* e = std::getenv("PBKD_GEMM_GRID_MAX");
        return e ? std::max(1, std::atoi(e)) : 1 << 30;
    }();
    return std::max({1, std::min({total, num_sms(), grid_cap}), (total + kMaxTiles - 1) / kMaxTiles});
}

bool encode_nhwc_box(CUtensorMap* m, const float* base, int n, int h, int w, int c, int bc, int bw, int bh, int bn) {
    static const bool on = [] {
        const char* e = std::getenv("PBKD_DW_TMA");
        return !(e && e[0] == '0');
    }();
    if (!on || base == nullptr || (reinterpret_cast<uintptr_t>(base) & 15) != 0 || c % 4 != 0 || n < 1 || h < 1 ||
        w < 1 || bc < 1 || bw < 1 || bh < 1 || bn < 1 || bc > 256 || bw > 256 || bh > 256 || bn > 256 || (bc * 4) % 16 != 0)
        return false;
    const cuuint64_t dims[4] = {static_cast<cuuint64_t>(c), static_cast<cuuint64_t>(w), static_cast<cuuint64_t>(h),
                                static_cast<cuuint64_t>(n)};
    const cuuint64_t strides[3] = {static_cast<cuuint64_t>(c) * 4, static_cast<cuuint64_t>(w) * c * 4,
                                   static_cast<cuuint64_t>(h) * w * c * 4};
    const cuuint32_t box[4] = {static_cast<cuuint32_t>(bc), static_cast<cuuint32_t>(bw), static_cast<cuuint32_t>(bh),
                               static_cast<cuuint32_t>(bn)};
    const cuuint32_t estr[4] = {1, 1, 1, 1};
    const CUresult r = encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(base), dims, strides, box,
                                   estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// Implicit-im2col A operand of a teacher conv as a 4-D map over the NHWC
// input {C, W, H, N}, box = one tap's 32 channels at the 128 output pixels
// of a tile, traversal stride = conv stride, out-of-image taps zero filled.
// Needs C % 32 == 0 and tiles made of whole output rows (ow | 128 and
// (128/ow) | oh) or whole images (oh*ow | 128).
// M tile of an implicit-GEMM conv: whole output rows of one image (bh rows,
// bh | oh, bh * ow <= 128) or whole images; 0 when no such tile exists.
int conv_tile_rows(const GemmOp& o, int* bh_out, int* bimg_out) {
    const int hw = o.oh * o.ow;
    if (hw > kBM) {
        if (o.ow > kBM) return 0;
        int bh = kBM / o.ow;
        while (bh > 1 && o.oh % bh != 0) --bh;
        *bh_out = bh, *bimg_out = 1;
        return bh * o.ow;
    }
    *bh_out = o.oh, *bimg_out = kBM / hw;
    return *bimg_out * hw;
}

bool encode_conv(CUtensorMap* m, const GemmOp& o, CUtensorMapSwizzle sw = CU_TENSOR_MAP_SWIZZLE_NONE) {
    if (o.ic % kBK != 0 || (reinterpret_cast<uintptr_t>(o.A) & 15) != 0) return false;
    const int hw = o.oh * o.ow;
    int bw = o.ow, bh = 0, bimg = 0;
    if (conv_tile_rows(o, &bh, &bimg) == 0) return false;
    const int s = o.cstride;
    const long long nimg = o.M / hw;
    const cuuint64_t dims[4] = {static_cast<cuuint64_t>(o.ic), static_cast<cuuint64_t>(o.iw),
                                static_cast<cuuint64_t>(o.ih), static_cast<cuuint64_t>(nimg)};
    const cuuint64_t strides[3] = {static_cast<cuuint64_t>(o.ic) * 4, static_cast<cuuint64_t>(o.iw) * o.ic * 4,
                                   static_cast<cuuint64_t>(o.ih) * o.iw * o.ic * 4};
    const cuuint32_t box[4] = {static_cast<cuuint32_t>(kBK), static_cast<cuuint32_t>(bw * s),
                               static_cast<cuuint32_t>(bh * s), static_cast<cuuint32_t>(bimg)};
    const cuuint32_t estr[4] = {1, static_cast<cuuint32_t>(s), static_cast<cuuint32_t>(s), 1};
    if (box[1] > 256 || box[2] > 256 || box[3] > 256) return false;
    const CUresult r = encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, const_cast<float*>(o.A), dims, strides, box,
                                   estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                                   CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

bool gemm_ts_enabled() {  // PBKD_GEMM_TS=0: pre-split planes for A as well
    static const bool on = [] {
        const char* e = std::getenv("PBKD_GEMM_TS");
        return !(e && e[0] == '0');
    }();
    return on;
}

bool gemm_bsplit_enabled() {
    static const bool on = [] {
        const char* e = std::getenv("PBKD_GEMM_BSPLIT");
        return !(e && e[0] == '0');
    }();
    return on && gemm_ts_enabled();
}

bool gemm_presplit_ok(long long ld) {
    static const bool on = [] {
        const char* t = std::getenv("PBKD_GEMM_TMA");
        const char* p = std::getenv("PBKD_PRESPLIT");
        const char* e = std::getenv("PBKD_TF32_TERMS");
        return !(t && t[0] == '0') && !(p && p[0] == '0') && (!e || std::atoi(e) == 3);
    }();
    return on && (ld * 4) % 16 == 0;
}

// Pre-split operands (tf32 hi / lo planes with the operand's own layout and
// leading dimension): 128-byte swizzled boxes land in the MMA's canonical
// SWIZZLE_128B layout (K-major: box {32 K, rows}; MN-major: box {32 MN, 32 K}
// per MN atom) with no conversion pass.  Only with the 3xTF32 split.
bool presplit_pair(CUtensorMap* mh, CUtensorMap* ml, const float* hi, const float* lo, bool kmajor, long long mn,
                   long long k, long long ld, int rows) {
    const auto sw = CU_TENSOR_MAP_SWIZZLE_128B;
    if (kmajor) return encode(mh, hi, k, mn, ld, kBK, rows, sw) && encode(ml, lo, k, mn, ld, kBK, rows, sw);
    const auto sw32 = CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B;  // tf32 MN-major smem layout
    return encode(mh, hi, mn, k, ld, 32, kBK, sw32) && encode(ml, lo, mn, k, ld, 32, kBK, sw32);
}

void presplit_maps(GemmOp& o) {
    o.b_presplit = 0;
    if (o.tf32x3 == 3 && o.b_hi && o.b_lo &&
        presplit_pair(&o.map_bh, &o.map_bl, o.b_hi, o.b_lo, o.b_kmajor != 0, o.N, o.K, o.ldb, o.bn))
        o.b_presplit = 1;
    o.a_presplit = 0;
    if (o.tf32x3 != 3 || !o.a_hi || !o.a_lo) return;
    if (o.conv) {
        GemmOp t = o;
        t.A = o.a_hi;
        if (!encode_conv(&o.map_ah, t, CU_TENSOR_MAP_SWIZZLE_128B)) return;
        t.A = o.a_lo;
        if (!encode_conv(&o.map_al, t, CU_TENSOR_MAP_SWIZZLE_128B)) return;
        o.a_presplit = 1;
    } else if (presplit_pair(&o.map_ah, &o.map_al, o.a_hi, o.a_lo, o.a_kmajor != 0, o.M, o.K, o.lda, kBM)) {
        o.a_presplit = 1;
    }
}

// C written through shared memory + TMA store: 3-D {N, M, ksplit} map with
// 128-byte swizzle (32-column boxes of 128 rows, clipped per split).
bool encode_c(GemmOp& o) {
    if (!o.C || (reinterpret_cast<uintptr_t>(o.C) & 15) != 0 || (o.ldc * 4) % 16 != 0) return false;
    const long long splits = o.epi == 2 ? o.ksplit : 1;
    const cuuint64_t dims[3] = {static_cast<cuuint64_t>(o.N), static_cast<cuuint64_t>(o.M),
                                static_cast<cuuint64_t>(splits)};
    const cuuint64_t strides[2] = {static_cast<cuuint64_t>(o.ldc) * 4, static_cast<cuuint64_t>(o.ldc) * o.M * 4};
    const cuuint32_t box[3] = {32, static_cast<cuuint32_t>(o.bm > 0 ? o.bm : kBM), 1};
    const cuuint32_t estr[3] = {1, 1, 1};
    return encode_fn()(&o.map_c, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, o.C, dims, strides, box, estr,
                       CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                       CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// TMA eligibility + tensor maps (called from gemm_finalize).
bool gemm_tma_prepare(GemmOp& o) {
    const int bn = o.bn;
    if (o.conv) {
        static const bool conv_on = [] {
            const char* e = std::getenv("PBKD_CONV_TMA");
            return !(e && e[0] == '0');
        }();
        if (!conv_on || o.ksplit != 1 || !o.b_kmajor) return false;
        o.a_gather = 0;
        if (o.ic % kBK != 0) {
            // channel counts the im2col boxes cannot address (the 3-channel
            // network input): 128-row tiles over any geometry, A gathered from
            // global by the converter warps of the A-through-TMEM kernel
            // (measured: 2.6x faster than the register-staged kernel for the
            // 3x3 / 3-channel conv, 10% slower for the 7x7 / 3-channel stem,
            // whose 5 gathered K chunks outweigh the MMAs: K <= 64 only)
            if (!(gemm_ts_enabled() && o.a_ts_req && o.tf32x3 == 3 && bn <= kTsBN && o.K <= 2 * kBK)) return false;
            o.bm = kBM;
            if (!encode(&o.map_b, o.B, o.K, o.N, o.ldb, kBK, bn)) return false;
            presplit_maps(o);
            o.a_presplit = 0;
            o.c_tma = encode_c(o) ? 1 : 0;
            if (!o.b_presplit || !o.c_tma) return false;
            o.a_tmem = 1;
            o.a_gather = 1;
            return true;
        }
        int bh = 0, bimg = 0;
        o.bm = conv_tile_rows(o, &bh, &bimg);
        if (o.bm == 0) {
            o.bm = kBM;
            return false;
        }
        if (!(encode_conv(&o.map_a, o) && encode(&o.map_b, o.B, o.K, o.N, o.ldb, kBK, bn))) return false;
        presplit_maps(o);
        o.c_tma = encode_c(o) ? 1 : 0;
        o.a_tmem = 0;
        if (o.c_tma && gemm_ts_enabled() && o.a_ts_req && o.b_presplit && o.tf32x3 == 3 && bn <= kTsBN) {
            CUtensorMap m;  // raw input, 128-byte swizzled im2col boxes for the converter warps
            if (encode_conv(&m, o, CU_TENSOR_MAP_SWIZZLE_128B)) {
                o.map_a = m;
                o.a_tmem = 1;
                o.a_presplit = 0;
            }
        }
        return o.c_tma != 0;
    }
    bool ok = o.a_kmajor ? encode(&o.map_a, o.A, o.K, o.M, o.lda, kBK, kBM) : encode(&o.map_a, o.A, o.M, o.K, o.lda, kBM, kBK);
    ok = ok && (o.b_kmajor ? encode(&o.map_b, o.B, o.K, o.N, o.ldb, kBK, bn) : encode(&o.map_b, o.B, o.N, o.K, o.ldb, bn, kBK));
    if (ok) {
        presplit_maps(o);
        o.c_tma = encode_c(o) ? 1 : 0;
    }
    o.a_tmem = 0;
    o.b_split = 0;
    // raw B without planes: boxes of the planes' geometry and swizzle, split in
    // place (hi) and into the lo plane's slot by the converter warps
    CUtensorMap mb_raw, mb_unused;
    const bool bsplit = ok && !o.b_presplit && o.b_split_req && o.epi != 1 && gemm_bsplit_enabled() &&
                        presplit_pair(&mb_raw, &mb_unused, o.B, o.B, o.b_kmajor != 0, o.N, o.K, o.ldb, o.bn);
    if (ok && gemm_ts_enabled() && o.a_ts_req && (o.b_presplit || bsplit) && o.tf32x3 == 3 && bn <= kTsBN) {
        // raw A for the converter warps: K-major 128-byte swizzled {32 k, 128 rows},
        // MN-major plain {128 m, 32 k}
        CUtensorMap m;
        const bool enc = o.a_kmajor ? encode(&m, o.A, o.K, o.M, o.lda, kBK, kBM, CU_TENSOR_MAP_SWIZZLE_128B)
                                    : encode(&m, o.A, o.M, o.K, o.lda, kBM, kBK);
        if (enc) {
            o.map_a = m;
            o.a_tmem = 1;
            o.a_presplit = 0;
            if (!o.b_presplit) o.map_bh = mb_raw, o.b_split = 1;
        }
    }
    return ok && o.c_tma != 0;  // the TMA kernel's epilogue stores through the C map
}

void tf32_split_host(const float* x, size_t n, float* hi, float* lo) {
    auto rne = [](float v) {
        uint32_t b;
        std::memcpy(&b, &v, 4);
        b = (b + 0xFFFu + ((b >> 13) & 1u)) & 0xFFFFE000u;
        float r;
        std::memcpy(&r, &b, 4);
        return r;
    };
    for (size_t i = 0; i < n; ++i) {
        const float h = rne(x[i]);
        volatile float d = std::isinf(x[i]) ? 0.0f : x[i] - h;  // exact (Sterbenz), no contraction; inf: lo 0
        hi[i] = h;
        lo[i] = rne(d);
    }
}


template <int KIND>
void launch_tma_kind(const GemmOp* d, int nd, int total, int cls, cudaStream_t st, const int* perm) {
    if (cls >= 3 * kGemmClassTma) {  // A through TMEM (kinds 0 / 1)
        if constexpr (KIND == 0 || KIND == 1 || KIND == kGemmKindConv) launch_ts_t<KIND>(d, nd, total, st, perm);
        else throw CudaError("umma_ts: unsupported epilogue kind");
        return;
    }
    switch (cls) {
        case kGemmClassTma + 32: launch_tma_t<32, false, KIND>(d, nd, total, st, perm); break;
        case kGemmClassTma + 64: launch_tma_t<64, false, KIND>(d, nd, total, st, perm); break;
        case kGemmClassTma + 128: launch_tma_t<128, false, KIND>(d, nd, total, st, perm); break;
        case 2 * kGemmClassTma + 32: launch_tma_t<32, true, KIND>(d, nd, total, st, perm); break;
        case 2 * kGemmClassTma + 64: launch_tma_t<64, true, KIND>(d, nd, total, st, perm); break;
        default: launch_tma_t<128, true, KIND>(d, nd, total, st, perm); break;
    }
}

// cls: gemm_bn_class of every op of the launch (kind, pre-split, N tile)
void launch_gemm_tma(const GemmOp* d, int nd, int total, int cls, cudaStream_t st, const int* perm) {
    const int kind = cls / kGemmClassKind, rest = cls % kGemmClassKind;
    switch (kind) {
        case 0: launch_tma_kind<0>(d, nd, total, rest, st, perm); break;
        case 1: launch_tma_kind<1>(d, nd, total, rest, st, perm); break;
        case 2: launch_tma_kind<2>(d, nd, total, rest, st, perm); break;
        default: launch_tma_kind<kGemmKindConv>(d, nd, total, rest, st, perm); break;
    }
}

}  // namespace pbkd_gpu
