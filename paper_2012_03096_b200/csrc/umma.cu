// umma.cu -- tcgen05 / TMEM GEMM for sm_100a (pointwise convs, teacher
// implicit-GEMM conv, weight gradients).
//
//   C[m][n] = sum_k A(m,k) * B(n,k),   fp32 in / fp32 out
//
// Tensor-core path: kind::tf32 MMAs (M=128, N=BN<=128, K=8) issued by one
// elected thread; accumulators live in TMEM and are read back with tcgen05.ld.
//
// fp32 parity (north_star: 1e-4 relative) with TF32 tensor cores:
//  * 3xTF32 split  a*b ~= a_hi*b_hi + a_hi*b_lo + a_lo*b_hi  (hi = tf32
//    round-to-nearest, lo = tf32 of the exact remainder);
//  * per-chunk drain: every 32-wide K chunk accumulates into its own TMEM slot
//    (two slots, double buffered) and the chunk results are summed in fp32
//    registers in chunk order.  Measured on B200, letting one TMEM accumulator
//    absorb all K/8 MMA steps loses ~K/8 * 2^-23 (biased rounding inside the
//    MMA); the drain keeps every accumulator short and the cross-chunk sum
//    round-to-nearest (tools/prec_probe.py: K=512 GEMM error 1.3e-5 vs 1.9e-5
//    for numpy fp32).
//
// 256 threads: two threads per tile row stage 16 of the chunk's 32 K values
// each (global -> registers -> shared, into the canonical K-major
// SWIZZLE_128B layout: row r at (r/8)*1024 + (r%8)*128 bytes, 16-byte chunk c
// at ((c ^ r%8) * 16)); the 8 warps split the TMEM drain and the epilogue by
// column halves (a warp may only touch TMEM lanes 32*(warp%4)..+31).  Register
// staging lets one kernel gather an implicit im2col (teacher conv), transpose
// MN-major sources (dgrad/wgrad) and split hi/lo, with no host relayout.
// Two smem stages / TMEM slots: threads refill and drain slot s^1 while the
// tensor core works on slot s.
#include <algorithm>
#include <cstdlib>

#include "gemm_epi.cuh"
#include "ops.cuh"
#include "tc.cuh"

namespace pbkd_gpu {

namespace {

using namespace tc;
constexpr int kKH = 16;   // K values staged per thread (half a row)
constexpr int kStages = 2;
constexpr int kThreadsG = 256;

// Store 16 K values (chunks h*4..h*4+3 of row r) as tf32 hi / lo.
__device__ __forceinline__ void put_half(uint8_t* hi, uint8_t* lo, int r, int h, const float* v, bool split) {
#pragma unroll
    for (int cc = 0; cc < 4; ++cc) {
        const int c = h * 4 + cc;
        uint32_t hv[4], lv[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const float x = v[cc * 4 + q];
            hv[q] = to_tf32(x);
            lv[q] = split && !isinf(x) ? to_tf32(__fsub_rn(x, __uint_as_float(hv[q]))) : 0u;
        }
        const int off = sw128(r, c);
        *reinterpret_cast<uint4*>(hi + off) = make_uint4(hv[0], hv[1], hv[2], hv[3]);
        if (split) *reinterpret_cast<uint4*>(lo + off) = make_uint4(lv[0], lv[1], lv[2], lv[3]);
    }
}

__device__ __forceinline__ void zero16(float* v) {
#pragma unroll
    for (int i = 0; i < kKH; ++i) v[i] = 0.0f;
}

__device__ __forceinline__ void load16_kmajor(const float* __restrict__ row, int k0, int kend, bool vec, float* v) {
    if (vec && k0 + kKH <= kend) {
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            const float4 q = __ldg(reinterpret_cast<const float4*>(row + k0) + c);
            v[4 * c] = q.x, v[4 * c + 1] = q.y, v[4 * c + 2] = q.z, v[4 * c + 3] = q.w;
        }
    } else {
#pragma unroll
        for (int i = 0; i < kKH; ++i) v[i] = (k0 + i < kend) ? __ldg(row + k0 + i) : 0.0f;
    }
}

// MN-major source X(r, k) = X[k*ld + r]: lanes of a warp read consecutive r
__device__ __forceinline__ void load16_mnmajor(const float* __restrict__ base, long long ld, int r, int k0,
                                               int kend, float* v) {
#pragma unroll
    for (int i = 0; i < kKH; ++i) v[i] = (k0 + i < kend) ? __ldg(base + static_cast<long long>(k0 + i) * ld + r) : 0.0f;
}

// A(m, k0..k0+15) into v[16]
__device__ __forceinline__ void load_a(const GemmOp& o, int m, int k0, int kend, float* v) {
    if (m >= o.M) {
        zero16(v);
        return;
    }
    if (o.conv) {
        const int ox = m % o.ow, t2 = m / o.ow;
        const int oy = t2 % o.oh, n = t2 / o.oh;
        if (o.ic % kKH == 0) {  // the 16 k values lie inside one tap: one 64-byte run
            const int tap = k0 / o.ic, j0 = k0 - tap * o.ic;
            const int ky = tap / o.ksz, kx = tap - ky * o.ksz;
            const int iy = oy * o.cstride - o.cpad + ky, ix = ox * o.cstride - o.cpad + kx;
            if (k0 >= kend || iy < 0 || iy >= o.ih || ix < 0 || ix >= o.iw) {
                zero16(v);
                return;
            }
            const float* p = o.A + ((static_cast<long long>(n) * o.ih + iy) * o.iw + ix) * o.ic + j0;
#pragma unroll
            for (int c = 0; c < 4; ++c) {
                const float4 q = __ldg(reinterpret_cast<const float4*>(p) + c);
                v[4 * c] = q.x, v[4 * c + 1] = q.y, v[4 * c + 2] = q.z, v[4 * c + 3] = q.w;
            }
            return;
        }
#pragma unroll
        for (int i = 0; i < kKH; ++i) {
            const int k = k0 + i;
            float x = 0.0f;
            if (k < kend) {
                const int tap = k / o.ic, j = k - tap * o.ic;
                const int ky = tap / o.ksz, kx = tap - ky * o.ksz;
                const int iy = oy * o.cstride - o.cpad + ky, ix = ox * o.cstride - o.cpad + kx;
                if (iy >= 0 && iy < o.ih && ix >= 0 && ix < o.iw)
                    x = __ldg(o.A + ((static_cast<long long>(n) * o.ih + iy) * o.iw + ix) * o.ic + j);
            }
            v[i] = x;
        }
        return;
    }
    if (o.a_kmajor)
        load16_kmajor(o.A + static_cast<long long>(m) * o.lda, k0, kend, (o.lda % 4) == 0, v);
    else
        load16_mnmajor(o.A, o.lda, m, k0, kend, v);
}

__device__ __forceinline__ void load_b(const GemmOp& o, int n, int k0, int kend, float* v) {
    if (n >= o.N) {
        zero16(v);
        return;
    }
    if (o.b_kmajor)
        load16_kmajor(o.B + static_cast<long long>(n) * o.ldb, k0, kend, (o.ldb % 4) == 0, v);
    else
        load16_mnmajor(o.B, o.ldb, n, k0, kend, v);
}

template <class Op>
__device__ __forceinline__ const Op& op_of_u(const Op* ops, int nd, int& local) {
    const int t = op_index(ops, nd, static_cast<int>(blockIdx.x));
    local = static_cast<int>(blockIdx.x) - ops[t].cta_begin;
    return ops[t];
}

}  // namespace

// BN: N tile of this launch (16..128, multiple of 16), compile time so the
// per-row fp32 sums stay in registers.
template <int BN>
__global__ void __launch_bounds__(kThreadsG, 1) umma_gemm_kernel(const GemmOp* __restrict__ ops, int nd) {
    pdl_enter();
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    __shared__ uint64_t bars[kStages];
    __shared__ uint32_t tmem_base_sh;
    __shared__ float red[8][32];
    int local;
    const GemmOp& o = op_of_u(ops, nd, local);
    if (o.failed != nullptr && *o.failed != 0) return;

    // 1024-byte aligned carve-up: [stage][A_hi | A_lo | B_hi | B_lo]
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    constexpr int a_bytes = kBM * kRowBytes;
    constexpr int b_bytes = BN * kRowBytes;
    constexpr int stage_bytes = 2 * a_bytes + 2 * b_bytes;
    constexpr int tmem_cols = (2 * BN <= 32) ? 32 : (2 * BN <= 64) ? 64 : (2 * BN <= 128) ? 128 : 256;
    constexpr int HB = BN / 2;  // columns per warp half in drain / epilogue (>= 8)

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int row_t = tid & (kBM - 1), half = tid >> 7;  // staging: row, K half
    const int wq = warp & 3, wh = warp >> 2;               // TMEM lane quarter, column half
    const int tiles_mn = o.tiles_m * o.tiles_n;
    const int split = local / tiles_mn;
    const int rem = local - split * tiles_mn;
    const int tm = rem / o.tiles_n, tn = rem - tm * o.tiles_n;
    const int m0 = tm * kBM, n0 = tn * BN;
    const int kbeg = split * o.kchunk;
    const int kend = min(o.K, kbeg + o.kchunk);
    const int nchunks = max(1, (kend - kbeg + kBK - 1) / kBK);
    const int terms = o.tf32x3;  // 1: tf32, 3: hi*hi+hi*lo+lo*hi, 4: + lo*lo
    const bool split3 = terms > 1;

    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base_sh)),
                     "r"(tmem_cols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    if (tid == 0) {
        for (int s = 0; s < kStages; ++s) mbar_init(&bars[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base_sh;
    const uint32_t idesc = instr_desc(BN);
    const uint32_t lane_off = static_cast<uint32_t>(wq * 32) << 16;

    float acc[HB];
#pragma unroll
    for (int j = 0; j < HB; ++j) acc[j] = 0.0f;
    auto drain = [&](int kc) {  // chunk kc's slot into acc, in chunk order
        mbar_wait(&bars[kc & 1], (kc >> 1) & 1);
        tc_fence_after();
        const uint32_t base = tmem + lane_off + (kc & 1) * BN + wh * HB;
        static_assert(HB % 16 == 0, "BN >= 32");
#pragma unroll
        for (int c0 = 0; c0 < HB; c0 += 16) tmem_add16(base + c0, acc + c0);
        tc_fence_before();
    };

    float v[kKH];
    for (int kc = 0; kc < nchunks; ++kc) {
        const int s = kc & 1;
        const int k0 = kbeg + kc * kBK + half * kKH;
        uint8_t* st = smem + s * stage_bytes;
        uint8_t *a_hi = st, *a_lo = st + a_bytes, *b_hi = st + 2 * a_bytes, *b_lo = st + 2 * a_bytes + b_bytes;
        if (kc >= kStages) drain(kc - kStages);  // frees smem stage s and TMEM slot s
        load_a(o, m0 + row_t, k0, kend, v);
        put_half(a_hi, a_lo, row_t, half, v, split3);
        if (row_t < BN) {
            load_b(o, n0 + row_t, k0, kend, v);
            put_half(b_hi, b_lo, row_t, half, v, split3);
        }
        fence_async_smem();
        __syncthreads();
        if (warp == 0) {
            tc_fence_after();
            if (lane == 0) {
                const uint32_t ah = smem_u32(a_hi), al = smem_u32(a_lo), bh = smem_u32(b_hi), bl = smem_u32(b_lo);
                mma_chunk(tmem + s * BN, ah, al, bh, bl, idesc, terms);
                mma_commit(&bars[s]);
            }
            __syncwarp();
        }
    }
    for (int kc = max(0, nchunks - kStages); kc < nchunks; ++kc) drain(kc);

    // ------------------------------------------------------------ epilogue
    // thread = (row wq*32+lane, columns wh*HB .. +HB)
    gemm_epilogue<BN>(o, acc, tm, tn, split, wq, wh, lane, tid, red, [] { __syncthreads(); });
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(tmem_cols));
}

// ------------------------------------------------------------------- host
namespace {
// N tile: 32 / 64 / 128.  (PBKD_BN64=0 folds the 64 class into the 128
// launches: one launch per step phase fewer, measured 2% slower on VGG-16.)
int bn_for(int n) {
    static const bool bn64 = [] {
        const char* e = std::getenv("PBKD_BN64");
        return !(e && e[0] == '0');
    }();
    if (n <= 32) return 32;
    if (n <= 64 && bn64) return 64;
    return 128;
}
}  // namespace

void gemm_finalize(GemmOp& o) {
    if (o.ksplit < 1) o.ksplit = 1;
    if (o.ksplit == 1) {
        o.kchunk = ((o.K + kBK - 1) / kBK) * kBK;
    } else {
        o.kchunk = ((ceil_div(o.K, o.ksplit) + kBK - 1) / kBK) * kBK;
        o.ksplit = ceil_div(o.K, o.kchunk);
    }
    // PBKD_BN64_K=<k>: run tiles whose K range is >= k on 64-wide N tiles (4
    // operand stages instead of 3, twice the tiles).  Measured on the VGG-16
    // epoch (tools/gpu_ab_env.sh, k = 64..512): neutral for the student GEMMs
    // and 22% slower teacher convs, so off by default.  Same bits either way.
    static const int longk = [] {
        const char* e = std::getenv("PBKD_BN64_K");
        return e ? std::atoi(e) : 0;
    }();
    o.bn = bn_for(o.N);
    if (o.bn == 128 && longk > 0 && o.kchunk >= longk) o.bn = 64;
    o.bm = kBM;
    o.tiles_m = ceil_div(o.M, kBM);
    o.tiles_n = ceil_div(o.N, o.bn);
    if (o.tf32x3 == 0) {  // parity mode: split fp32 into tf32 hi+lo
        static const int terms = [] {
            const char* e = std::getenv("PBKD_TF32_TERMS");
            return e ? std::atoi(e) : 3;
        }();
        o.tf32x3 = terms;
    }
    // TMA + warp-specialised kernel for the plain (non-conv) GEMMs whose
    // operands satisfy the tensor-map constraints (16-byte aligned rows);
    // PBKD_GEMM_TMA=0 forces the register-staged kernel
    static const bool tma_on = [] {
        const char* e = std::getenv("PBKD_GEMM_TMA");
        return !(e && e[0] == '0');
    }();
    o.tma = (tma_on && gemm_tma_prepare(o)) ? 1 : 0;
    if (!o.tma) o.bm = kBM;  // the register-staged kernel tiles by 128 rows
    o.tiles_m = ceil_div(o.M, o.bm);
}

int ctas_gemm(const GemmOp& o) { return o.tiles_m * o.tiles_n * o.ksplit; }
// + kGemmClassTma: TMA kernel; + 2 kGemmClassTma: TMA kernel, both operands pre-split
int gemm_bn_class(const GemmOp& o) {
    if (!o.tma) return o.bn;
    const int kind = o.conv ? kGemmKindConv : o.epi;
    // pre-split student ops of every N tile share one launch of the 128-wide
    // kernel (per-op MMA width, B box and epilogue passes): one launch per
    // phase instead of a parallel section of 1-CTA-per-SM persistent kernels
    // queueing for the SMs.  PBKD_GEMM_MERGE=0: one launch per N tile.
    static const bool merge = [] {
        const char* e = std::getenv("PBKD_GEMM_MERGE");
        return !(e && e[0] == '0');
    }();
    // Plain stores (epi 0) and split-K partial stores (epi 2) share kernel
    // kind 0 (the store's split coordinate is 0 without split-K), so a
    // unit's dgrad and wgrad can run as one launch.
    if (o.a_tmem)  // A through TMEM (umma_ts_kernel), one launch per phase
        return 128 + 3 * kGemmClassTma + (kind == 2 ? 0 : kind) * kGemmClassKind;
    if (merge && !o.conv && o.a_presplit && o.b_presplit)
        return 128 + 2 * kGemmClassTma + (kind == 2 ? 0 : kind) * kGemmClassKind;
    return o.bn + kGemmClassTma + (o.a_presplit && o.b_presplit ? kGemmClassTma : 0) + kind * kGemmClassKind;
}

template <int BN>
static void launch_bn_t(const GemmOp* d, int nd, int ctas, cudaStream_t st) {
    constexpr size_t smem = 1024 + kStages * (2 * kBM * kRowBytes + 2 * BN * kRowBytes);
    static bool attr = false;
    if (!attr) {
        PBKD_CUDA(cudaFuncSetAttribute(umma_gemm_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem)));
        attr = true;
    }
    launch_k(umma_gemm_kernel<BN>, dim3(ctas), dim3(kThreadsG), smem, st, d, nd);
    PBKD_LAUNCH_CHECK();
}

// All ops of one launch share the N tile and the kernel (the caller groups
// ops by gemm_bn_class; narrower ops would pad their B rows with zeros).
void launch_gemm_bn(const GemmOp* d, int nd, int ctas, int cls, cudaStream_t st, const int* perm) {
    if (cls % kGemmClassKind >= kGemmClassTma) {
        launch_gemm_tma(d, nd, ctas, cls, st, perm);
        return;
    }
    switch (bn_for(cls)) {
        case 32: launch_bn_t<32>(d, nd, ctas, st); break;
        case 64: launch_bn_t<64>(d, nd, ctas, st); break;
        default: launch_bn_t<128>(d, nd, ctas, st); break;
    }
}


}  // namespace pbkd_gpu
