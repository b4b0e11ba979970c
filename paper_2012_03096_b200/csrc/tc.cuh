// tc.cuh -- sm_100a tcgen05 / TMEM / mbarrier / TMA helpers shared by the
// GEMM kernels (umma.cu: register-staged, umma_tma.cu: TMA + warp roles).
#pragma once
#include <cuda.h>

#include "common.cuh"

namespace pbkd_gpu {
namespace tc {

constexpr int kBM = 128;       // MMA M (TMEM lanes)
constexpr int kBK = 32;        // fp32 K per stage = one 128-byte swizzle row
constexpr int kRowBytes = 128;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

// Round fp32 to the nearest tf32 (ties to even) with the 13 dropped bits
// cleared, so the MMA's operand read is exact and x - hi is the exact
// remainder.  cvt.rn.tf32.f32 is one F2FP.TF32.F32 instruction on sm_100a
// (cvt.rna is emulated with 4); the mask makes the cleared low bits explicit.
// tools/probes/tf32_cvt.cu checks it against the integer RNE formula
// (b + 0xFFF + ((b >> 13) & 1)) & ~0x1FFF, which the host side uses.
__device__ __forceinline__ uint32_t to_tf32(float x) {
    uint32_t r;
    asm("cvt.rn.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return r & 0xFFFFE000u;
}

// K-major SWIZZLE_128B shared-memory matrix descriptor (sm_100 format):
// start>>4 [0,14), LBO>>4 [16,30) (=1, unused for swizzled K-major),
// SBO>>4 [32,46) (=1024 B between 8-row groups), version 1 [46,48),
// layout type SWIZZLE_128B = 2 at [61,64).
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((addr >> 4) & 0x3FFF);
    d |= static_cast<uint64_t>(1) << 16;
    d |= static_cast<uint64_t>(1024 >> 4) << 32;
    d |= static_cast<uint64_t>(1) << 46;
    d |= static_cast<uint64_t>(2) << 61;
    return d;
}

// MN-major descriptor for 32-bit (tf32) operands.  The only MN-major layout
// the tensor core takes for tf32 is SWIZZLE_128B_BASE32B (layout type 1;
// CUTLASS sm100_common.inl): atoms of 32 MN elements (128 B) x 4 K rows
// (512 B), 32-byte chunks XOR-swizzled by the row; LBO = byte stride between
// MN atoms, SBO = between 4-row K groups (make_umma_desc<Major::MN>).  The
// TMA twin is CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B.
__device__ __forceinline__ uint64_t smem_desc_mn(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= static_cast<uint64_t>((addr >> 4) & 0x3FFF);
    d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
    d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
    d |= static_cast<uint64_t>(1) << 46;
    d |= static_cast<uint64_t>(1) << 61;
    return d;
}

// Byte offset of 16-byte chunk c (0..7) of row r in a K-major SWIZZLE_128B
// tile (rows of 128 bytes, 8-row groups of 1024 bytes).
__device__ __forceinline__ int sw128(int r, int c) { return (r >> 3) * 1024 + (r & 7) * kRowBytes + ((c ^ (r & 7)) << 4); }

// Instruction descriptor: kind::tf32, D fp32, M=128, N=n; A/B K-major unless
// a_mn / b_mn (bits 15 / 16: MN-major operand).
__device__ __forceinline__ uint32_t instr_desc(int n, bool a_mn = false, bool b_mn = false) {
    return (1u << 4) | (2u << 7) | (2u << 10) | (a_mn ? 1u << 15 : 0u) | (b_mn ? 1u << 16 : 0u) |
           (static_cast<uint32_t>(n >> 3) << 17) | (static_cast<uint32_t>(kBM >> 4) << 24);
}

__device__ __forceinline__ void mma_tf32(uint32_t d_tmem, uint64_t a, uint64_t b, uint32_t idesc,
                                         uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(d_tmem),
        "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

// Spin on try_wait without a suspend-time hint: the pipeline hand-offs are
// latency critical (a suspended waiter wakes late).
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@P1 bra DONE_%=;\n\t"
        "bra WAIT_%=;\n"
        "DONE_%=:\n\t}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}

// 2-D TMA tile load global -> shared, completion counted on bar (bytes).
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
        : "memory");
}

// 4-D TMA box load (e.g. an NHWC tile {C, W, H, N}, out-of-range zero filled).
__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2,
                                            int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
        : "memory");
}

__device__ __forceinline__ void prefetch_map(const CUtensorMap* map) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}

__device__ __forceinline__ void fence_async_smem() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void named_bar(int id, int threads) {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

// acc[0..15] += TMEM row (this thread's lane), 16 columns at addr
__device__ __forceinline__ void tmem_add16(uint32_t addr, float* acc) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) acc[i] = __fadd_rn(acc[i], __uint_as_float(r[i]));
}

// acc[0..31] += TMEM row (this thread's lane), 32 columns at addr (one load,
// one wait: half the round trips of two tmem_add16)
__device__ __forceinline__ void tmem_add32(uint32_t addr, float* acc) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
        "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]),
          "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]),
          "=r"(r[24]), "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(addr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) acc[i] = __fadd_rn(acc[i], __uint_as_float(r[i]));
}

__device__ __forceinline__ bool elect_one() {
    uint32_t p;
    asm volatile(
        "{\n\t.reg .pred P;\n\t"
        "elect.sync _|P, 0xffffffff;\n\t"
        "selp.u32 %0, 1, 0, P;\n\t}\n"
        : "=r"(p));
    return p != 0;
}

// One 32-wide K chunk of the 3xTF32 split (hi*lo + lo*hi + hi*hi per 8-wide
// k step, small terms first; the chunk's first MMA overwrites the TMEM slot)
// as a single asm block: 12 tcgen05.mma with descriptors advanced in
// registers, no per-instruction uniform moves or reconvergence.
__device__ __forceinline__ void mma_chunk3d(uint32_t d, uint64_t dah, uint64_t dal, uint64_t dbh, uint64_t dbl,
                                            uint64_t inc_a, uint64_t inc_b, uint32_t idesc) {
    asm volatile(
        "{\n\t"
        ".reg .pred F, T;\n\t"
        ".reg .b64 ah, al, bh, bl;\n\t"
        "setp.ne.b32 F, 0, 0;\n\t"
        "setp.eq.b32 T, 0, 0;\n\t"
        "mov.b64 ah, %1;\n\tmov.b64 al, %2;\n\tmov.b64 bh, %3;\n\tmov.b64 bl, %4;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], ah, bl, %5, F;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], al, bh, %5, T;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], ah, bh, %5, T;\n\t"
        "add.s64 ah, ah, %6;\n\tadd.s64 al, al, %6;\n\tadd.s64 bh, bh, %7;\n\tadd.s64 bl, bl, %7;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], ah, bl, %5, T;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], al, bh, %5, T;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], ah, bh, %5, T;\n\t"
        "add.s64 ah, ah, %6;\n\tadd.s64 al, al, %6;\n\tadd.s64 bh, bh, %7;\n\tadd.s64 bl, bl, %7;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], ah, bl, %5, T;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], al, bh, %5, T;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], ah, bh, %5, T;\n\t"
        "add.s64 ah, ah, %6;\n\tadd.s64 al, al, %6;\n\tadd.s64 bh, bh, %7;\n\tadd.s64 bl, bl, %7;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], ah, bl, %5, T;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], al, bh, %5, T;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], ah, bh, %5, T;\n\t"
        "}\n" ::"r"(d),
        "l"(dah), "l"(dal), "l"(dbh), "l"(dbl), "r"(idesc), "l"(inc_a), "l"(inc_b)
        : "memory");
}

// One 32-wide K chunk of the 3xTF32 split with A in tensor memory (tcgen05
// "ts" form): ah / al = TMEM addresses of the chunk's 32 columns of the A hi /
// lo planes (lane = row, column = k), B from shared-memory descriptors.  Same
// MMA order as mma_chunk3d (hi*lo, lo*hi, hi*hi per 8-wide k step), so the
// accumulated bits match the all-shared-memory form.
__device__ __forceinline__ void mma_chunk3_ts(uint32_t d, uint32_t ah, uint32_t al, uint64_t dbh, uint64_t dbl,
                                              uint64_t inc_b, uint32_t idesc) {
    asm volatile(
        "{\n\t"
        ".reg .pred F, T;\n\t"
        ".reg .b32 ah, al;\n\t"
        ".reg .b64 bh, bl;\n\t"
        "setp.ne.b32 F, 0, 0;\n\t"
        "setp.eq.b32 T, 0, 0;\n\t"
        "mov.b32 ah, %1;\n\tmov.b32 al, %2;\n\tmov.b64 bh, %3;\n\tmov.b64 bl, %4;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah], bl, %5, F;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [al], bh, %5, T;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah], bh, %5, T;\n\t"
        "add.u32 ah, ah, 8;\n\tadd.u32 al, al, 8;\n\tadd.s64 bh, bh, %6;\n\tadd.s64 bl, bl, %6;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah], bl, %5, T;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [al], bh, %5, T;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah], bh, %5, T;\n\t"
        "add.u32 ah, ah, 8;\n\tadd.u32 al, al, 8;\n\tadd.s64 bh, bh, %6;\n\tadd.s64 bl, bl, %6;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah], bl, %5, T;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [al], bh, %5, T;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah], bh, %5, T;\n\t"
        "add.u32 ah, ah, 8;\n\tadd.u32 al, al, 8;\n\tadd.s64 bh, bh, %6;\n\tadd.s64 bl, bl, %6;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah], bl, %5, T;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [al], bh, %5, T;\n\t"
        "tcgen05.mma.cta_group::1.kind::tf32 [%0], [ah], bh, %5, T;\n\t"
        "}\n" ::"r"(d),
        "r"(ah), "r"(al), "l"(dbh), "l"(dbl), "r"(idesc), "l"(inc_b)
        : "memory");
}

// 32 consecutive TMEM columns of this thread's lane <- v[0..31]
__device__ __forceinline__ void tmem_st32(uint32_t addr, const uint32_t* v) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(addr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]), "r"(v[8]), "r"(v[9]),
        "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]),
        "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]),
        "r"(v[28]), "r"(v[29]), "r"(v[30]), "r"(v[31])
        : "memory");
}
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

// K-major SW128 operands: the k-step advances 32 bytes (+2 in the >>4 field).
__device__ __forceinline__ void mma_chunk3(uint32_t d, uint32_t ah, uint32_t al, uint32_t bh, uint32_t bl,
                                           uint32_t idesc) {
    mma_chunk3d(d, smem_desc(ah), smem_desc(al), smem_desc(bh), smem_desc(bl), 2, 2, idesc);
}

// Issue one 32-wide K chunk (4 k-steps of 8) into TMEM column d:
// terms 1: hi*hi; 3: hi*lo + lo*hi + hi*hi (small terms first); 4: + lo*lo.
__device__ __forceinline__ void mma_chunk(uint32_t d, uint32_t ah, uint32_t al, uint32_t bh, uint32_t bl,
                                          uint32_t idesc, int terms) {
    if (terms == 3) {
        mma_chunk3(d, ah, al, bh, bl, idesc);
        return;
    }
#pragma unroll
    for (int kk = 0; kk < kBK / 8; ++kk) {
        const uint32_t off = kk * 32;  // 8 tf32 = 32 bytes along the swizzled row
        if (terms > 1) {
            if (terms > 3) mma_tf32(d, smem_desc(al + off), smem_desc(bl + off), idesc, kk > 0 ? 1u : 0u);
            mma_tf32(d, smem_desc(ah + off), smem_desc(bl + off), idesc, (kk > 0 || terms > 3) ? 1u : 0u);
            mma_tf32(d, smem_desc(al + off), smem_desc(bh + off), idesc, 1u);
            mma_tf32(d, smem_desc(ah + off), smem_desc(bh + off), idesc, 1u);
        } else {
            mma_tf32(d, smem_desc(ah + off), smem_desc(bh + off), idesc, kk > 0 ? 1u : 0u);
        }
    }
}

}  // namespace tc
}  // namespace pbkd_gpu
