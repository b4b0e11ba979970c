// common.cuh -- shared helpers for the pbkd B200 kernels (sm_100a).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

namespace pbkd_gpu {

struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

#define PBKD_CUDA(expr)                                                                     \
    do {                                                                                    \
        cudaError_t e__ = (expr);                                                           \
        if (e__ != cudaSuccess)                                                             \
            throw ::pbkd_gpu::CudaError(std::string("CUDA error ") + cudaGetErrorString(e__) + \
                                        " at " __FILE__ ":" + std::to_string(__LINE__));   \
    } while (0)

#define PBKD_LAUNCH_CHECK() PBKD_CUDA(cudaGetLastError())

constexpr int kThreads = 256;
constexpr int kMaxUnits = 3;

inline int ceil_div(long long a, long long b) { return static_cast<int>((a + b - 1) / b); }

// Programmatic dependent launch: every kernel is launched with programmatic
// stream serialisation (also inside the epoch CUDA graphs), triggers its
// dependents as soon as it starts and waits for its predecessor's results
// (griddepcontrol.wait) before touching global memory, so the next kernel's
// launch and block scheduling overlap this one's tail.  On by default
// (PBKD_PDL=0 disables): VGG-16 epoch 14.7 -> 14.0 ms once the GEMM classes
// were merged into one persistent launch per phase (round 1, with parallel
// class launches, it measured neutral).
bool pdl_enabled();

#ifdef __CUDACC__
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// Every CTA triggers its dependents on entry (a no-op without the launch
// attribute): the next kernel's CTAs are scheduled once this grid's last
// wave is resident, and run their static setup before pdl_wait.
__device__ __forceinline__ void pdl_enter() {
    pdl_trigger();
    pdl_wait();
}

template <typename... KArgs, typename... Args>
void launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, Args... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    PBKD_CUDA(cudaLaunchKernelEx(&cfg, kern, static_cast<KArgs>(args)...));
}
#endif

#ifdef __CUDACC__
// Exact-rounding arithmetic: the reference build has no FMA contraction
// (SURVEY Appendix B), so every elementwise expression that must match it bit
// for bit is spelled with the _rn intrinsics, which nvcc never fuses.
__device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float sub(float a, float b) { return __fsub_rn(a, b); }

// ops.hpp:290-293: y = gamma * ((x - mean) * inv_std) + beta
__device__ __forceinline__ float bn_train_apply(float x, float mean, float inv, float g, float b) {
    return add(mul(g, mul(sub(x, mean), inv)), b);
}
// ops.hpp:304-321 inference affine: y = scale * x + shift
__device__ __forceinline__ float bn_infer_apply(float x, float scale, float shift) {
    return add(mul(scale, x), shift);
}
__device__ __forceinline__ float relu(float x) { return x > 0.0f ? x : 0.0f; }

// tf32 hi part of x: round to nearest even, 13 low bits cleared (one F2FP);
// identical to tc::to_tf32 and tf32_split_host.  lo = hi(x - hi).
__device__ __forceinline__ uint32_t tc_split_hi(float x) {
    uint32_t r;
    asm("cvt.rn.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return r & 0xFFFFE000u;
}
// lo = hi(x - hi); for x = +-inf the remainder inf - inf would be NaN, but
// the fp32 product the split stands for is (+-inf) * b: lo is 0 so that
// hi*b_hi + hi*b_lo + lo*b_hi keeps the infinity (NaN x stays NaN)
__device__ __forceinline__ uint32_t tc_split_lo(float x, float hv) {
    return isinf(x) ? 0u : tc_split_hi(__fsub_rn(x, hv));
}

// Packed fp32x2 arithmetic (FFMA2: two lanes per instruction, each rounded
// exactly like the scalar _rn op).  mul / add / sub are spelled as single
// fma.rn.f32x2 with a -0 addend / a 1 or -1 multiplier; those constants are
// loaded from memory (pk_consts) so that ptxas cannot simplify the fma back
// into a mul + add pair and contract it with a neighbour.
static __device__ __align__(16) float g_pk_consts[4] = {1.0f, -0.0f, -1.0f, 0.0f};  // per translation unit
struct PkConsts {
    float2 one, nz, mone, z;
};
__device__ __forceinline__ PkConsts pk_consts() {
    float a, b, c, d;
    asm volatile("ld.global.nc.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(a), "=f"(b), "=f"(c), "=f"(d) : "l"(g_pk_consts));
    return PkConsts{make_float2(a, a), make_float2(b, b), make_float2(c, c), make_float2(d, d)};
}
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
    float2 d;
    asm("{\n\t.reg .b64 ra, rb, rc, rd;\n\t"
        "mov.b64 ra, {%2, %3};\n\tmov.b64 rb, {%4, %5};\n\tmov.b64 rc, {%6, %7};\n\t"
        "fma.rn.f32x2 rd, ra, rb, rc;\n\t"
        "mov.b64 {%0, %1}, rd;\n\t}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
    return d;
}
// rn(a * b) and rn(a + b), rn(a - b) per lane
__device__ __forceinline__ float2 mul2(const PkConsts& k, float2 a, float2 b) { return fma2(a, b, k.nz); }
__device__ __forceinline__ float2 add2(const PkConsts& k, float2 a, float2 b) { return fma2(a, k.one, b); }
__device__ __forceinline__ float2 sub2(const PkConsts& k, float2 a, float2 b) { return fma2(b, k.mone, a); }

// Which op of a grouped launch owns work item t (ops sorted by cta_begin,
// ops[0].cta_begin == 0).  Must be called by all 32 lanes of a warp with the
// same t: lane l reads ops[l].cta_begin, one ballot -- a single global-load
// latency instead of a chain of nd dependent loads.
template <class Op>
__device__ __forceinline__ int op_index(const Op* __restrict__ ops, int nd, int t) {
    const int lane = static_cast<int>(threadIdx.x & 31);
    int idx = 0;
    for (int base = 0; base < nd; base += 32) {
        const int i = base + lane;
        const bool ge = i < nd && t >= ops[i].cta_begin;
        const unsigned b = __ballot_sync(0xffffffffu, ge);
        idx += __popc(b);
        if (b != 0xffffffffu) break;
    }
    return idx - 1;
}

// Which task of a grouped launch owns this CTA (offs has nd+1 entries).
__device__ __forceinline__ int find_task(const int* __restrict__ offs, int nd, int& local) {
    int t = 0;
    while (t + 1 < nd && static_cast<int>(blockIdx.x) >= offs[t + 1]) ++t;
    local = static_cast<int>(blockIdx.x) - offs[t];
    return t;
}
#endif  // __CUDACC__

}  // namespace pbkd_gpu
