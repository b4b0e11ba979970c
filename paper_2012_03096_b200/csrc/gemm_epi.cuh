// gemm_epi.cuh -- GEMM epilogue shared by the tcgen05 kernels.
//
// 256 epilogue threads = 8 warps: warp (q, h) owns TMEM lane quarter q (tile
// rows 32q..32q+31, one row per lane) and column half h (BN/2 columns), with
// the fp32 accumulator of its row/columns in registers (acc[BN/2]).
//   epi 0: C = acc [teacher conv: y = scale*acc + shift (+ skip), relu]
//   epi 1: C = acc, plus per-(m-tile, column) sum and sum of squares for the
//          batch-norm statistics (ops.hpp:273-283), fixed-order trees
//   epi 2: split-K partial, C + split*M*ldc
#pragma once
#include "ops.cuh"
#include "tc.cuh"

namespace pbkd_gpu {

// sync(): barrier over the 256 epilogue threads.  red: [8][32] shared floats.
// The op's fields are copied to registers first: the C stores could alias the
// descriptor as far as the compiler knows, which would force a reload of every
// field after every store.
template <int BN, class Sync>
__device__ __forceinline__ void gemm_epilogue(const GemmOp& op, float* acc, int tm, int tn, int split, int q,
                                              int h, int lane, int et, float (*red)[32], Sync sync) {
    constexpr int HB = BN / 2;
    const int M = op.M, N = op.N, epi = op.epi, relu_on = op.relu;
    const long long ldc = op.ldc;
    const float* __restrict__ scale = op.scale;
    const float* __restrict__ shift = op.shift;
    const float* __restrict__ skip = op.skip;
    float* __restrict__ part0 = op.part0;
    float* __restrict__ part1 = op.part1;
    const int m0 = tm * tc::kBM, n0 = tn * BN;
    const int row = m0 + q * 32 + lane;
    const bool row_ok = row < M;
    float* __restrict__ C = op.C + (epi == 2 ? static_cast<long long>(split) * M * ldc : 0);
    float* __restrict__ Ch = op.c_hi;  // tf32 planes of the output for the next GEMM
    float* __restrict__ Cl = op.c_lo;
    const bool vec_st = (ldc % 4) == 0;
    constexpr int SL = HB >= 16 ? 16 : HB;
#pragma unroll
    for (int c0 = 0; c0 < HB; c0 += SL) {
        float* val = acc + c0;
        const int ncol = n0 + h * HB + c0;
        if (scale || skip || relu_on) {
#pragma unroll
            for (int j = 0; j < SL; ++j) {
                const int n = ncol + j;
                float x = val[j];
                if (row_ok && n < N) {
                    if (scale) x = bn_infer_apply(x, __ldg(scale + n), __ldg(shift + n));
                    if (skip) x = add(x, __ldg(skip + static_cast<long long>(row) * ldc + n));
                    if (relu_on) x = relu(x);
                }
                val[j] = x;
            }
        }
#pragma unroll
        for (int j = 0; j < SL; ++j)
            if (!(row_ok && ncol + j < N)) val[j] = 0.0f;
        if (row_ok) {
            const long long off = static_cast<long long>(row) * ldc + ncol;
            float* dst = C + off;
            if (vec_st && ncol + SL <= N) {
#pragma unroll
                for (int qq = 0; qq < SL / 4; ++qq)
                    reinterpret_cast<float4*>(dst)[qq] =
                        make_float4(val[4 * qq], val[4 * qq + 1], val[4 * qq + 2], val[4 * qq + 3]);
            } else {
#pragma unroll
                for (int j = 0; j < SL; ++j)
                    if (ncol + j < N) dst[j] = val[j];
            }
            if (Ch) {
#pragma unroll
                for (int j = 0; j < SL; ++j)
                    if (ncol + j < N) {
                        const float hv = __uint_as_float(tc_split_hi(val[j]));
                        Ch[off + j] = hv;
                        Cl[off + j] = __uint_as_float(tc_split_lo(val[j], hv));
                    }
            }
        }
        if (epi == 1) {  // per-(m-tile, column) sum / sum of squares, fixed-order trees
#pragma unroll
            for (int j = 0; j < SL; ++j) {
                float s = val[j], sq = __fmul_rn(val[j], val[j]);
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) {
                    s = __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, off));
                    sq = __fadd_rn(sq, __shfl_xor_sync(0xffffffffu, sq, off));
                }
                if (lane == 0) {
                    red[h * 4 + q][j] = s;
                    red[h * 4 + q][16 + j] = sq;
                }
            }
            sync();
            if (et < 2 * SL) {  // column (half hh, j): 4 row quarters in order
                const int hh = et / SL, j = et % SL;
                const int col = n0 + hh * HB + c0 + j;
                if (col < N) {
                    const float s = __fadd_rn(__fadd_rn(red[4 * hh][j], red[4 * hh + 1][j]),
                                              __fadd_rn(red[4 * hh + 2][j], red[4 * hh + 3][j]));
                    const float sq = __fadd_rn(__fadd_rn(red[4 * hh][16 + j], red[4 * hh + 1][16 + j]),
                                               __fadd_rn(red[4 * hh + 2][16 + j], red[4 * hh + 3][16 + j]));
                    part0[static_cast<long long>(tm) * N + col] = s;
                    part1[static_cast<long long>(tm) * N + col] = sq;
                }
            }
            sync();
        }
    }
}

}  // namespace pbkd_gpu
