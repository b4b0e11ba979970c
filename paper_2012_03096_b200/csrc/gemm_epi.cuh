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
template <int BN, class Sync>
__device__ __forceinline__ void gemm_epilogue(const GemmOp& o, float* acc, int tm, int tn, int split, int q,
                                              int h, int lane, int et, float (*red)[32], Sync sync) {
    constexpr int HB = BN / 2;
    const int m0 = tm * tc::kBM, n0 = tn * BN;
    const int row = m0 + q * 32 + lane;
    const bool row_ok = row < o.M;
    float* C = o.C + (o.epi == 2 ? static_cast<long long>(split) * o.M * o.ldc : 0);
    const bool vec_st = (o.ldc % 4) == 0;
    constexpr int SL = HB >= 16 ? 16 : HB;
#pragma unroll
    for (int c0 = 0; c0 < HB; c0 += SL) {
        float* val = acc + c0;
        const int ncol = n0 + h * HB + c0;
#pragma unroll
        for (int j = 0; j < SL; ++j) {
            const int n = ncol + j;
            float x = val[j];
            if (row_ok && n < o.N) {
                if (o.scale) x = bn_infer_apply(x, o.scale[n], o.shift[n]);
                if (o.skip) x = add(x, o.skip[static_cast<long long>(row) * o.ldc + n]);
                if (o.relu) x = relu(x);
            } else {
                x = 0.0f;
            }
            val[j] = x;
        }
        if (row_ok) {
            float* dst = C + static_cast<long long>(row) * o.ldc + ncol;
            if (vec_st && ncol + SL <= o.N) {
#pragma unroll
                for (int qq = 0; qq < SL / 4; ++qq)
                    reinterpret_cast<float4*>(dst)[qq] =
                        make_float4(val[4 * qq], val[4 * qq + 1], val[4 * qq + 2], val[4 * qq + 3]);
            } else {
#pragma unroll
                for (int j = 0; j < SL; ++j)
                    if (ncol + j < o.N) dst[j] = val[j];
            }
        }
        if (o.epi == 1) {  // per-(m-tile, column) sum / sum of squares, fixed-order trees
#pragma unroll
            for (int j = 0; j < SL; ++j) {
                float s = val[j], sq = val[j] * val[j];
#pragma unroll
                for (int off = 16; off > 0; off >>= 1) {
                    s += __shfl_xor_sync(0xffffffffu, s, off);
                    sq += __shfl_xor_sync(0xffffffffu, sq, off);
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
                if (col < o.N) {
                    const float s = (red[4 * hh][j] + red[4 * hh + 1][j]) + (red[4 * hh + 2][j] + red[4 * hh + 3][j]);
                    const float sq = (red[4 * hh][16 + j] + red[4 * hh + 1][16 + j]) +
                                     (red[4 * hh + 2][16 + j] + red[4 * hh + 3][16 + j]);
                    o.part0[static_cast<long long>(tm) * o.N + col] = s;
                    o.part1[static_cast<long long>(tm) * o.N + col] = sq;
                }
            }
            sync();
        }
    }
}

}  // namespace pbkd_gpu
