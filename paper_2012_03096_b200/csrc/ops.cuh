// ops.cuh -- operation descriptors for the grouped (multi-task) kernels.
//
// Every kernel of the student step runs as ONE launch for all distillation
// tasks resident on the GPU: the host writes an array of per-task descriptors
// (each carrying its own first-CTA index `cta_begin`), the kernel maps
// blockIdx.x to its task with find_task().  Tiling and reduction partitions
// depend only on a task's own shape, never on which other tasks share the
// launch, so a block's bits do not depend on the schedule (the GPU analogue of
// test_runtime.cpp:206-253).
//
// Layout: activations are channels-last (NHWC) rows; a "row" is one pixel of
// one sample, channels contiguous.  Depthwise weights are tap-major [9][C];
// pointwise weights keep the reference's [C_out][C_in] (model.cpp:157-171).
#pragma once
#include <cuda.h>

#include "common.cuh"

namespace pbkd_gpu {

// Spatial tiling of the depthwise kernels: a CTA owns `ni` images x `th`
// output rows x all columns x 32 channels, staged (with the 1-pixel halo,
// zero padded) in shared memory as [pixel][32 channels].  Depends only on the
// op's own shape (schedule-independent partials).
struct DwTile {
    int ni, th;         // images, output rows per tile
    int tiles_y, tiles; // row tiles per image group, spatial tiles
    int cslices;        // 32-channel slices
    int tr, tw;         // staged input rows / cols (halo included)
    int xsh;            // log2 of the x segments per output row (packed kernels)
};
DwTile dw_tile(int n, int ho, int wo, int c, int stride, int arrays);

// Depthwise 3x3 forward (ops.hpp:114-147), optional fused prologue that
// rebuilds the input from the previous unit's pointwise output:
//   pro 0: x as stored
//   pro 1: relu(gamma*((x-mean)*inv)+beta)   (train-mode BN, ops.hpp:290-293)
//   pro 2: relu(scale*x+shift)               (inference-mode BN, ops.hpp:304-321)
struct DwFwdOp {
    const float* x;
    const float* w;  // [9][c]
    float* y;        // fp32 output, or (y_hi, y_lo) tf32 planes when set
    float *y_hi, *y_lo;
    int n, h, wd, c, ho, wo, stride, pad;
    int pro;
    int y_both;  // with planes, also the fp32 output (a GEMM taking A through TMEM reads it)
    const float *pa, *pb, *pc, *pd;  // mean,inv,gamma,beta | scale,shift
    const int* failed;
    int cta_begin;
    // optional gather: batch image i is image rows[i] of x (nsrc images), e.g.
    // a teacher boundary buffer read in the task's epoch order
    const int* rows;
    int nsrc;
    DwTile tile;  // set by dw_fwd_finalize
    int tma;      // x tile staged by one 4-D TMA box (dw_fwd_finalize), else cp.async
    CUtensorMap map_x;
};

// Depthwise 3x3 backward of a stride-1 unit u>0 (ops.hpp:149-178) fused with
// the ReLU (ops.hpp:387-393) and the batch-norm partial sums (ops.hpp:333-342)
// of the previous unit:  gx -> gy_prev = gx * [y_prev > 0], partial sums
// sum(gy_prev), sum(gy_prev * xhat_prev) and the weight gradient partials.
struct DwBwdOp {
    const float* gy;     // [rows][c] gradient wrt the dw output
    const float* xp;     // previous unit's pointwise output (pre-BN)
    const float* w;      // [9][c]
    float* gyprev;       // [rows][c] gradient wrt previous BN output (masked)
    float* part_gk;      // [ctas][9][c]
    float* part_sg;      // [ctas][c]
    float* part_sgx;     // [ctas][c]
    const float *mean, *inv, *gamma, *beta;  // previous unit BN (train mode)
    int n, h, wd, c;
    int ctas, rows_per;  // ctas: partial rows (= spatial tiles, dw_bwd_finalize)
    const int* failed;
    int cta_begin;
    DwTile tile;
    int tma;  // gy / xp tiles staged by 4-D TMA boxes (dw_bwd_finalize)
    CUtensorMap map_g, map_x;
};

// Depthwise weight-gradient partials only (unit 0, any stride; model.cpp:570
// skips gx for the first layer).
struct DwGkOp {
    const float* gy;  // [n*ho*wo][c]
    const float* x;   // [n*h*wd][c]
    float* part_gk;   // [ctas][9][c]
    int n, h, wd, c, ho, wo, stride, pad;
    int ctas, rows_per;  // ctas: partial rows (= spatial tiles, dw_gk_finalize)
    const int* failed;
    int cta_begin;
    const int* rows;  // optional gather of x images (as DwFwdOp)
    int nsrc;
    DwTile tile;
    int tma;  // x / gy tiles staged by 4-D TMA boxes (dw_gk_finalize)
    CUtensorMap map_x, map_g;
};

// Sum `parts` rows of width `width` in fixed order into out (optionally
// through a per-element op).  Used for dw gk partials and split-K GEMM.
struct ReduceOp {
    const float* part;
    float* out;
    float* out2;  // optional second copy of the sums (e.g. sum_g -> sg and gbeta)
    int parts, width;
    int layout;  // 0: out[i] = sum ; 1: dw [9][c] -> out [9][c] (same)
    const int* failed;
    int cta_begin;
};

// Generic fp32 GEMM  C[m][n] = sum_k A(m,k) * B(n,k)
//   A(m,k) = a_kmajor ? A[m*lda+k] : A[k*lda+m]   (or implicit conv, see conv)
//   B(n,k) = b_kmajor ? B[n*ldb+k] : B[k*ldb+n]
// epi 0: store C; 1: store C and per-(m-tile, column) partial sum / sum of
// squares for batch-norm statistics; 2: split-K partial: C + split*M*ldc.
// conv != 0: A is the implicit im2col of an NHWC input (teacher conv,
// ops.hpp:37-75): k = tap*ic + j.  Teacher epilogue: y = scale*acc + shift
// (+ skip), then optional relu (model.cpp:540-546, ops.hpp:460-466).
struct GemmOp {
    int M, N, K;
    const float* A;
    long long lda;
    int a_kmajor;
    const float* B;
    long long ldb;
    int b_kmajor;
    float* C;
    long long ldc;
    int epi;
    float *part0, *part1;
    int ksplit, kchunk;
    int tiles_m, tiles_n;
    int conv, ih, iw, ic, oh, ow, ksz, cstride, cpad;
    const float *scale, *shift, *skip;
    int relu;
    int bn;              // N tile (multiple of 16, <= 256), set by gemm_finalize
    int bm;              // M rows per tile: 128, or fewer for an implicit-GEMM conv whose
                         // tiles are whole output rows / images (gemm_tma_prepare)
    int tf32x3, tf32x1;  // 3xTF32 split (fp32 parity, default) or plain TF32
    const int* failed;
    int cta_begin;
    int tma;             // 1: umma_tma.cu kernel (tensor maps below valid)
    // optional pre-split operands: tf32 hi / lo planes (RNE split, same
    // layout and leading dimension as A / B; for conv, as the NHWC input).
    // The TMA kernel loads them straight into its MMA operand ring.
    const float *a_hi, *a_lo, *b_hi, *b_lo;
    int a_presplit, b_presplit;   // set by gemm_finalize when usable
    float *c_hi, *c_lo;           // optional tf32 planes of the output (epi 0)
    CUtensorMap map_a, map_b;     // 2-D fp32 maps of A and B (64-byte aligned)
    CUtensorMap map_ah, map_al;   // SWIZZLE_128B maps of the planes
    CUtensorMap map_bh, map_bl;
    // a_ts_req (caller): A is valid raw fp32 (not only planes); gemm_finalize
    // then sets a_tmem when the A-through-TMEM kernel takes the op (B pre-split)
    int a_ts_req, a_tmem;
    // b_split_req (caller): B has no planes, only raw fp32; when the
    // A-through-TMEM kernel takes the op, its converter warps split the raw B
    // box in shared memory (b_split set; map_bh then addresses raw B)
    int b_split_req, b_split;
    int a_gather;  // a_tmem conv with ic % 32 != 0: converter warps gather the im2col rows from global
    int c_tma;                    // epilogue stores C through shared memory + TMA
    CUtensorMap map_c;            // 3-D {N, M, ksplit} SWIZZLE_128B map of C
};

// tf32 hi/lo split on the host, bit-identical to tc::to_tf32 on the device
// (round to nearest even, 13 low bits cleared): hi = rne(x), lo = rne(x - hi).
void tf32_split_host(const float* x, size_t n, float* hi, float* lo);

// Fills tiling fields (bn, tiles, kchunk/ksplit) of a GemmOp (umma.cu).
void gemm_finalize(GemmOp& o);
// Launch class of o: N tile (32/64/128), + kGemmClassTma for the TMA kernel.
constexpr int kGemmClassTma = 1000;
// TMA kernels are specialised per launch kind (class + kind * kGemmClassKind):
// 0 plain store (dgrad, inference), 1 store + batch-norm partials (fwd),
// 2 split-K partials (wgrad), 3 teacher conv (im2col + BN affine / skip /
// ReLU / output planes); each kernel carries only its kind's code
constexpr int kGemmClassKind = 10000;
constexpr int kGemmKindConv = 3;
int gemm_bn_class(const GemmOp& o);
bool gemm_tma_prepare(GemmOp& o);  // umma_tma.cu: tensor maps, false if ineligible
// Whether GEMM operands with leading dimension `ld` (floats) will be consumed
// as pre-split tf32 planes (TMA kernel on, 3xTF32, 16-byte rows): producers
// then write planes instead of fp32.
bool gemm_presplit_ok(long long ld);
// Whether ops flagged a_ts_req run on the A-through-TMEM kernel (PBKD_GEMM_TS)
bool gemm_ts_enabled();
// Whether raw-B ops (b_split_req) are split in the A-through-TMEM kernel
// (PBKD_GEMM_BSPLIT, default on with PBKD_GEMM_TS): producers then skip the
// B operand's planes
bool gemm_bsplit_enabled();

// Batch-norm statistics from the GEMM column partials (ops.hpp:273-299):
// mean, var = E[x^2]-mean^2 clamped, inv_std, moving-stat update.
struct BnStatOp {
    const float *part_sum, *part_sq;
    int tiles, c;
    long long m;  // rows in the batch
    float *mean, *inv, *mm, *mv;
    int update_moving;
    const int* failed;
    int cta_begin;
};

// Last unit: student output s = relu(bn(p)), loss partials sum (s-t)^2 and
// batch-norm backward partials of g = [y>0] * k*(s-t) (ops.hpp:518-539,
// 387-393, 333-342).  rows/ctas partition fixed per task shape.
struct LossOp {
    const float* p;
    const float* t;
    const float *mean, *inv, *gamma, *beta;
    float* part_sg;
    float* part_sgx;
    float* part_loss;  // [ctas]
    int rows, c, ctas, rows_per;
    float kmse;        // (scale*2)/count
    const int* failed;
    int cta_begin;
    const int* trows;  // optional gather of t: sample i is sample trows[i] (srow elements each)
    long long srow;
};

// Reduce batch-norm backward partials -> sum_g, sum_gx, parameter gradients
// (ggamma += sum_gx, gbeta += sum_g; ops.hpp:343-344); for the last unit also
// the step loss, its non-finite check (distill.cpp:236-244) and failure flag.
struct BnBwdFinOp {
    const float *part_sg, *part_sgx, *part_loss;
    int ctas, c;
    float *sg, *sgx, *ggamma, *gbeta;
    float* loss_out;   // nullptr unless last unit
    double count;      // elements in the MSE
    int* failed;       // written when loss is non-finite
    int cta_begin;
};

// g_p = (gamma*inv) * ((g - inv_m*sum_g) - (xhat*inv_m)*sum_gx)  (ops.hpp:345-354)
// with g either read (gin) or rebuilt from (p, t) for the last unit.
struct BnBwdApplyOp {
    const float* p;
    const float* t;    // non-null -> last unit, g rebuilt from the MSE gradient
    const float* gin;  // else the masked gradient from the dw backward
    float* gout;       // fp32 output, or (gout_hi, gout_lo) tf32 planes when set
    float *gout_hi, *gout_lo;
    const float *mean, *inv, *gamma, *beta, *sg, *sgx;
    long long total;   // rows*c
    int c;
    float inv_m, kmse;
    const int* failed;
    int cta_begin;
    const int* trows;  // optional gather of t (as LossOp)
    long long srow;
};

// Momentum SGD over a task's flat parameter buffer (ops.hpp:545-558).
struct SgdOp {
    float *w, *v;
    const float* g;
    long long n;
    float lr, mom;
    const int* failed;
    int cta_begin;
    float *w_hi, *w_lo;  // optional tf32 planes of the updated w (GEMM operands)
};

// dst row pos[i] <- src row i   (activation streaming into a task's epoch order);
// kScatterCtas CTAs per op
constexpr int kScatterCtas = 148;
// dst row pos[r] = src row r.  cd > 0: rows are pixels x cs channels in src
// and pixels x cd channels in dst (cd > cs; the extra channels are left as
// they are: zeroed by the owner once)
struct ScatterOp {
    const float* src;
    float* dst;
    const int* pos;
    int rows, width;
    int cs, cd;
    int cta_begin;
};

// Host-side helpers (defined in ops.cu) ------------------------------------
int rows_part_ctas(long long rows, int c);  // deterministic partition size
int rows_part_per(long long rows, int ctas);

void launch_dw_fwd(const DwFwdOp* d_ops, int nd, int ctas, cudaStream_t st);
void launch_dw_bwd(const DwBwdOp* d_ops, int nd, int ctas, cudaStream_t st);
void launch_dw_gk(const DwGkOp* d_ops, int nd, int ctas, cudaStream_t st);
void launch_reduce(const ReduceOp* d_ops, int nd, int ctas, cudaStream_t st);
// ctas: the ops' total tile count (sum of ctas_gemm); cls: gemm_bn_class
// perm (optional, TMA classes): tile slots of the persistent grid -- CTA b
// takes slots b, b + G, b + 2G, ... (G = gemm_tma_grid(tiles)), slot -> tile id
// or -1; tiles = G * slots per CTA.  Null: slot = tile (round robin).
void launch_gemm_bn(const GemmOp* d_ops, int nd, int ctas, int cls, cudaStream_t st, const int* perm = nullptr);
void launch_gemm_tma(const GemmOp* d_ops, int nd, int tiles, int cls, cudaStream_t st,
                     const int* perm = nullptr);  // cls: gemm_bn_class
int gemm_tma_grid(int tiles);  // persistent grid of a TMA GEMM launch over `tiles` tile slots
void launch_bn_stat(const BnStatOp* d_ops, int nd, int ctas, cudaStream_t st);
void launch_loss(const LossOp* d_ops, int nd, int ctas, cudaStream_t st);       // c <= 1024
void launch_loss_wide(const LossOp* d_ops, int nd, int ctas, cudaStream_t st);  // any c (channel passes)
void launch_bn_bwd_fin(const BnBwdFinOp* d_ops, int nd, int ctas, cudaStream_t st);
void launch_bn_bwd_apply(const BnBwdApplyOp* d_ops, int nd, int ctas, cudaStream_t st);
void launch_sgd(const SgdOp* d_ops, int nd, int ctas, cudaStream_t st);
void launch_scatter(const ScatterOp* d_ops, int nd, int ctas, cudaStream_t st);

// CTA counts for one op (host)
int ctas_dw_fwd(const DwFwdOp& o);
int ctas_reduce(const ReduceOp& o);
int ctas_dw_bwd(const DwBwdOp& o);
int ctas_dw_gk(const DwGkOp& o);
// fill the tile geometry (and partial-row count `ctas` for bwd / gk)
// 4-D map {C, W, H, N} over an NHWC fp32 tensor, box {bc, bw, bh, bn},
// out-of-range elements zero filled (umma_tma.cu); false if TMA cannot
// address it (16-byte alignment, C % 4, box limits).
bool encode_nhwc_box(CUtensorMap* m, const float* base, int n, int h, int w, int c, int bc, int bw, int bh, int bn);
void dw_fwd_finalize(DwFwdOp& o);
void dw_bwd_finalize(DwBwdOp& o);
void dw_gk_finalize(DwGkOp& o);
int ctas_gemm(const GemmOp& o);
int ctas_elem(long long total);  // bn_bwd_apply
int ctas_sgd(long long n);
int ctas_cols(int c);  // bn_stat / bn_bwd_fin CTAs per task

// Non-grouped helpers used by evaluation / teacher / tests -----------------
void launch_gather_nhwc(const float* images_nchw, const int* idx, int n, int c, int h, int w,
                        float* out_nhwc, cudaStream_t st);
void launch_bn_infer_prep(const float* gamma, const float* beta, const float* mm,
                          const float* mv, int c, float* scale, float* shift, cudaStream_t st);
void launch_bn_infer_relu(const float* x, float* y, long long total, int c, const float* scale,
                          const float* shift, cudaStream_t st);
// teacher conv weights [cout][cin][kk] -> [cout][kk][cin] + tf32 planes
void launch_conv_weight_prep(const float* raw, int cout, int cin, int kk, int kp, float* w, float* hi, float* lo,
                             cudaStream_t st);
// 3x3 / stride 2 / pad 1 max pooling over NHWC (the ResNet-50 stem, SURVEY
// 8f-4): out-of-image taps are skipped; optional tf32 planes of the output
void launch_maxpool3x3(const float* x, float* y, float* y_hi, float* y_lo, int n, int h, int w, int c,
                       cudaStream_t st);
// its backward: each input pixel gathers gy of the outputs whose first
// maximum (ky, kx order) it is, in ascending output order (deterministic)
void launch_maxpool3x3_bwd(const float* x, const float* gy, float* gx, int n, int h, int w, int c,
                           cudaStream_t st);
// tf32 hi / lo planes of n floats (the 3xTF32 operand split)
void launch_tf32_split(const float* x, long long n, float* hi, float* lo, cudaStream_t st);
// per-segment MSE sums (segment = one batch of the epoch-0 baseline)
void launch_mse_segments(const float* s, const float* t, long long seg_elems, long long total,
                         int nseg, double* out_sums, cudaStream_t st);
// classifier head: GAP -> [relu] -> dense -> argmax (first max) == label
void launch_classifier_count(const float* x_nhwc, int n, int hw, int c, const int* layer_kinds,
                             int nlayers, const float* dense_w, const float* dense_b, int nout,
                             const int* labels, int* correct, cudaStream_t st);

}  // namespace pbkd_gpu
