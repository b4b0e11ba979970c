// netexec.hpp -- layer-by-layer execution of any reference block on the GPU.
//
// The grouped engine (engine.cu) runs the hot path: many TwoLayer / ThreeLayer
// students trained against cached teacher boundaries.  Everything else the
// reference does with blocks -- block_forward / block_backward with caches
// (model.cpp:498-656), frozen-teacher remainders with inference-mode batch
// norm (distill.cpp:57-84), whole-network training for fine-tuning and the
// teacher (model.cpp:658-686, distill.cpp:297-394), network inference and
// accuracy (distill.cpp:38-55) -- runs here: each layer is one or a few
// device kernels over NHWC tensors resident in HBM, convolutions and
// pointwise layers on the tcgen05 GEMM (implicit im2col forward, explicit
// im2col + GEMM + ordered col2im gather backward).
//
// Inference arithmetic is the engine's: the same conv / pointwise GEMM and
// the same rounding for batch-norm affine, skip add and ReLU (epilogue order
// relu((scale*x + shift) + skip)), the reference's serial 9-term depthwise
// sum, GAP and dense in the reference's serial order -- so a teacher block or
// a candidate run here gives the engine's bits.  Train-mode statistics and
// weight gradients are fixed-order device reductions (tolerance, like the
// engine).
#pragma once
#include <cuda_runtime.h>

#include <memory>
#include <vector>

#include "pbkd/model.hpp"

namespace pbkd_gpu {

// Device tensor, NHWC fp32 (rows = n*h*w, channels contiguous); shared owner.
struct DTensor {
    std::shared_ptr<float> mem;
    float* p = nullptr;
    int n = 0, c = 0, h = 0, w = 0;
    long long rows() const { return static_cast<long long>(n) * h * w; }
    long long size() const { return rows() * c; }
    explicit operator bool() const { return p != nullptr; }
};

// A block resident on the device.  arrays: for_each_block_array order
// (model.cpp:448-478), the reference layouts; grads / vel: same offsets
// (moving-statistics slots unused).
struct DevBlock {
    struct Layer {
        pbkd::LayerKind kind;
        int cin = 0, cout = 0, k = 0, stride = 1, pad = 0;
        long long w = -1, wn = 0, b = -1, gamma = -1, beta = -1, mm = -1, mv = -1;
        DTensor wk, whi, wlo;  // conv / projection: [cout][k*k][cin] + tf32 planes; depthwise: [9][c];
                               // pointwise: an aligned copy of the weight (GEMM / TMA operand)
    };
    std::vector<Layer> layers;
    DTensor arrays, grads, vel;
    long long n = 0;
    bool derived_ok = false;  // wk / whi / wlo match arrays
    float* at(long long off) const { return arrays.p + off; }
    float* grad_at(long long off) const { return grads.p + off; }
};

struct LayerCacheDev {
    DTensor input;      // the layer's input (model.cpp:505 LayerCache::input)
    DTensor xhat, inv;  // train-mode batch norm (ops.hpp BnCache)
};
struct BlockCacheDev {
    bool train = false;
    std::vector<LayerCacheDev> layers;
};

class NetExec {
public:
    explicit NetExec(cudaStream_t st);
    cudaStream_t stream() const { return st_; }

    DTensor alloc(int n, int c, int h, int w, bool zero = false);
    DTensor upload_nchw(const float* x, int n, int c, int h, int w);  // host NCHW -> NHWC
    void download_nchw(const DTensor& t, float* out);                  // NHWC -> host NCHW
    DTensor gather(const float* images_nchw, const int* idx_dev, int n, int c, int h, int w);
    DTensor upload_ints(const std::vector<int>& v);            // int32 payload
    DTensor take_samples(const DTensor& src, const int* pos_dev, int n);  // out[i] = src sample pos[i]
    DTensor slice_samples(const DTensor& src, int first, int n);          // contiguous samples (copy)
    void put_samples(DTensor& dst, int first, const DTensor& src);

    // block <-> device (arrays in for_each_block_array order)
    // src: the arrays in for_each_block_array order (host or device); null:
    // taken from the block's own tensors (the block always gives the layout)
    DevBlock make_block(const pbkd::Block& b, const float* src = nullptr, bool src_on_device = false);
    void load_arrays(DevBlock& d, const float* host);  // host -> device arrays
    void arrays_to_host(const DevBlock& d, float* host);
    void grads_to_host(const DevBlock& d, float* host);

    DTensor forward(DevBlock& b, const DTensor& x, bool train, BlockCacheDev* cache);
    // model.cpp:559-656: param gradients accumulate into b.grads
    DTensor backward(DevBlock& b, const BlockCacheDev& cache, const DTensor& gy, bool need_gx, bool param_grads);

    // losses (ops.hpp:474-539); scalar results read back to the host
    float mse(const DTensor& s, const DTensor& t);  // the engine's epoch-0 baseline order
    // the engine's training-step loss order (loss_kernel + bn_bwd_fin): the
    // same partitions and trees, so a step loss here equals the grouped path's
    float mse_step(const DTensor& s, const DTensor& t);
    void mse_bwd(const DTensor& s, const DTensor& t, float scale, DTensor& g);  // g += k*(s-t)
    double softmax_ce(const DTensor& logits, const int* labels_dev, DTensor* probs);
    void softmax_ce_bwd(const DTensor& probs, const int* labels_dev, float scale, DTensor& g);
    long long count_correct(const DTensor& logits, const int* labels_dev);  // first-max argmax

    void zero_grads(DevBlock& b);
    void sgd(DevBlock& b, float lr, float momentum);  // trainable tensors only (ops.hpp:545-558)
    void axpy(DTensor& y, const DTensor& x);          // y += x
    void sync();

private:
    void prepare(DevBlock& b);
    void gemm(int M, int N, int K, const float* A, long long lda, bool akm, const float* B, long long ldb,
              bool bkm, float* C, long long ldc, bool accumulate);
    DTensor conv_fwd(DevBlock::Layer& l, const DTensor& x);
    std::pair<DTensor, DTensor> pw_bn_stats(const DTensor& x, const float* w, int cin, int cout, float* y, float* mm,
                                            float* mv);
    void conv_bwd(DevBlock& b, DevBlock::Layer& l, const DTensor& x, const DTensor& gy, DTensor* gx, bool wgrad);
    cudaStream_t st_;
};

}  // namespace pbkd_gpu
