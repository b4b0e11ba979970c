#pragma once
// pbkd-b200 host API: the driver-level ops entry points of the reference's
// include/pbkd/ops.hpp (:23-31 conv_out_dim, :243-251 BnCache, :474-514
// softmax cross-entropy, :516-539 MSE loss, :541-558 SGD).  The reference's header-only CPU kernels (conv,
// depthwise, pointwise, batch norm, ...) are not re-exported: on this path
// they run as GPU kernels behind block_forward / block_backward
// (model.hpp).  The float entry points below run on the GPU through the C
// ABI (pbkd_mse_local_loss, pbkd_mse_local_loss_bwd, pbkd_sgd_host); other
// element types are not provided.
#include <cstdint>
#include <span>
#include <string>
#include <vector>

#include "pbkd/tensor.hpp"

namespace pbkd::ops {

inline int conv_out_dim(int in, int kernel, int stride, int pad) {
    const int span = in + 2 * pad - kernel;
    if (span < 0)
        throw ShapeError("conv: kernel " + std::to_string(kernel) + " larger than padded input " +
                         std::to_string(in + 2 * pad));
    const int out = span / stride + 1;
    if (out < 1) throw ShapeError("conv: output dim < 1");
    return out;
}

constexpr double kBnEps = 1e-5;

template <typename T>
struct BnCache {
    Tensor4<T> xhat;
    std::vector<T> inv_std;
};

template <typename T>
T mse_local_loss(const Tensor4<T>& student, const Tensor4<T>& teacher);
template <typename T>
void mse_local_loss_bwd(const Tensor4<T>& student, const Tensor4<T>& teacher, T* gstudent, T scale = T(1));
template <typename T>
T softmax_cross_entropy_fwd(const Tensor4<T>& logits, std::span<const int> labels, Tensor4<T>* probs = nullptr);
template <typename T>
void softmax_cross_entropy_bwd(const Tensor4<T>& probs, std::span<const int> labels, T* glogits, T scale = T(1));
template <typename T>
void sgd_step(std::span<T> weights, std::span<const T> grads, std::span<T> velocity, T lr, T momentum);

template <>
float mse_local_loss<float>(const Tensor4<float>& student, const Tensor4<float>& teacher);
template <>
void mse_local_loss_bwd<float>(const Tensor4<float>& student, const Tensor4<float>& teacher, float* gstudent,
                               float scale);
template <>
float softmax_cross_entropy_fwd<float>(const Tensor4<float>& logits, std::span<const int> labels,
                                       Tensor4<float>* probs);
template <>
void softmax_cross_entropy_bwd<float>(const Tensor4<float>& probs, std::span<const int> labels, float* glogits,
                                      float scale);
template <>
void sgd_step<float>(std::span<float> weights, std::span<const float> grads, std::span<float> velocity, float lr,
                     float momentum);

}  // namespace pbkd::ops
