#pragma once
// pbkd-b200 host API: network graph.  Declarations match the reference's
// include/pbkd/model.hpp:19-214 (tests/cpp compiles reference callers
// against them); the
// implementations live in csrc/host/model.cpp and, for execution, run on the
// GPU behind the C ABI (include/pbkd_b200.h).
#include <array>
#include <cstdint>
#include <functional>
#include <memory>
#include <random>
#include <string>
#include <vector>

#include "pbkd/ops.hpp"
#include "pbkd/tensor.hpp"

struct pbkd_block_cache;  // device-side cache (include/pbkd_b200.h)

namespace pbkd {

struct SpecError : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};

enum class LayerKind {
    Conv3x3,
    Conv1x1,
    DepthwiseConv3x3,
    PointwiseConv,
    BatchNorm,
    ReLU,
    GlobalAvgPool,
    Dense,
    Add,
    // beyond the reference vocabulary (ResNet-50 / ImageNet):
    Conv7x7,     // the 7x7 stride-2 stem convolution
    MaxPool3x3,  // 3x3 stride-2 pad-1 max pooling after the stem
};

const char* layer_kind_name(LayerKind k);
LayerKind layer_kind_from_name(const std::string& name);

struct LayerParams {
    LayerKind kind;
    int in_channels = 0;
    int out_channels = 0;
    int kernel = 0;
    int stride = 1;
    int padding = 0;
    Tensor weight;
    Tensor bias;
    Tensor gamma, beta, moving_mean, moving_var;
};

struct Block {
    std::string name;
    std::string spec_kind;
    bool replaceable = false;
    int in_channels = 0;
    int out_channels = 0;
    int stride = 1;
    int padding = 1;
    std::vector<LayerParams> layers;
};

struct Network {
    std::string name;
    int in_c = 0, in_h = 0, in_w = 0;
    std::vector<Block> blocks;
    Block classifier;
    bool has_classifier() const { return !classifier.layers.empty(); }
};

LayerParams make_conv_layer(LayerKind kind, int in_c, int out_c, int kernel, int stride, int padding);
LayerParams make_batchnorm_layer(int channels);
LayerParams make_relu_layer(int channels);
LayerParams make_gap_layer(int channels);
LayerParams make_dense_layer(int in_features, int out_features);
LayerParams make_add_layer(int in_c, int out_c, int stride);
LayerParams make_maxpool_layer(int channels);

Network parse_model_spec(const std::string& text, const std::string& origin = "<memory>");
Network load_model_spec_file(const std::string& path);

Network subnetwork_prefix(const Network& net, int k, bool inclusive);
std::vector<int> identify_replaceable(const Network& net);

void init_block_weights(Block& b, std::mt19937_64& rng);
void init_weights(Network& net, uint64_t seed);

std::vector<Tensor*> collect_block_trainable(Block& b);
std::vector<Tensor*> collect_trainable(Network& net);

void for_each_array(Network& net, const std::function<void(const std::string&, Tensor&)>& fn);
void for_each_block_array(Block& b, const std::function<void(const std::string&, Tensor&)>& fn);
uint64_t network_weight_hash(const Network& net);

// Shape bookkeeping used by the GPU driver: (c,h,w) at the entrance of block
// k (1-based; k = blocks+1 gives the classifier input).
void block_input_shape(const Network& net, int k, int& c, int& h, int& w);

// ---- execution (model.hpp:134-186 of the reference), on the GPU through
// the C ABI (pbkd_block_forward / pbkd_block_backward, pbkd_prefix_infer).
// A BlockCache keeps the forward's intermediate tensors on the device
// (`device`); `layers` is sized like the block but its host tensors are left
// empty (the reference fills them with host copies, which only its own
// backward reads).
struct LayerCache {
    Tensor input;
    ops::BnCache<float> bn;
};

struct BlockCache {
    bool train_mode = false;
    std::vector<LayerCache> layers;
    std::shared_ptr<pbkd_block_cache> device;
    std::array<int, 4> in_shape{};  // (n, c, h, w) of the block input
};

Tensor block_forward(Block& b, const Tensor& x, bool train, BlockCache* cache = nullptr);
Tensor block_infer(const Block& b, const Tensor& x);
Tensor block_backward(Block& b, const BlockCache& cache, const Tensor& gy, bool need_input_grad,
                      bool param_grads);

struct NetCache {
    std::vector<BlockCache> blocks;
    BlockCache classifier;
};

Tensor network_forward_train(Network& net, const Tensor& x, NetCache& cache,
                             const std::vector<bool>& train_mask = {});
void network_backward(Network& net, const NetCache& cache, const Tensor& glogits,
                      const std::vector<bool>& train_mask = {}, bool freeze_classifier = false);
Tensor network_infer(const Network& net, const Tensor& x);
Tensor prefix_infer(const Network& net, const Tensor& x, int k, bool inclusive);

struct CostRow {
    std::string layer;
    LayerKind kind;
    long long macs = 0;
    long long params = 0;
};

struct CostTable {
    std::vector<CostRow> rows;
    long long total_macs = 0;
    long long total_params = 0;
    long long conv_macs() const;
    long long conv_params() const;
};

CostTable count_block_cost(const Block& b, int c, int h, int w);
CostTable count_macs_params(const Network& net, int c, int h, int w);
CostTable count_macs_params(const Network& net);

}  // namespace pbkd
