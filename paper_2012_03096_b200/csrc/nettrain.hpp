// nettrain.hpp -- whole-network and generic-candidate training on the GPU.
//
// Device-resident loops over NetExec (netexec.hpp) for the parts of the
// reference that train through more than one block:
//   * train_block for any candidate kind (skip kinds included) and for the
//     Combined objective  lambda * MSE + CE through the frozen teacher
//     remainder (distill.cpp:57-84, :135-262);
//   * finetune of an assembled student and train_teacher (distill.cpp:325-441):
//     network_forward_train / network_backward (model.cpp:658-686) with the
//     reference's train masks, softmax cross-entropy, momentum SGD;
//   * evaluate_network / evaluate_with_student_block (distill.cpp:264-295).
// Batches are gathered on the device from the engine's resident dataset; the
// host only shuffles indices (std::shuffle, bit-exact) and reads back scalars.
#pragma once
#include <cstdint>
#include <vector>

#include "engine.hpp"
#include "netexec.hpp"

namespace pbkd_gpu {

struct DevNet {
    std::vector<DevBlock> blocks;
    DevBlock cls;
    bool has_cls = false;
    std::vector<bool> replacement;  // is_replacement_block (replacement.cpp:78-82)
};

// flat: the network's arrays in for_each_array order (host or device)
DevNet make_devnet(NetExec& X, const pbkd::Network& net, const float* flat, bool flat_on_device);
void devnet_to_host(NetExec& X, const DevNet& d, float* flat);

struct DataView {
    const float* images = nullptr;  // device, NCHW
    std::vector<int> labels;        // host copy
    int count = 0, c = 0, h = 0, w = 0, classes = 0;
};

struct FitResult {
    double initial_eval = 0.0, final_eval = 0.0;
    std::vector<double> loss_history;
    std::vector<pbkd::EvalPoint> eval_history;
};

class NetTrainer {
public:
    NetTrainer(NetExec& x, DataView d) : X_(x), d_(std::move(d)) {}
    DTensor images(const std::vector<int>& idx);
    DTensor labels(const std::vector<int>& idx);  // device int32 (in a float-sized buffer)
    // blocks [from, end) then the classifier (when `head`), inference mode
    DTensor infer(DevNet& net, DTensor x, size_t from, bool head);
    double evaluate(DevNet& net, const std::vector<int>& idx, int batch);
    // finetune (teacher_mode false) / train_teacher (true), distill.cpp:325-441
    FitResult fit(DevNet& net, const std::vector<int>& train, const std::vector<int>& eval, int epochs,
                  bool freeze_non_replaced, float lr, float momentum, int batch, uint64_t seed, bool teacher_mode);
    // train_block (distill.cpp:135-262), any kind and loss mode
    TaskOutcome train_block(DevNet& teacher, const pbkd::Network& shape, const pbkd::DistillTask& t,
                            const std::vector<int>& train, const std::vector<int>& eval, bool baseline_and_eval);

private:
    NetExec& X_;
    DataView d_;
};

}  // namespace pbkd_gpu
