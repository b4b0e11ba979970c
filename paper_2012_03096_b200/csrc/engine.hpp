// engine.hpp -- the per-GPU distillation engine behind the C ABI.
//
// One Engine owns one device.  run() executes a set of distillation tasks
// (pbkd::DistillTask, distill.hpp:24-37) with train_block semantics
// (distill.cpp:135-262) for every task, all tasks of the same batch size and
// unit count advancing in lockstep as grouped launches:
//
//   once per run: teacher forward over the training split, every block
//               boundary kept in HBM in train order (replaces prefix_infer +
//               block_infer per block per batch, distill.cpp:210-211)
//   per epoch:  ceil(N/B) grouped student steps (fwd, MSE, bwd, SGD) reading
//               their batches through the epoch order
//   the whole epoch is one CUDA graph; the host only uploads the epoch's
//   permutation (std::shuffle + mt19937_64, bit-exact).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>
#include <functional>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "pbkd/distill.hpp"
#include "pbkd/model.hpp"

namespace pbkd_gpu {

class NetExec;
class NcclComm;
class NetTrainer;
struct DevNet;

struct TaskOutcome {
    int block_index = 0;
    std::string kind;
    bool failed = false;
    std::string failure;
    std::vector<float> best_block;   // for_each_block_array order (empty if none)
    std::vector<float> final_block;  // weights after the last executed step
    std::vector<pbkd::EvalPoint> eval_history;
    std::vector<double> loss_history;
    std::vector<float> step_losses;
    double final_local_loss = 0.0;
    double best_eval = -1.0;
    double wall_time_s = 0.0;
};

struct RunOptions {
    bool baseline_and_eval = true;  // epoch-0 baseline + evaluations (train_block semantics)
    bool use_graphs = true;
    // device events bracket epochs [timed_from_epoch, last]; for a step-only
    // run with timed_from_epoch <= 1 the window also holds the one-time
    // teacher boundary pass
    int timed_from_epoch = 1;
    // Sample-sharded teacher (multi-GPU).  global_blocks lists every block
    // being distilled on any rank with its owner; this engine trains only the
    // tasks passed to run() (owner == rank), runs the teacher forward once on
    // its shard of the training split for every boundary any block reads,
    // and exchanges boundary rows with NCCL (set_comm) once per run.
    // virtual_shards > 1 on a single GPU computes the boundaries shard by
    // shard (tests: results must not move a bit).
    std::vector<std::pair<int, int>> global_blocks;  // (block index, owner rank)
    int virtual_shards = 1;
    std::vector<double> shard_share;  // teacher share per rank (empty: uniform)
    // after the last epoch, replay that epoch's program (and the teacher
    // boundary pass) once more eagerly with a CUDA event after every launch
    // (per-kernel-class device time and algorithmic work, RunTiming::prof);
    // the training state is saved before and restored after the replay
    bool profile = false;
};

// Per kernel class of a profiled epoch: launches, device ms (events on the
// engine stream), algorithmic bytes / flops of those launches.
struct KernelStat {
    int launches = 0;
    double ms = 0.0, bytes = 0.0, flops = 0.0;
};

// Timing of the last run (device events around the epoch graphs).
struct RunTiming {
    double epoch_ms_total = 0.0;  // sum over training epochs (teacher pass + steps)
    std::vector<double> epoch_ms; // per training epoch (graph only)
    double timed_ms = 0.0;        // events around epochs >= timed_from_epoch, host gaps included
    int timed_epochs = 0;
    double teacher_ms = 0.0;      // the run's one-time teacher boundary pass (+ NCCL exchange)
    bool timed_includes_teacher = false;  // timed window began before the teacher pass
    int epochs = 0;
    long long student_steps = 0;  // per task
    long long launches = 0;       // kernel launches in the timed window
    std::map<std::string, KernelStat> prof;  // RunOptions::profile
};

class Engine {
public:
    explicit Engine(int device);
    ~Engine();
    Engine(const Engine&) = delete;
    Engine& operator=(const Engine&) = delete;

    void set_teacher(const pbkd::Network& net);
    void set_teacher(pbkd::Network&& net);
    // flat: the same weights in for_each_array order (one H2D copy from it)
    void set_teacher(pbkd::Network&& net, const float* flat, size_t n);
    // Moves the loaded teacher network (host tensors) out of the engine, which
    // then holds no teacher until the next set_teacher: a reload with the same
    // spec refills these tensors instead of parsing and allocating anew.
    pbkd::Network take_teacher();
    const pbkd::Network& teacher() const;
    bool has_teacher() const;
    void set_dataset(const float* images, const int* labels, int count, int c, int h, int w,
                     int classes, bool images_on_device = false);
    std::vector<TaskOutcome> run(const std::vector<pbkd::DistillTask>& tasks,
                                 const std::vector<int>& train_idx,
                                 const std::vector<int>& eval_idx, const RunOptions& opt);
    const RunTiming& timing() const;
    // validate_task (distill.cpp:86-100) and the split checks of train_block
    // (distill.cpp:144-145, dataset.cpp:166-179) with the reference's messages
    void validate(const pbkd::DistillTask& t) const;
    void check_split(const std::vector<int>& train_idx, const std::vector<int>& eval_idx) const;

    // Inference helpers (host NCHW in/out), used by the C ABI.
    pbkd::Tensor prefix_infer(const pbkd::Tensor& x, int k, bool inclusive);
    pbkd::Tensor candidate_infer(const pbkd::Block& cand, const pbkd::Tensor& x);
    double eval_with_student(int block_index, const pbkd::Block& student,
                             const std::vector<int>& eval_idx);
    // Times one representative launch of a hot kernel in isolation (CUDA
    // events on the engine stream).  which: 0 teacher conv implicit GEMM,
    // 1 student pointwise GEMM (fwd), 2 depthwise fwd, 3 depthwise bwd
    // (fused), 4 loss + batch-norm backward sums.  Shapes: the teacher block
    // with the most MACs, `batch` samples.
    void bench_kernel(int which, int batch, int iters, double* ms, double* bytes, double* flops);

    // Layer-by-layer executor on this engine's stream (netexec.hpp), a trainer
    // over the resident dataset (nettrain.hpp) and the resident teacher as a
    // device network.  Each call makes this engine's device current.
    NetExec& exec();
    NetTrainer trainer();
    DevNet& teacher_net();

    int device() const;
    cudaStream_t stream() const;
    // join an NCCL communicator (id from nccl_unique_id on rank 0)
    void set_comm(const char* nccl_id128, int rank, int world);
    void set_comm(std::unique_ptr<NcclComm> comm);  // a member of an in-process clique
    int comm_rank() const;
    int comm_world() const;

    struct Impl;

private:
    std::unique_ptr<Impl> impl_;
};

// Flat conversions between pbkd::Block (reference array order / layouts) and
// the engine's device layout ([9][C] depthwise, [Cout][Cin] pointwise).
int candidate_units(const pbkd::Block& b);

}  // namespace pbkd_gpu
