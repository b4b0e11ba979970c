// ref_shim.cpp -- TEST INFRASTRUCTURE ONLY.
//
// Exposes the UNMODIFIED reference library (/root/reference/proj/src/*.cpp,
// compiled beside this file by oracle/Makefile with -Dpbkd=pbkd_ref) through the
// C ABI in oracle_api.h with the ref_ prefix.  Every function below is a thin
// adapter over the reference's public API; no arithmetic is done here.
#define ORC(name) ref_##name
#include "oracle_api.h"

#include <algorithm>
#include <cstring>
#include <random>
#include <span>
#include <string>
#include <vector>

#include "pbkd/dataset.hpp"
#include "pbkd/distill.hpp"
#include "pbkd/model.hpp"
#include "pbkd/runtime.hpp"
#include "pbkd/ops.hpp"
#include "pbkd/replacement.hpp"
#include "pbkd/scheduler.hpp"
#include "pbkd/weights_io.hpp"

using namespace pbkd;

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

Network load_teacher(const char* spec, const float* tw) {
    Network net = parse_model_spec(spec, "spec");
    if (tw) {
        size_t at = 0;
        for_each_array(net, [&](const std::string&, Tensor& t) {
            std::copy(tw + at, tw + at + t.data.size(), t.data.begin());
            at += t.data.size();
        });
    }
    return net;
}

size_t flatten_block(Block& b, float* out, size_t cap) {
    size_t at = 0;
    for_each_block_array(b, [&](const std::string&, Tensor& t) {
        if (out && at + t.data.size() <= cap) std::copy(t.data.begin(), t.data.end(), out + at);
        at += t.data.size();
    });
    if (out && at > cap) throw std::length_error("output buffer too small");
    return at;
}

void load_block(Block& b, const float* in) {
    size_t at = 0;
    for_each_block_array(b, [&](const std::string&, Tensor& t) {
        std::copy(in + at, in + at + t.data.size(), t.data.begin());
        at += t.data.size();
    });
}

Dataset to_dataset(const orc_dataset* d) {
    Dataset ds;
    ds.c = d->c;
    ds.h = d->h;
    ds.w = d->w;
    ds.classes = d->classes;
    ds.images.assign(d->images, d->images + static_cast<size_t>(d->count) * d->c * d->h * d->w);
    ds.labels.assign(d->labels, d->labels + d->count);
    return ds;
}

SplitIndices to_split(const orc_split* s) {
    SplitIndices sp;
    sp.train_idx.assign(s->train_idx, s->train_idx + s->n_train);
    sp.eval_idx.assign(s->eval_idx, s->eval_idx + s->n_eval);
    return sp;
}

DistillTask to_task(const orc_task* t) {
    DistillTask dt;
    dt.block_index = t->block_index;
    dt.kind = static_cast<CandidateKind>(t->kind);
    dt.epochs = t->epochs;
    dt.eval_every = t->eval_every;
    dt.seed = t->seed;
    dt.threshold = t->threshold;
    dt.loss_mode = static_cast<LossMode>(t->loss_mode);
    dt.lambda_local = t->lambda_local;
    dt.lr = t->lr;
    dt.momentum = t->momentum;
    dt.batch_size = t->batch_size;
    dt.max_steps = static_cast<long>(t->max_steps);
    return dt;
}

Tensor wrap(const float* p, int n, int c, int h, int w) {
    Tensor t(n, c, h, w);
    std::copy(p, p + t.size(), t.data.begin());
    return t;
}

void plan_out(const SchedulePlan& p, int* out_ids, int* out_counts) {
    int at = 0;
    for (size_t w = 0; w < p.assignments.size(); ++w) {
        out_counts[w] = static_cast<int>(p.assignments[w].size());
        for (int id : p.assignments[w]) out_ids[at++] = id;
    }
}
}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

uint64_t ref_mix_seed(uint64_t a, uint64_t b) { return mix_seed(a, b); }

void ref_shuffle(int* idx, int n, uint64_t seed) {
    std::mt19937_64 rng(seed);
    std::shuffle(idx, idx + n, rng);
}

int ref_stratified_split(const int* labels, int n, double frac, uint64_t seed, int* train_out,
                         int* n_train, int* eval_out, int* n_eval) {
    return guard([&] {
        Dataset d;
        d.labels.assign(labels, labels + n);
        SplitIndices s = stratified_split(d, frac, seed);
        std::copy(s.train_idx.begin(), s.train_idx.end(), train_out);
        std::copy(s.eval_idx.begin(), s.eval_idx.end(), eval_out);
        *n_train = static_cast<int>(s.train_idx.size());
        *n_eval = static_cast<int>(s.eval_idx.size());
    });
}

int ref_synthetic_dataset(int count, uint64_t seed, int threads, float* images, int* labels) {
    return guard([&] {
        Dataset d = make_synthetic_dataset(count, seed, threads);
        std::copy(d.images.begin(), d.images.end(), images);
        std::copy(d.labels.begin(), d.labels.end(), labels);
    });
}

int ref_round_robin(const int* ids, int n, int workers, int* out_ids, int* out_counts) {
    return guard([&] {
        plan_out(round_robin(std::vector<int>(ids, ids + n), workers), out_ids, out_counts);
    });
}

int ref_wfd(const int* ids, const double* weights, int n, int workers, int* out_ids,
            int* out_counts, double* mk) {
    return guard([&] {
        std::vector<TaskWeight> tw;
        for (int i = 0; i < n; ++i) tw.push_back({ids[i], weights[i]});
        SchedulePlan p = wfd_bin_pack(tw, workers);
        plan_out(p, out_ids, out_counts);
        *mk = p.predicted_makespan;
    });
}

int ref_teacher_num_floats(const char* spec, size_t* n) {
    return guard([&] {
        Network net = parse_model_spec(spec, "spec");
        size_t at = 0;
        for_each_array(net, [&](const std::string&, Tensor& t) { at += t.data.size(); });
        *n = at;
    });
}

int ref_teacher_num_blocks(const char* spec, int* n) {
    return guard([&] { *n = static_cast<int>(parse_model_spec(spec, "spec").blocks.size()); });
}

int ref_teacher_init(const char* spec, uint64_t seed, float* out, size_t cap) {
    return guard([&] {
        Network net = parse_model_spec(spec, "spec");
        init_weights(net, seed);
        size_t at = 0;
        for_each_array(net, [&](const std::string&, Tensor& t) {
            if (at + t.data.size() > cap) throw std::length_error("teacher buffer too small");
            std::copy(t.data.begin(), t.data.end(), out + at);
            at += t.data.size();
        });
    });
}

int ref_block_macs(const char* spec, int k, long long* macs) {
    return guard([&] {
        Network net = parse_model_spec(spec, "spec");
        const CostTable table = count_macs_params(net);
        const std::string prefix = net.blocks.at(static_cast<size_t>(k) - 1).name + "/";
        long long s = 0;
        for (const CostRow& r : table.rows)
            if (r.layer.rfind(prefix, 0) == 0) s += r.macs;
        *macs = s;
    });
}

int ref_candidate_num_floats(int kind, int c_in, int c_out, int stride, size_t* n) {
    return guard([&] {
        ReplacementBlock r = build_candidate(static_cast<CandidateKind>(kind), c_in, c_out, stride, 0);
        *n = flatten_block(r.block, nullptr, 0);
    });
}

int ref_build_candidate(int kind, int c_in, int c_out, int stride, uint64_t seed, float* out,
                        size_t cap) {
    return guard([&] {
        ReplacementBlock r =
            build_candidate(static_cast<CandidateKind>(kind), c_in, c_out, stride, seed);
        flatten_block(r.block, out, cap);
    });
}

void ref_dw_fwd(const float* x, int n, int c, int h, int w, const float* k, int kk, int stride,
                int pad, float* y) {
    Tensor t = ops::depthwise_conv2d_fwd(wrap(x, n, c, h, w), wrap(k, c, 1, kk, kk), stride, pad);
    std::copy(t.data.begin(), t.data.end(), y);
}

void ref_dw_bwd(const float* x, int n, int c, int h, int w, const float* k, int kk, int stride,
                int pad, const float* gy, float* gx, float* gk) {
    const int ho = ops::conv_out_dim(h, kk, stride, pad), wo = ops::conv_out_dim(w, kk, stride, pad);
    ops::depthwise_conv2d_bwd(wrap(x, n, c, h, w), wrap(k, c, 1, kk, kk), wrap(gy, n, c, ho, wo),
                              stride, pad, gx, gk);
}

void ref_pw_fwd(const float* x, int n, int c, int h, int w, const float* k, int co, int stride,
                float* y) {
    Tensor t = ops::pointwise_conv2d_fwd(wrap(x, n, c, h, w), wrap(k, co, c, 1, 1), stride);
    std::copy(t.data.begin(), t.data.end(), y);
}

void ref_pw_bwd(const float* x, int n, int c, int h, int w, const float* k, int co, int stride,
                const float* gy, float* gx, float* gk) {
    const int ho = ops::conv_out_dim(h, 1, stride, 0), wo = ops::conv_out_dim(w, 1, stride, 0);
    ops::pointwise_conv2d_bwd(wrap(x, n, c, h, w), wrap(k, co, c, 1, 1), wrap(gy, n, co, ho, wo),
                              stride, gx, gk);
}

void ref_conv_fwd(const float* x, int n, int c, int h, int w, const float* k, int co, int kk,
                  int stride, int pad, float* y) {
    Tensor t = ops::conv2d_fwd(wrap(x, n, c, h, w), wrap(k, co, c, kk, kk), stride, pad);
    std::copy(t.data.begin(), t.data.end(), y);
}

void ref_bn_train_fwd(const float* x, int n, int c, int h, int w, const float* gamma,
                      const float* beta, float* mm, float* mv, float momentum, float* y,
                      float* xhat, float* inv_std) {
    ops::BnCache<float> cache;
    Tensor t = ops::batch_norm_fwd_train<float>(
        wrap(x, n, c, h, w), std::span<const float>(gamma, c), std::span<const float>(beta, c),
        std::span<float>(mm, c), std::span<float>(mv, c), momentum, &cache);
    std::copy(t.data.begin(), t.data.end(), y);
    if (xhat) std::copy(cache.xhat.data.begin(), cache.xhat.data.end(), xhat);
    if (inv_std) std::copy(cache.inv_std.begin(), cache.inv_std.end(), inv_std);
}

void ref_bn_train_bwd(const float* xhat, const float* inv_std, const float* gamma,
                      const float* gy, int n, int c, int h, int w, float* gx, float* ggamma,
                      float* gbeta) {
    ops::BnCache<float> cache;
    cache.xhat = wrap(xhat, n, c, h, w);
    cache.inv_std.assign(inv_std, inv_std + c);
    ops::batch_norm_bwd_train<float>(cache, std::span<const float>(gamma, c), wrap(gy, n, c, h, w),
                                     gx, ggamma ? std::span<float>(ggamma, c) : std::span<float>(),
                                     gbeta ? std::span<float>(gbeta, c) : std::span<float>());
}

void ref_bn_infer_fwd(const float* x, int n, int c, int h, int w, const float* gamma,
                      const float* beta, const float* mm, const float* mv, float* y) {
    Tensor t = ops::batch_norm_fwd_infer<float>(
        wrap(x, n, c, h, w), std::span<const float>(gamma, c), std::span<const float>(beta, c),
        std::span<const float>(mm, c), std::span<const float>(mv, c));
    std::copy(t.data.begin(), t.data.end(), y);
}

float ref_mse(const float* s, const float* t, size_t count) {
    return ops::mse_local_loss(wrap(s, 1, 1, 1, static_cast<int>(count)),
                               wrap(t, 1, 1, 1, static_cast<int>(count)));
}

void ref_mse_bwd(const float* s, const float* t, size_t count, float scale, float* g) {
    ops::mse_local_loss_bwd<float>(wrap(s, 1, 1, 1, static_cast<int>(count)),
                                   wrap(t, 1, 1, 1, static_cast<int>(count)), g, scale);
}

void ref_sgd(float* w, const float* g, float* v, size_t n, float lr, float momentum) {
    ops::sgd_step<float>(std::span<float>(w, n), std::span<const float>(g, n),
                         std::span<float>(v, n), lr, momentum);
}

int ref_prefix_infer(const char* spec, const float* tw, const float* x, int n, int k,
                     int inclusive, float* out, size_t cap, int* shape) {
    return guard([&] {
        Network net = load_teacher(spec, tw);
        Tensor y = prefix_infer(net, wrap(x, n, net.in_c, net.in_h, net.in_w), k, inclusive != 0);
        if (y.size() > cap) throw std::length_error("prefix buffer too small");
        std::copy(y.data.begin(), y.data.end(), out);
        shape[0] = y.n, shape[1] = y.c, shape[2] = y.h, shape[3] = y.w;
    });
}

int ref_candidate_infer(int kind, int c_in, int c_out, int stride, const float* bw,
                        const float* x, int n, int h, int w, float* out, size_t cap) {
    return guard([&] {
        ReplacementBlock r = build_candidate(static_cast<CandidateKind>(kind), c_in, c_out, stride, 0);
        load_block(r.block, bw);
        Tensor y = block_infer(r.block, wrap(x, n, c_in, h, w));
        if (y.size() > cap) throw std::length_error("output buffer too small");
        std::copy(y.data.begin(), y.data.end(), out);
    });
}

int ref_eval_with_student(const char* spec, const float* tw, const orc_dataset* d,
                          const int* eval_idx, int n_eval, int block_index, int kind,
                          const float* student_w, int batch_size, double* acc) {
    return guard([&] {
        Network net = load_teacher(spec, tw);
        const Block& tb = net.blocks.at(static_cast<size_t>(block_index) - 1);
        ReplacementBlock r = build_candidate(static_cast<CandidateKind>(kind), tb.in_channels,
                                             tb.out_channels, tb.stride, 0);
        load_block(r.block, student_w);
        *acc = evaluate_with_student_block(net, block_index, r.block, to_dataset(d),
                                           std::vector<int>(eval_idx, eval_idx + n_eval),
                                           batch_size);
    });
}

int ref_train_block(const char* spec, const float* tw, const orc_dataset* d, const orc_split* s,
                    const orc_task* t, orc_result* r, float* block_w, size_t cap) {
    return guard([&] {
        Network net = load_teacher(spec, tw);
        TrainedBlockResult res = train_block(net, to_task(t), to_dataset(d), to_split(s));
        std::memset(r, 0, sizeof(*r));
        r->n_loss = static_cast<int>(res.loss_history.size());
        for (int i = 0; i < r->n_loss && i < 256; ++i) r->loss_history[i] = res.loss_history[i];
        r->n_eval = static_cast<int>(res.eval_history.size());
        for (int i = 0; i < r->n_eval && i < 256; ++i) {
            r->eval_epoch[i] = res.eval_history[i].epoch;
            r->eval_acc[i] = res.eval_history[i].accuracy;
        }
        r->final_local_loss = res.final_local_loss;
        r->best_eval = res.best_eval;
        r->failed = res.failed ? 1 : 0;
        std::strncpy(r->failure, res.failure.c_str(), sizeof(r->failure) - 1);
        if (block_w && !res.block.layers.empty()) flatten_block(res.block, block_w, cap);
    });
}

int ref_train_replay(const char* spec, const float* tw, const orc_dataset* d, const orc_split* s,
                     const orc_task* t, int n_steps, float* step_loss, float* final_w,
                     size_t cap) {
    return ref_train_replay_f64(spec, tw, d, s, t, n_steps, step_loss, nullptr, final_w, cap);
}

int ref_train_replay_f64(const char* spec, const float* tw, const orc_dataset* d, const orc_split* s,
                         const orc_task* t, int n_steps, float* step_loss, double* loss64,
                         float* final_w, size_t cap) {
    // The train_block inner loop (distill.cpp:197-253) spelled through the
    // reference's public API, LocalOnly mode.
    return guard([&] {
        Network net = load_teacher(spec, tw);
        const Dataset data = to_dataset(d);
        const SplitIndices split = to_split(s);
        const DistillTask task = to_task(t);
        const int k = task.block_index;
        const Block& tb = net.blocks.at(static_cast<size_t>(k) - 1);
        Block student = build_candidate(task.kind, tb.in_channels, tb.out_channels, tb.stride,
                                        mix_seed(task.seed, 0))
                            .block;
        SgdState opt(collect_block_trainable(student));
        int done = 0;
        for (int epoch = 1; done < n_steps; ++epoch) {
            std::vector<int> order = split.train_idx;
            std::mt19937_64 rng(mix_seed(task.seed, static_cast<uint64_t>(epoch)));
            std::shuffle(order.begin(), order.end(), rng);
            for (size_t at = 0; at < order.size() && done < n_steps; at += task.batch_size) {
                const size_t end = std::min(order.size(), at + static_cast<size_t>(task.batch_size));
                std::vector<int> batch(order.begin() + at, order.begin() + end);
                const Tensor x = gather_batch(data, batch);
                const Tensor a_prev = prefix_infer(net, x, k, false);
                const Tensor t_out = block_infer(tb, a_prev);
                BlockCache cache;
                const Tensor s_out = block_forward(student, a_prev, true, &cache);
                step_loss[done] = ops::mse_local_loss(s_out, t_out);
                if (loss64) {
                    double acc = 0.0;
                    for (size_t q = 0; q < s_out.data.size(); ++q) {
                        const double df = static_cast<double>(s_out.data[q]) - t_out.data[q];
                        acc += df * df;
                    }
                    loss64[done] = acc / static_cast<double>(s_out.data.size());
                }
                Tensor gs(s_out.n, s_out.c, s_out.h, s_out.w);
                ops::mse_local_loss_bwd<float>(s_out, t_out, gs.data.data(), 1.0f);
                opt.zero_grads();
                block_backward(student, cache, gs, false, true);
                opt.step(task.lr, task.momentum);
                ++done;
            }
        }
        flatten_block(student, final_w, cap);
    });
}

// run_parallel through the reference's own runtime (runtime.cpp:124-243).
__attribute__((visibility("default"))) int ref_run_parallel(
    const char* spec, const float* tw, const orc_dataset* d, const orc_split* s, const orc_task* tasks,
    int n_tasks, const int* plan_ids, const int* plan_counts, int workers, int policy, orc_result* results,
    float* block_w, const size_t* w_off) {
    return guard([&] {
        Network net = load_teacher(spec, tw);
        std::vector<DistillTask> tv;
        for (int i = 0; i < n_tasks; ++i) tv.push_back(to_task(&tasks[i]));
        SchedulePlan plan;
        plan.worker_count = workers;
        plan.policy = static_cast<SchedulePolicy>(policy);
        for (int w = 0, at = 0; w < workers; ++w) {
            plan.assignments.emplace_back(plan_ids + at, plan_ids + at + plan_counts[w]);
            at += plan_counts[w];
        }
        RunParallelResult out = run_parallel(net, to_dataset(d), to_split(s), tv, plan);
        for (size_t i = 0; i < out.results.size(); ++i) {
            TrainedBlockResult& res = out.results[i];
            orc_result* r = &results[i];
            std::memset(r, 0, sizeof(*r));
            r->n_loss = static_cast<int>(res.loss_history.size());
            for (int q = 0; q < r->n_loss && q < 256; ++q) r->loss_history[q] = res.loss_history[q];
            r->n_eval = static_cast<int>(res.eval_history.size());
            for (int q = 0; q < r->n_eval && q < 256; ++q) {
                r->eval_epoch[q] = res.eval_history[q].epoch;
                r->eval_acc[q] = res.eval_history[q].accuracy;
            }
            r->final_local_loss = res.final_local_loss;
            r->best_eval = res.best_eval;
            r->failed = res.failed ? 1 : 0;
            std::strncpy(r->failure, res.failure.c_str(), sizeof(r->failure) - 1);
            if (!res.block.layers.empty()) flatten_block(res.block, block_w + w_off[i], w_off[i + 1] - w_off[i]);
        }
    });
}

// PBKD weight files written / rebuilt by the reference (weights_io.cpp), for
// byte-level comparison with the product's writer.  k = 0: the teacher as is;
// else block k replaced by a candidate named like the teacher block (as
// reassemble does, distill.cpp:319).
__attribute__((visibility("default"))) int ref_save_network_file(const char* spec, uint64_t teacher_seed, int k, int kind, uint64_t cand_seed,
                          const char* path) {
    return guard([&] {
        Network net = parse_model_spec(spec, "spec");
        init_weights(net, teacher_seed);
        if (k > 0) {
            Block& tb = net.blocks.at(static_cast<size_t>(k) - 1);
            Block nb = build_candidate(static_cast<CandidateKind>(kind), tb.in_channels, tb.out_channels, tb.stride,
                                       cand_seed)
                           .block;
            nb.name = tb.name;
            tb = std::move(nb);
        }
        save_weights(path, arrays_from_network(net));
    });
}

// rebuild_network_from_arrays of a file against spec: network_weight_hash of
// the result and each block's spec_kind (0 teacher structure, 1 + candidate)
__attribute__((visibility("default"))) int ref_rebuild_network_file(const char* spec, const char* path, uint64_t* hash, int* kinds, int max_blocks) {
    return guard([&] {
        const Network teacher = parse_model_spec(spec, "spec");
        const Network net = rebuild_network_from_arrays(teacher, load_weights(path), path);
        *hash = network_weight_hash(net);
        for (size_t i = 0; i < net.blocks.size() && static_cast<int>(i) < max_blocks; ++i) {
            int kd = 0;
            for (int c = 0; c < 4; ++c)
                if (net.blocks[i].spec_kind == candidate_kind_name(static_cast<CandidateKind>(c))) kd = 1 + c;
            kinds[i] = kd;
        }
    });
}

__attribute__((visibility("default"))) int ref_file_hash(const char* path, uint64_t* out) {
    return guard([&] { *out = file_hash(path); });
}


// finetune (distill.cpp:325-391) or train_teacher (:393-441) through the
// reference.  The network: the teacher of `spec` with weights tw, blocks
// reps[i] (1-based) replaced as reassemble does (distill.cpp:313-318) by
// build_candidate(kinds[i], ..., seeds[i]).  net_out receives the trained
// network's arrays (for_each_array order); hist: loss[epochs], eval[epochs+1].
__attribute__((visibility("default"))) int ref_fit_network(
    const char* spec, const float* tw, const int* reps, const int* kinds, const uint64_t* seeds, int n_reps,
    const orc_dataset* d, const orc_split* s, int epochs, int freeze, float lr, float momentum, int batch,
    uint64_t seed, int teacher_mode, double* loss_hist, double* eval_acc, int* n_eval, double* init_final,
    float* net_out, size_t cap) {
    return guard([&] {
        Network net = load_teacher(spec, tw);
        for (int i = 0; i < n_reps; ++i) {
            Block& tb = net.blocks.at(static_cast<size_t>(reps[i]) - 1);
            Block nb = build_candidate(static_cast<CandidateKind>(kinds[i]), tb.in_channels, tb.out_channels,
                                       tb.stride, seeds[i])
                           .block;
            nb.name = tb.name;
            nb.replaceable = false;
            tb = std::move(nb);
        }
        const Dataset data = to_dataset(d);
        const SplitIndices split = to_split(s);
        std::vector<EvalPoint> ev;
        std::vector<double> lh;
        if (teacher_mode) {
            TeacherTrainResult r = train_teacher(net, data, split, epochs, lr, momentum, batch, seed);
            ev = r.eval_history, lh = r.loss_history;
            init_final[0] = ev.front().accuracy, init_final[1] = r.final_eval;
        } else {
            FinetuneResult r = finetune(net, data, split, epochs, freeze != 0, lr, momentum, batch, seed);
            ev = r.eval_history, lh = r.loss_history;
            init_final[0] = r.initial_eval, init_final[1] = r.final_eval;
        }
        for (size_t i = 0; i < lh.size(); ++i) loss_hist[i] = lh[i];
        for (size_t i = 0; i < ev.size(); ++i) eval_acc[i] = ev[i].accuracy;
        *n_eval = static_cast<int>(ev.size());
        size_t at = 0;
        for_each_array(net, [&](const std::string&, Tensor& t) {
            if (at + t.data.size() > cap) throw std::length_error("network buffer too small");
            std::copy(t.data.begin(), t.data.end(), net_out + at);
            at += t.data.size();
        });
    });
}

}  // extern "C"
