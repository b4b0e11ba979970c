// The reference's C++ entry points (distill.hpp:72-79, runtime.hpp:41-43,
// model.hpp:154-186) implemented over the C ABI in include/pbkd_b200.h.
// Everything numeric runs on the GPU; this file only marshals pbkd:: types.
#include <chrono>
#include <cstdlib>
#include <mutex>
#include <sstream>

#include <json.hpp>

#include "pbkd/runtime.hpp"
#include "pbkd_b200.h"

namespace pbkd {

namespace {

[[noreturn]] void rethrow_abi() {
    const std::string msg = pbkd_last_error();
    switch (pbkd_last_error_kind()) {
        case PBKD_ERR_SPEC: throw SpecError(msg);
        case PBKD_ERR_SHAPE: throw ShapeError(msg);
        case PBKD_ERR_RANGE: throw std::out_of_range(msg);
        case PBKD_ERR_LOGIC: throw std::logic_error(msg);
        default: throw std::runtime_error(msg);
    }
}

void check(int rc) {
    if (rc != 0) rethrow_abi();
}

// One process-wide context on PBKD_DEVICE (default 0); teacher and dataset
// uploads are cached by content hash so repeated train_block calls on the
// same teacher/data do not re-upload.
struct Shared {
    std::mutex m;
    pbkd_ctx* ctx = nullptr;
    uint64_t teacher_hash = 0;
    uint64_t data_hash = 0;
    pbkd_ctx* get() {
        if (!ctx) {
            const char* dev = std::getenv("PBKD_DEVICE");
            check(pbkd_ctx_create(dev ? std::atoi(dev) : 0, &ctx));
        }
        return ctx;
    }
};

Shared& shared() {
    static Shared s;
    return s;
}

std::string spec_json_of(const Network& net) {
    using nlohmann::json;
    json doc;
    doc["name"] = net.name;
    doc["input_shape"] = {net.in_c, net.in_h, net.in_w};
    json blocks = json::array();
    for (const Block& b : net.blocks) {
        if (b.spec_kind != "conv3x3" && b.spec_kind != "conv1x1" && b.spec_kind != "residual3x3")
            throw SpecError("block '" + b.name + "' of kind '" + b.spec_kind +
                            "' cannot be uploaded as a teacher block");
        blocks.push_back({{"name", b.name}, {"kind", b.spec_kind}, {"out_channels", b.out_channels},
                          {"stride", b.stride}, {"padding", b.padding}});
    }
    doc["blocks"] = blocks;
    json cls = json::array();
    for (const LayerParams& l : net.classifier.layers) {
        if (l.kind == LayerKind::GlobalAvgPool) cls.push_back({{"kind", "global_avg_pool"}});
        else if (l.kind == LayerKind::ReLU) cls.push_back({{"kind", "relu"}});
        else if (l.kind == LayerKind::Dense) cls.push_back({{"kind", "dense"}, {"out_features", l.out_channels}});
    }
    doc["classifier"] = cls;
    return doc.dump();
}

pbkd_ctx* bind(const Network& teacher, const Dataset* data) {
    Shared& s = shared();
    pbkd_ctx* ctx = s.get();
    const uint64_t th = network_weight_hash(teacher) ^ fnv1a64(teacher.name.data(), teacher.name.size());
    if (th != s.teacher_hash) {
        std::vector<float> w;
        for_each_array(const_cast<Network&>(teacher),
                       [&](const std::string&, Tensor& t) { w.insert(w.end(), t.data.begin(), t.data.end()); });
        check(pbkd_teacher_load(ctx, spec_json_of(teacher).c_str(), w.data(), w.size()));
        s.teacher_hash = th;
    }
    if (data) {
        uint64_t dh = fnv1a64(data->images.data(), data->images.size() * sizeof(float));
        dh = fnv1a64(data->labels.data(), data->labels.size() * sizeof(int), dh);
        if (dh != s.data_hash) {
            check(pbkd_dataset_load(ctx, data->images.data(), data->labels.data(), data->count(), data->c,
                                    data->h, data->w, data->classes));
            s.data_hash = dh;
        }
    }
    return ctx;
}

pbkd_task to_abi(const DistillTask& t) {
    pbkd_task a{};
    a.block_index = t.block_index;
    a.kind = static_cast<int>(t.kind);
    a.epochs = t.epochs;
    a.eval_every = t.eval_every;
    a.seed = t.seed;
    a.threshold = t.threshold;
    a.loss_mode = static_cast<int>(t.loss_mode);
    a.lambda_local = t.lambda_local;
    a.lr = t.lr;
    a.momentum = t.momentum;
    a.batch_size = t.batch_size;
    a.max_steps = t.max_steps;
    return a;
}

Block block_from(const Network& teacher, const DistillTask& t, const std::vector<float>& flat) {
    const Block& tb = teacher.blocks.at(static_cast<size_t>(t.block_index) - 1);
    Block b = build_candidate(t.kind, tb.in_channels, tb.out_channels, tb.stride, 0).block;
    size_t at = 0;
    for_each_block_array(b, [&](const std::string&, Tensor& x) {
        std::copy(flat.begin() + static_cast<long>(at), flat.begin() + static_cast<long>(at + x.data.size()),
                  x.data.begin());
        at += x.data.size();
    });
    return b;
}

TrainedBlockResult result_of(const Network& teacher, const DistillTask& t, const pbkd_results* r, int i) {
    pbkd_result_info info{};
    check(pbkd_run_info(r, i, &info));
    TrainedBlockResult out;
    out.block_index = info.block_index;
    out.kind = info.kind;
    out.failed = info.failed != 0;
    out.failure = info.failure;
    out.loss_history.resize(static_cast<size_t>(info.n_loss));
    check(pbkd_run_loss_history(r, i, out.loss_history.data(), info.n_loss));
    std::vector<int> ep(static_cast<size_t>(info.n_eval));
    std::vector<double> acc(static_cast<size_t>(info.n_eval));
    check(pbkd_run_eval_history(r, i, ep.data(), acc.data(), info.n_eval));
    for (int k = 0; k < info.n_eval; ++k) out.eval_history.push_back({ep[static_cast<size_t>(k)], acc[static_cast<size_t>(k)]});
    out.final_local_loss = info.final_local_loss;
    out.best_eval = info.best_eval;
    out.wall_time_s = info.wall_time_s;
    if (info.has_best) {
        std::vector<float> flat(info.n_block_floats);
        check(pbkd_run_block(r, i, 0, flat.data(), flat.size()));
        out.block = block_from(teacher, t, flat);
    }
    return out;
}

}  // namespace

const char* trace_event_kind_name(TraceEventKind k) {
    switch (k) {
        case TraceEventKind::Dispatch: return "dispatch";
        case TraceEventKind::TaskStart: return "task_start";
        case TraceEventKind::TaskEnd: return "task_end";
        case TraceEventKind::Steal: return "steal";
        case TraceEventKind::Gather: return "gather";
    }
    return "unknown";
}

TraceEventKind trace_event_kind_from_name(const std::string& name) {
    for (TraceEventKind k : {TraceEventKind::Dispatch, TraceEventKind::TaskStart, TraceEventKind::TaskEnd,
                             TraceEventKind::Steal, TraceEventKind::Gather})
        if (name == trace_event_kind_name(k)) return k;
    throw SpecError("unknown trace event kind '" + name + "'");
}

TrainedBlockResult train_block(const Network& teacher, const DistillTask& task, const Dataset& data,
                               const SplitIndices& split) {
    std::lock_guard<std::mutex> lk(shared().m);
    pbkd_ctx* ctx = bind(teacher, &data);
    const pbkd_task t = to_abi(task);
    pbkd_results* r = nullptr;
    check(pbkd_run(ctx, &t, 1, split.train_idx.data(), static_cast<int>(split.train_idx.size()),
                   split.eval_idx.data(), static_cast<int>(split.eval_idx.size()), 0, &r));
    TrainedBlockResult out = result_of(teacher, task, r, 0);
    pbkd_run_free(r);
    return out;
}

RunParallelResult run_parallel(const Network& teacher, const Dataset& data, const SplitIndices& split,
                               const std::vector<DistillTask>& tasks, const SchedulePlan& plan) {
    std::lock_guard<std::mutex> lk(shared().m);
    pbkd_ctx* ctx = bind(teacher, &data);
    std::vector<pbkd_task> ts;
    for (const DistillTask& t : tasks) ts.push_back(to_abi(t));
    std::vector<int> ids, counts;
    for (const auto& q : plan.assignments) {
        counts.push_back(static_cast<int>(q.size()));
        ids.insert(ids.end(), q.begin(), q.end());
    }
    if (plan.assignments.size() != static_cast<size_t>(std::max(plan.worker_count, 0)))
        throw SpecError("plan has " + std::to_string(plan.assignments.size()) + " worker lists for worker_count " +
                        std::to_string(plan.worker_count));
    pbkd_results* r = nullptr;
    check(pbkd_run_parallel(ctx, ts.data(), static_cast<int>(ts.size()), split.train_idx.data(),
                            static_cast<int>(split.train_idx.size()), split.eval_idx.data(),
                            static_cast<int>(split.eval_idx.size()), plan.worker_count,
                            static_cast<int>(plan.policy), ids.data(), counts.data(), 0, &r));
    RunParallelResult out;
    for (int i = 0; i < pbkd_run_count(r); ++i) {
        pbkd_result_info info{};
        check(pbkd_run_info(r, i, &info));
        const DistillTask* t = nullptr;
        for (const DistillTask& x : tasks)
            if (x.block_index == info.block_index) t = &x;
        out.results.push_back(result_of(teacher, *t, r, i));
    }
    int n = 0;
    check(pbkd_run_trace(r, nullptr, 0, &n));
    std::vector<pbkd_trace_event> ev(static_cast<size_t>(n));
    check(pbkd_run_trace(r, ev.data(), n, &n));
    for (const pbkd_trace_event& e : ev)
        out.trace.push_back({e.timestamp_s, e.worker_id, e.task_id, static_cast<TraceEventKind>(e.kind)});
    out.wall_time_s = pbkd_run_wall_time(r);
    pbkd_run_free(r);
    return out;
}

double evaluate_with_student_block(const Network& teacher, int block_index, const Block& student,
                                   const Dataset& data, const std::vector<int>& eval_idx, int batch_size) {
    std::lock_guard<std::mutex> lk(shared().m);
    pbkd_ctx* ctx = bind(teacher, &data);
    int kind = -1;
    for (CandidateKind k : kAllCandidates)
        if (student.spec_kind == candidate_kind_name(k)) kind = static_cast<int>(k);
    if (kind < 0) throw SpecError("student block is not a replacement candidate");
    std::vector<float> w;
    for_each_block_array(const_cast<Block&>(student),
                         [&](const std::string&, Tensor& t) { w.insert(w.end(), t.data.begin(), t.data.end()); });
    double acc = 0.0;
    check(pbkd_eval_with_student(ctx, block_index, kind, w.data(), eval_idx.data(),
                                 static_cast<int>(eval_idx.size()), batch_size, &acc));
    return acc;
}

Tensor prefix_infer(const Network& net, const Tensor& x, int k, bool inclusive) {
    std::lock_guard<std::mutex> lk(shared().m);
    pbkd_ctx* ctx = bind(net, nullptr);
    int c = 0, h = 0, w = 0;
    const int take = inclusive ? k : k - 1;
    if (k < 1 || k > static_cast<int>(net.blocks.size())) throw std::out_of_range("prefix_infer: k out of range");
    block_input_shape(net, take + 1, c, h, w);
    Tensor y(x.n, c, h, w);
    int shape[4];
    check(pbkd_prefix_infer(ctx, x.data.data(), x.n, k, inclusive ? 1 : 0, y.data.data(), y.size(), shape));
    return y;
}

Tensor block_infer(const Block& b, const Tensor& x) {
    std::lock_guard<std::mutex> lk(shared().m);
    pbkd_ctx* ctx = shared().get();
    int kind = -1;
    for (CandidateKind k : kAllCandidates)
        if (b.spec_kind == candidate_kind_name(k)) kind = static_cast<int>(k);
    if (kind < 0) throw SpecError("block_infer on the GPU path supports replacement candidates");
    std::vector<float> w;
    for_each_block_array(const_cast<Block&>(b),
                         [&](const std::string&, Tensor& t) { w.insert(w.end(), t.data.begin(), t.data.end()); });
    const int ho = (x.h - 1) / b.stride + 1, wo = (x.w - 1) / b.stride + 1;
    Tensor y(x.n, b.out_channels, ho, wo);
    check(pbkd_candidate_infer(ctx, kind, b.in_channels, b.out_channels, b.stride, w.data(), x.data.data(), x.n,
                               x.h, x.w, y.data.data(), y.size()));
    return y;
}

SgdState::SgdState(std::vector<Tensor*> p) : params(std::move(p)) {
    for (Tensor* t : params) velocity.emplace_back(t->data.size(), 0.0f);
}

void SgdState::zero_grads() {
    for (Tensor* t : params) {
        t->ensure_grad();
        t->zero_grad();
    }
}

void SgdState::step(float lr, float momentum) {
    for (size_t i = 0; i < params.size(); ++i) {
        Tensor& t = *params[i];
        t.ensure_grad();
        check(pbkd_sgd_host(t.data.data(), t.grad.data(), velocity[i].data(), t.data.size(), lr, momentum));
    }
}

}  // namespace pbkd
