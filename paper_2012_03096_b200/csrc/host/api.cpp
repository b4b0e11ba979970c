// The reference's C++ entry points (distill.hpp:72-79, runtime.hpp:41-43,
// model.hpp:154-186) implemented over the C ABI in include/pbkd_b200.h.
// Everything numeric runs on the GPU; this file only marshals pbkd:: types.
#include <algorithm>
#include <chrono>
#include <type_traits>
#include <cstdlib>
#include <mutex>
#include <sstream>

#include <json.hpp>

#include "pbkd/distill.hpp"
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
    // PBKD_DEVICES="0,1,..." (or, unset, every visible GPU when there is more
    // than one): a context over that GPU list, so run_parallel's workers map
    // onto GPUs (runtime.cpp:226-233); else PBKD_DEVICE (default 0)
    pbkd_ctx* get() {
        if (!ctx) {
            std::vector<int> devs;
            if (const char* list = std::getenv("PBKD_DEVICES")) {
                std::stringstream ss(list);
                for (std::string tok; std::getline(ss, tok, ',');)
                    if (!tok.empty()) devs.push_back(std::atoi(tok.c_str()));
            } else if (!std::getenv("PBKD_DEVICE")) {
                int n = 0;
                if (pbkd_device_count(&n) == 0 && n > 1)
                    for (int i = 0; i < n; ++i) devs.push_back(i);
            }
            if (!devs.empty()) {
                check(pbkd_ctx_create_multi(devs.data(), static_cast<int>(devs.size()), &ctx));
            } else {
                const char* dev = std::getenv("PBKD_DEVICE");
                check(pbkd_ctx_create(dev ? std::atoi(dev) : 0, &ctx));
            }
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
        if (b.spec_kind != "conv3x3" && b.spec_kind != "conv1x1" && b.spec_kind != "residual3x3" &&
            b.spec_kind != "bottleneck" && b.spec_kind != "stem7x7")
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

namespace {

std::vector<pbkd_layer_desc> descs_of(const Block& b) {
    std::vector<pbkd_layer_desc> out;
    for (const LayerParams& l : b.layers) {
        pbkd_layer_desc d{};
        d.kind = static_cast<int>(l.kind);
        d.in_channels = l.in_channels;
        d.out_channels = l.out_channels;
        d.kernel = l.kernel;
        d.stride = l.stride;
        d.padding = l.padding;
        d.has_weight = l.weight.data.empty() ? 0 : 1;
        d.has_bias = l.bias.data.empty() ? 0 : 1;
        out.push_back(d);
    }
    return out;
}

std::vector<float> flat_of(const Block& b) {
    std::vector<float> w;
    for_each_block_array(const_cast<Block&>(b),
                         [&](const std::string&, Tensor& t) { w.insert(w.end(), t.data.begin(), t.data.end()); });
    return w;
}

void unflat(Block& b, const float* w) {
    for_each_block_array(b, [&](const std::string&, Tensor& t) {
        std::copy(w, w + t.data.size(), t.data.begin());
        w += t.data.size();
    });
}

// A network as the C ABI's pbkd_net_desc (blocks, then the classifier).
struct NetDesc {
    std::vector<int> counts;
    std::vector<pbkd_layer_desc> layers;
    std::vector<std::string> kinds;
    std::vector<const char*> kind_ptrs;
    std::vector<float> arrays;
    pbkd_net_desc d{};
    explicit NetDesc(const Network& net) {
        auto add = [&](const Block& b) {
            const auto L = descs_of(b);
            counts.push_back(static_cast<int>(L.size()));
            layers.insert(layers.end(), L.begin(), L.end());
            kinds.push_back(b.spec_kind);
            const auto w = flat_of(b);
            arrays.insert(arrays.end(), w.begin(), w.end());
        };
        for (const Block& b : net.blocks) add(b);
        add(net.classifier);
        for (const std::string& k : kinds) kind_ptrs.push_back(k.c_str());
        d.n_blocks = static_cast<int>(net.blocks.size());
        d.layer_counts = counts.data();
        d.layers = layers.data();
        d.spec_kinds = kind_ptrs.data();
        d.in_c = net.in_c, d.in_h = net.in_h, d.in_w = net.in_w;
    }
    void write_back(Network& net) const {
        const float* w = arrays.data();
        for (Block& b : net.blocks) {
            unflat(b, w);
            w += flat_of(b).size();
        }
        unflat(net.classifier, w);
    }
};

pbkd_ctx* bind_data(const Dataset& data) {
    Shared& s = shared();
    pbkd_ctx* ctx = s.get();
    uint64_t dh = fnv1a64(data.images.data(), data.images.size() * sizeof(float));
    dh = fnv1a64(data.labels.data(), data.labels.size() * sizeof(int), dh);
    if (dh != s.data_hash) {
        check(pbkd_dataset_load(ctx, data.images.data(), data.labels.data(), data.count(), data.c, data.h, data.w,
                                data.classes));
        s.data_hash = dh;
    }
    return ctx;
}

double evaluate_locked(const Network& net, const Dataset& data, const std::vector<int>& idx, int batch_size) {
    if (idx.empty()) throw SpecError("evaluation split is empty");
    if (batch_size < 1) throw SpecError("batch_size must be at least 1");
    pbkd_ctx* ctx = bind_data(data);
    NetDesc nd(net);
    double acc = 0.0;
    check(pbkd_evaluate_network(ctx, &nd.d, nd.arrays.data(), nd.arrays.size(), idx.data(),
                                static_cast<int>(idx.size()), batch_size, &acc));
    return acc;
}

Tensor block_forward_locked(Block& b, const Tensor& x, bool train, BlockCache* cache) {
    pbkd_ctx* ctx = shared().get();
    const auto L = descs_of(b);
    std::vector<float> w = flat_of(b);
    // output shape: from the layer list (model.cpp shape rules)
    Network probe;
    probe.in_c = x.c, probe.in_h = x.h, probe.in_w = x.w;
    probe.blocks.push_back(b);
    int c = 0, h = 0, ww = 0;
    block_input_shape(probe, 2, c, h, ww);
    Tensor y(x.n, c, h, ww);
    int shape[4];
    pbkd_block_cache* hc = nullptr;
    check(pbkd_block_forward(ctx, L.data(), static_cast<int>(L.size()), w.data(), w.size(), x.data.data(), x.n, x.c,
                             x.h, x.w, train ? 1 : 0, y.data.data(), y.size(), shape, cache ? &hc : nullptr));
    if (train) unflat(b, w.data());  // moving statistics updated in place
    if (cache) {
        cache->train_mode = train;
        cache->layers.assign(b.layers.size(), LayerCache{});
        cache->device = std::shared_ptr<pbkd_block_cache>(hc, pbkd_block_cache_free);
        cache->in_shape = {x.n, x.c, x.h, x.w};
    }
    return y;
}

Tensor block_backward_locked(Block& b, const BlockCache& cache, const Tensor& gy, bool need_input_grad,
                             bool param_grads) {
    if (cache.layers.size() != b.layers.size())
        throw std::logic_error("block_backward: cache does not match block " + b.name);
    if (!cache.train_mode && param_grads)
        throw std::logic_error("block_backward: parameter gradients require a train-mode cache");
    if (!cache.device) throw std::logic_error("block_backward: cache holds no forward state");
    pbkd_ctx* ctx = shared().get();
    const auto L = descs_of(b);
    const std::vector<float> w = flat_of(b);
    std::vector<float> g(w.size(), 0.0f);
    const auto& s = cache.in_shape;
    Tensor gx;
    if (need_input_grad) gx = Tensor(s[0], s[1], s[2], s[3]);
    check(pbkd_block_backward(ctx, L.data(), static_cast<int>(L.size()), w.data(), w.size(), cache.device.get(),
                              gy.data.data(), gy.n, gy.c, gy.h, gy.w, need_input_grad ? 1 : 0, param_grads ? 1 : 0,
                              g.data(), need_input_grad ? gx.data.data() : nullptr, gx.data.size()));
    if (param_grads) {  // accumulate into each trainable tensor's grad (model.cpp:568-571)
        size_t at = 0;
        for_each_block_array(b, [&](const std::string& name, Tensor& t) {
            const bool stat = name.size() >= 11 && (name.compare(name.size() - 11, 11, "moving_mean") == 0 ||
                                                     name.compare(name.size() - 10, 10, "moving_var") == 0);
            if (!stat) {
                t.ensure_grad();
                for (size_t i = 0; i < t.data.size(); ++i) t.grad[i] += g[at + i];
            }
            at += t.data.size();
        });
    }
    return gx;
}

}  // namespace

double evaluate_with_student_block(const Network& teacher, int block_index, const Block& student,
                                   const Dataset& data, const std::vector<int>& eval_idx, int batch_size) {
    std::lock_guard<std::mutex> lk(shared().m);
    if (eval_idx.empty()) throw SpecError("evaluation split is empty");
    if (batch_size < 1) throw SpecError("batch_size must be at least 1");
    if (block_index < 1 || block_index > static_cast<int>(teacher.blocks.size()))
        throw SpecError("block index " + std::to_string(block_index) + " out of range for '" + teacher.name + "'");
    int kind = -1;
    for (CandidateKind k : kAllCandidates)
        if (student.spec_kind == candidate_kind_name(k)) kind = static_cast<int>(k);
    if (kind < 0) {  // any other block: the network with it swapped in
        Network swapped = teacher;
        swapped.blocks[static_cast<size_t>(block_index) - 1] = student;
        return evaluate_locked(swapped, data, eval_idx, batch_size);
    }
    const Block& tb = teacher.blocks[static_cast<size_t>(block_index) - 1];
    if (student.in_channels != tb.in_channels || student.out_channels != tb.out_channels ||
        student.stride != tb.stride)
        throw ShapeError("student block (" + std::to_string(student.in_channels) + "->" +
                         std::to_string(student.out_channels) + ", stride " + std::to_string(student.stride) +
                         ") does not match teacher block " + std::to_string(block_index));
    pbkd_ctx* ctx = bind(teacher, &data);
    const std::vector<float> w = flat_of(student);
    double acc = 0.0;
    check(pbkd_eval_with_student(ctx, block_index, kind, w.data(), eval_idx.data(),
                                 static_cast<int>(eval_idx.size()), batch_size, &acc));
    return acc;
}

double evaluate_network(const Network& net, const Dataset& data, const std::vector<int>& idx, int batch_size) {
    std::lock_guard<std::mutex> lk(shared().m);
    return evaluate_locked(net, data, idx, batch_size);
}

Tensor prefix_infer(const Network& net, const Tensor& x, int k, bool inclusive) {
    std::lock_guard<std::mutex> lk(shared().m);
    const int count = static_cast<int>(net.blocks.size());
    if (k < 1 || k > count)
        throw std::out_of_range("prefix_infer: k=" + std::to_string(k) + " out of range [1," +
                                std::to_string(count) + "]");
    if (x.c != net.in_c || x.h != net.in_h || x.w != net.in_w)
        throw ShapeError("prefix_infer: input " + x.shape_str() + " does not match the network input (" +
                         std::to_string(net.in_c) + "," + std::to_string(net.in_h) + "," + std::to_string(net.in_w) + ")");
    const int take = inclusive ? k : k - 1;
    if (take == 0) return x;
    pbkd_ctx* ctx = bind(net, nullptr);
    int c = 0, h = 0, w = 0;
    block_input_shape(net, take + 1, c, h, w);
    Tensor y(x.n, c, h, w);
    int shape[4];
    check(pbkd_prefix_infer(ctx, x.data.data(), x.n, k, inclusive ? 1 : 0, y.data.data(), y.size(), shape));
    return y;
}

Tensor block_forward(Block& b, const Tensor& x, bool train, BlockCache* cache) {
    std::lock_guard<std::mutex> lk(shared().m);
    return block_forward_locked(b, x, train, cache);
}

Tensor block_infer(const Block& b, const Tensor& x) {
    std::lock_guard<std::mutex> lk(shared().m);
    return block_forward_locked(const_cast<Block&>(b), x, false, nullptr);  // inference mutates nothing
}

Tensor block_backward(Block& b, const BlockCache& cache, const Tensor& gy, bool need_input_grad, bool param_grads) {
    std::lock_guard<std::mutex> lk(shared().m);
    return block_backward_locked(b, cache, gy, need_input_grad, param_grads);
}

// model.cpp:658-693: the reference's compositions over the block calls
Tensor network_forward_train(Network& net, const Tensor& x, NetCache& cache, const std::vector<bool>& train_mask) {
    if (!train_mask.empty() && train_mask.size() != net.blocks.size())
        throw std::invalid_argument("network_forward_train: mask size " + std::to_string(train_mask.size()) +
                                    " vs " + std::to_string(net.blocks.size()) + " blocks");
    cache.blocks.assign(net.blocks.size(), BlockCache{});
    Tensor cur = x;
    for (size_t i = 0; i < net.blocks.size(); ++i)
        cur = block_forward(net.blocks[i], cur, train_mask.empty() || train_mask[i], &cache.blocks[i]);
    if (net.has_classifier()) cur = block_forward(net.classifier, cur, true, &cache.classifier);
    return cur;
}

void network_backward(Network& net, const NetCache& cache, const Tensor& glogits, const std::vector<bool>& train_mask,
                      bool freeze_classifier) {
    if (!train_mask.empty() && train_mask.size() != net.blocks.size())
        throw std::invalid_argument("network_backward: mask size mismatch");
    Tensor g = glogits;
    if (net.has_classifier())
        g = block_backward(net.classifier, cache.classifier, g, !net.blocks.empty(), !freeze_classifier);
    for (int i = static_cast<int>(net.blocks.size()) - 1; i >= 0; --i)
        g = block_backward(net.blocks[static_cast<size_t>(i)], cache.blocks[static_cast<size_t>(i)], g, i > 0,
                           train_mask.empty() || train_mask[static_cast<size_t>(i)]);
}

Tensor network_infer(const Network& net, const Tensor& x) {
    Tensor cur = x;
    for (const Block& b : net.blocks) cur = block_infer(b, cur);
    if (net.has_classifier()) cur = block_infer(net.classifier, cur);
    return cur;
}

// distill.cpp:297-323 (host bookkeeping: no arithmetic)
AssembledStudent reassemble(const Network& teacher, const std::vector<TrainedBlockResult>& results,
                            double threshold) {
    AssembledStudent out;
    out.net = teacher;
    std::vector<int> seen;
    for (const TrainedBlockResult& r : results) {
        if (r.block_index < 1 || r.block_index > static_cast<int>(teacher.blocks.size()))
            throw SpecError("result references block " + std::to_string(r.block_index) + ", which '" +
                            teacher.name + "' does not have");
        if (std::find(seen.begin(), seen.end(), r.block_index) != seen.end())
            throw SpecError("two results reference block " + std::to_string(r.block_index));
        seen.push_back(r.block_index);
        ReplacementDecision d;
        d.block_index = r.block_index;
        d.kind = r.kind;
        d.failed = r.failed;
        d.best_eval = r.best_eval;
        d.threshold = threshold;
        if (r.failed) {
            d.note = r.failure;
        } else if (r.best_eval > threshold) {
            Block nb = r.block;
            nb.name = teacher.blocks[static_cast<size_t>(r.block_index) - 1].name;
            nb.replaceable = false;
            out.net.blocks[static_cast<size_t>(r.block_index) - 1] = std::move(nb);
            d.replaced = true;
        } else {
            d.note = "accuracy not above threshold";
        }
        out.decisions.push_back(d);
    }
    std::sort(out.decisions.begin(), out.decisions.end(),
              [](const ReplacementDecision& a, const ReplacementDecision& b) { return a.block_index < b.block_index; });
    return out;
}

namespace {
// finetune / train_teacher: the whole epoch loop on the device (pbkd_fit_network)
template <class R>
R fit_locked(Network& net, const Dataset& data, const SplitIndices& split, int epochs, bool freeze, float lr,
             float momentum, int batch_size, uint64_t seed, bool teacher_mode) {
    pbkd_ctx* ctx = bind_data(data);
    NetDesc nd(net);
    std::vector<double> loss(static_cast<size_t>(std::max(epochs, 0)) + 1);
    std::vector<int> ee(static_cast<size_t>(std::max(epochs, 0)) + 1);
    std::vector<double> ea(ee.size());
    double init = 0.0, fin = 0.0;
    int ne = 0;
    check(pbkd_fit_network(ctx, &nd.d, nd.arrays.data(), nd.arrays.size(), split.train_idx.data(),
                           static_cast<int>(split.train_idx.size()), split.eval_idx.data(),
                           static_cast<int>(split.eval_idx.size()), epochs, freeze ? 1 : 0, lr, momentum, batch_size,
                           seed, teacher_mode ? 1 : 0, &init, &fin, loss.data(), ee.data(), ea.data(), &ne));
    nd.write_back(net);
    R r;
    for (int i = 0; i < ne; ++i) r.eval_history.push_back({ee[static_cast<size_t>(i)], ea[static_cast<size_t>(i)]});
    r.loss_history.assign(loss.begin(), loss.begin() + std::max(0, ne - 1));
    r.final_eval = fin;
    if constexpr (std::is_same_v<R, FinetuneResult>) r.initial_eval = init;
    return r;
}
}  // namespace

FinetuneResult finetune(Network& student, const Dataset& data, const SplitIndices& split, int epochs,
                        bool freeze_non_replaced, float lr, float momentum, int batch_size, uint64_t seed) {
    std::lock_guard<std::mutex> lk(shared().m);
    return fit_locked<FinetuneResult>(student, data, split, epochs, freeze_non_replaced, lr, momentum, batch_size,
                                      seed, false);
}

TeacherTrainResult train_teacher(Network& net, const Dataset& data, const SplitIndices& split, int epochs, float lr,
                                 float momentum, int batch_size, uint64_t seed) {
    std::lock_guard<std::mutex> lk(shared().m);
    return fit_locked<TeacherTrainResult>(net, data, split, epochs, false, lr, momentum, batch_size, seed, true);
}

namespace ops {
template <>
float mse_local_loss<float>(const Tensor4<float>& s, const Tensor4<float>& t) {
    require_same_shape("mse_local_loss", s.n, s.c, s.h, s.w, t.n, t.c, t.h, t.w);
    std::lock_guard<std::mutex> lk(shared().m);
    float loss = 0.0f;
    check(pbkd_mse_local_loss(shared().get(), s.data.data(), t.data.data(), s.data.size(), &loss));
    return loss;
}
template <>
void mse_local_loss_bwd<float>(const Tensor4<float>& s, const Tensor4<float>& t, float* g, float scale) {
    require_same_shape("mse_local_loss_bwd", s.n, s.c, s.h, s.w, t.n, t.c, t.h, t.w);
    if (!g) return;
    std::lock_guard<std::mutex> lk(shared().m);
    check(pbkd_mse_local_loss_bwd(shared().get(), s.data.data(), t.data.data(), s.data.size(), scale, g));
}
template <>
float softmax_cross_entropy_fwd<float>(const Tensor4<float>& logits, std::span<const int> labels,
                                       Tensor4<float>* probs) {
    if (logits.h != 1 || logits.w != 1)
        throw ShapeError("softmax_cross_entropy: logits must be (N,K,1,1), got " + logits.shape_str());
    if (static_cast<int>(labels.size()) != logits.n)
        throw std::invalid_argument("softmax_cross_entropy: " + std::to_string(labels.size()) +
                                    " labels for batch of " + std::to_string(logits.n));
    std::lock_guard<std::mutex> lk(shared().m);
    if (probs) *probs = Tensor4<float>(logits.n, logits.c, 1, 1);
    float loss = 0.0f;
    check(pbkd_softmax_ce(shared().get(), logits.data.data(), logits.n, logits.c, labels.data(), &loss,
                          probs ? probs->data.data() : nullptr));
    return loss;
}
template <>
void softmax_cross_entropy_bwd<float>(const Tensor4<float>& probs, std::span<const int> labels, float* g, float scale) {
    if (!g) return;
    std::lock_guard<std::mutex> lk(shared().m);
    check(pbkd_softmax_ce_bwd(shared().get(), probs.data.data(), probs.n, probs.c, labels.data(), scale, g));
}
template <>
void sgd_step<float>(std::span<float> w, std::span<const float> g, std::span<float> v, float lr, float momentum) {
    if (w.size() != g.size() || w.size() != v.size())
        throw ShapeError("sgd_step: weights/grads/velocity length mismatch (" + std::to_string(w.size()) + "/" +
                         std::to_string(g.size()) + "/" + std::to_string(v.size()) + ")");
    check(pbkd_sgd_host(w.data(), g.data(), v.data(), w.size(), lr, momentum));
}
}  // namespace ops

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
