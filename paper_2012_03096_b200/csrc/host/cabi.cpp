// cabi.cu -- extern "C" boundary (include/pbkd_b200.h) over the engine.
#include <algorithm>
#include <chrono>
#include <deque>
#include <cstring>
#include <map>
#include <memory>
#include <set>
#include <string>
#include <thread>
#include <vector>

#include "pbkd_b200.h"
#include "ctx.hpp"
#include "../comm.hpp"
#include "../engine.hpp"
#include "../ops.cuh"
#include "pbkd/dataset.hpp"
#include "pbkd/replacement.hpp"
#include "pbkd/weights_io.hpp"
#include "pbkd/scheduler.hpp"

using namespace pbkd_gpu;



struct pbkd_results {
    RunTiming timing;
    std::vector<TaskOutcome> res;
    std::vector<pbkd_trace_event> trace;
    double wall = 0.0;
    double epoch_ms = 0.0;
};

namespace {
thread_local std::string g_err;
thread_local int g_kind = 0;

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const pbkd::ShapeError& e) {
        g_err = e.what(), g_kind = PBKD_ERR_SHAPE;
    } catch (const pbkd::WeightsError& e) {
        g_err = e.what(), g_kind = PBKD_ERR_WEIGHTS;
    } catch (const pbkd_gpu::CudaError& e) {
        g_err = e.what(), g_kind = PBKD_ERR_CUDA;
    } catch (const std::out_of_range& e) {
        g_err = e.what(), g_kind = PBKD_ERR_RANGE;
    } catch (const std::invalid_argument& e) {
        g_err = e.what(), g_kind = PBKD_ERR_SPEC;
    } catch (const std::logic_error& e) {
        g_err = e.what(), g_kind = PBKD_ERR_LOGIC;
    } catch (const std::exception& e) {
        g_err = e.what(), g_kind = PBKD_ERR_OTHER;
    }
    return 1;
}

}  // namespace

// error state shared with cabi_net.cpp (not part of the public header)
extern "C" void pbkd_internal_set_error(const char* msg, int kind) {
    g_err = msg ? msg : "";
    g_kind = kind;
}

namespace {
void need(bool c, const char* msg) {
    if (!c) throw std::invalid_argument(msg);
}

pbkd::DistillTask to_task(const pbkd_task& t) {
    pbkd::DistillTask d;
    d.block_index = t.block_index;
    need(t.kind >= 0 && t.kind <= 3, "task kind out of range");
    d.kind = static_cast<pbkd::CandidateKind>(t.kind);
    d.epochs = t.epochs;
    d.eval_every = t.eval_every;
    d.seed = t.seed;
    d.threshold = t.threshold;
    need(t.loss_mode == 0 || t.loss_mode == 1, "loss mode out of range");
    d.loss_mode = static_cast<pbkd::LossMode>(t.loss_mode);
    d.lambda_local = t.lambda_local;
    d.lr = t.lr;
    d.momentum = t.momentum;
    d.batch_size = t.batch_size;
    d.max_steps = static_cast<long>(t.max_steps);
    return d;
}

pbkd::Network spec_net(const char* spec) {
    need(spec != nullptr, "null model spec");
    return pbkd::parse_model_spec(spec, "spec");
}

size_t net_floats(pbkd::Network& net) {
    size_t n = 0;
    pbkd::for_each_array(net, [&](const std::string&, pbkd::Tensor& t) { n += t.data.size(); });
    return n;
}

TaskOutcome failed_outcome(const pbkd::DistillTask& t, const std::string& why) {
    TaskOutcome r;
    r.block_index = t.block_index;
    r.kind = pbkd::candidate_kind_name(t.kind);
    r.failed = true;
    r.failure = why;
    return r;
}

double now_s(std::chrono::steady_clock::time_point t0) {
    return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// One-op launch helper for the kernel-level ABI.
template <class Op>
void launch_one(cudaStream_t st, void (*launch)(const Op*, int, int, cudaStream_t), const Op& in, int ctas) {
    Op op = in;
    op.cta_begin = 0;
    Op* d = nullptr;
    PBKD_CUDA(cudaMalloc(&d, sizeof(Op)));
    PBKD_CUDA(cudaMemcpyAsync(d, &op, sizeof(Op), cudaMemcpyHostToDevice, st));
    launch(d, 1, std::max(1, ctas), st);
    PBKD_CUDA(cudaStreamSynchronize(st));
    cudaFree(d);
}

void launch_gemm_one(cudaStream_t st, const GemmOp& g) {
    GemmOp op = g;
    op.cta_begin = 0;
    GemmOp* d = nullptr;
    PBKD_CUDA(cudaMalloc(&d, sizeof(GemmOp)));
    PBKD_CUDA(cudaMemcpyAsync(d, &op, sizeof(GemmOp), cudaMemcpyHostToDevice, st));
    launch_gemm_bn(d, 1, std::max(1, ctas_gemm(op)), gemm_bn_class(op), st);
    PBKD_CUDA(cudaStreamSynchronize(st));
    cudaFree(d);
}

struct Scratch {
    float* p = nullptr;
    explicit Scratch(size_t n) { PBKD_CUDA(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(float))); }
    ~Scratch() { cudaFree(p); }
};
}  // namespace

extern "C" {

const char* pbkd_last_error(void) { return g_err.c_str(); }
int pbkd_last_error_kind(void) { return g_kind; }
const char* pbkd_version(void) { return "pbkd-b200 0.1 (sm_100a)"; }

int pbkd_device_count(int* n) {
    return guard([&] { PBKD_CUDA(cudaGetDeviceCount(n)); });
}

int pbkd_ctx_create(int device, pbkd_ctx** out) {
    return guard([&] {
        auto c = std::make_unique<pbkd_ctx>();
        c->eng = std::make_unique<Engine>(device);
        *out = c.release();
    });
}

int pbkd_ctx_create_multi(const int* devices, int n, pbkd_ctx** out) {
    return guard([&] {
        need(n >= 1 && devices != nullptr, "device list is empty");
        std::vector<int> devs(devices, devices + n);
        for (size_t i = 0; i < devs.size(); ++i)
            for (size_t j = 0; j < i; ++j)
                if (devs[i] == devs[j]) throw std::invalid_argument("device list repeats device " + std::to_string(devs[i]));
        auto c = std::make_unique<pbkd_ctx>();
        c->eng = std::make_unique<Engine>(devs[0]);
        for (size_t i = 1; i < devs.size(); ++i) c->peers.push_back(std::make_unique<Engine>(devs[i]));
        // one NCCL clique over the list (ncclCommInitAll); a one-GPU list
        // still gets a one-rank communicator, so the exchange path is the same
        auto comms = NcclComm::clique(devs);
        const auto engs = c->engines();
        for (size_t i = 0; i < engs.size(); ++i) engs[i]->set_comm(std::move(comms[i]));
        c->multi = true;
        *out = c.release();
    });
}

int pbkd_ctx_device_count(const pbkd_ctx* ctx, int* n) {
    return guard([&] {
        need(ctx != nullptr, "null context");
        *n = static_cast<int>(ctx->engines().size());
    });
}

void pbkd_ctx_destroy(pbkd_ctx* ctx) { delete ctx; }

int pbkd_spec_num_floats(const char* spec, size_t* n) {
    return guard([&] {
        pbkd::Network net = spec_net(spec);
        *n = net_floats(net);
    });
}

int pbkd_spec_num_blocks(const char* spec, int* n) {
    return guard([&] { *n = static_cast<int>(spec_net(spec).blocks.size()); });
}

int pbkd_teacher_load(pbkd_ctx* ctx, const char* spec, const float* w, size_t n) {
    return guard([&] {
        static const bool tr = std::getenv("PBKD_TRACE") != nullptr;
        auto t0 = std::chrono::steady_clock::now();
        auto mark = [&](const char* what) {
            if (!tr) return;
            const auto now = std::chrono::steady_clock::now();
            std::fprintf(stderr, "[pbkd] teacher_load: %-22s %9.3f ms\n", what,
                         std::chrono::duration<double, std::milli>(now - t0).count());
            t0 = now;
        };
        // same spec as the loaded teacher (single engine): refill its host
        // tensors in place (no parse, no fresh pages for tens of MB)
        const bool reuse = ctx->peers.empty() && ctx->eng->has_teacher() && spec != nullptr && ctx->spec == spec &&
                           net_floats(const_cast<pbkd::Network&>(ctx->eng->teacher())) == n;
        pbkd::Network net = reuse ? ctx->eng->take_teacher() : spec_net(spec);
        mark(reuse ? "host tensors (reused)" : "parse + host tensors");
        const size_t need_n = net_floats(net);
        if (n != need_n)
            throw std::invalid_argument("teacher weights: got " + std::to_string(n) + " floats, spec needs " +
                                        std::to_string(need_n));
        // host network tensors from the caller's buffer, large tensors split
        // over a few threads (tens of MB for VGG-16)
        std::vector<std::pair<pbkd::Tensor*, size_t>> parts;
        size_t at = 0;
        pbkd::for_each_array(net, [&](const std::string&, pbkd::Tensor& t) {
            parts.emplace_back(&t, at);
            at += t.data.size();
        });
        const int nth = static_cast<int>(std::min<size_t>(8, std::max<size_t>(1, at >> 21)));
        auto copy_range = [&](size_t lo, size_t hi) {  // flat element range [lo, hi)
            for (const auto& [t, off] : parts) {
                const size_t b = std::max(lo, off), e = std::min(hi, off + t->data.size());
                if (b < e) std::copy(w + b, w + e, t->data.begin() + static_cast<std::ptrdiff_t>(b - off));
            }
        };
        std::vector<std::thread> th;
        for (int i = 1; i < nth; ++i) th.emplace_back(copy_range, at * i / nth, at * (i + 1) / nth);
        copy_range(0, at / nth);
        for (std::thread& x : th) x.join();
        mark("copy into host tensors");
        for (auto& p : ctx->peers) p->set_teacher(pbkd::Network(net), w, n);
        ctx->eng->set_teacher(std::move(net), w, n);  // device copy straight from the caller's buffer
        mark("engine load (async)");
        ctx->spec = spec;
    });
}

int pbkd_teacher_init(pbkd_ctx* ctx, const char* spec, uint64_t seed) {
    return guard([&] {
        pbkd::Network net = spec_net(spec);
        pbkd::init_weights(net, seed);
        for (auto& p : ctx->peers) p->set_teacher(net);
        ctx->eng->set_teacher(std::move(net));
        ctx->spec = spec;
    });
}

int pbkd_teacher_weights(pbkd_ctx* ctx, float* out, size_t cap) {
    return guard([&] {
        pbkd::Network net = ctx->eng->teacher();
        size_t at = 0;
        pbkd::for_each_array(net, [&](const std::string&, pbkd::Tensor& t) {
            if (at + t.data.size() > cap) throw std::length_error("buffer too small");
            std::copy(t.data.begin(), t.data.end(), out + at);
            at += t.data.size();
        });
    });
}

int pbkd_teacher_save_file(pbkd_ctx* ctx, const char* path) {
    return guard([&] { pbkd::save_weights(path, pbkd::arrays_from_network(ctx->eng->teacher())); });
}

int pbkd_teacher_load_file(pbkd_ctx* ctx, const char* spec, const char* path) {
    return guard([&] {
        pbkd::Network net = spec_net(spec);
        pbkd::load_into_network(net, pbkd::load_weights(path), path);
        for (auto& p : ctx->peers) p->set_teacher(net);
        ctx->eng->set_teacher(std::move(net));
        ctx->spec = spec;
    });
}

int pbkd_save_student_network(const char* spec, const float* teacher, size_t n_teacher, int block_index, int kind,
                              const float* block, size_t n_block, const char* path) {
    return guard([&] {
        pbkd::Network net = spec_net(spec);
        if (n_teacher != net_floats(net)) throw std::invalid_argument("teacher weights: wrong float count");
        size_t at = 0;
        pbkd::for_each_array(net, [&](const std::string&, pbkd::Tensor& t) {
            std::copy(teacher + at, teacher + at + t.data.size(), t.data.begin());
            at += t.data.size();
        });
        if (block_index < 1 || block_index > static_cast<int>(net.blocks.size()))
            throw std::out_of_range("save_student_network: block index out of range");
        pbkd::Block& tb = net.blocks[static_cast<size_t>(block_index) - 1];
        pbkd::Block sb = pbkd::build_candidate(static_cast<pbkd::CandidateKind>(kind), tb.in_channels,
                                               tb.out_channels, tb.stride, 0).block;
        sb.name = tb.name;
        size_t bn = 0;
        pbkd::for_each_block_array(sb, [&](const std::string&, pbkd::Tensor& t) { bn += t.data.size(); });
        if (bn != n_block) throw std::invalid_argument("save_student_network: wrong block float count");
        at = 0;
        pbkd::for_each_block_array(sb, [&](const std::string&, pbkd::Tensor& t) {
            std::copy(block + at, block + at + t.data.size(), t.data.begin());
            at += t.data.size();
        });
        tb = std::move(sb);
        pbkd::save_weights(path, pbkd::arrays_from_network(net));
    });
}

int pbkd_load_network_file(const char* spec, const char* path, int* block_kinds, int max_blocks, float* out,
                           size_t cap, size_t* n_out) {
    return guard([&] {
        const pbkd::Network teacher = spec_net(spec);
        const pbkd::Network net = pbkd::rebuild_network_from_arrays(teacher, pbkd::load_weights(path), path);
        for (size_t i = 0; i < net.blocks.size() && static_cast<int>(i) < max_blocks; ++i) {
            int k = 0;
            for (int c = 0; c < 4; ++c)
                if (net.blocks[i].spec_kind == pbkd::candidate_kind_name(static_cast<pbkd::CandidateKind>(c))) k = 1 + c;
            block_kinds[i] = k;
        }
        size_t at = 0;
        pbkd::for_each_array(const_cast<pbkd::Network&>(net), [&](const std::string&, pbkd::Tensor& t) {
            if (at + t.data.size() > cap) throw std::length_error("buffer too small");
            std::copy(t.data.begin(), t.data.end(), out + at);
            at += t.data.size();
        });
        *n_out = at;
    });
}

int pbkd_file_hash(const char* path, uint64_t* out) {
    return guard([&] { *out = pbkd::file_hash(path); });
}

int pbkd_dataset_load(pbkd_ctx* ctx, const float* img, const int* lab, int count, int c, int h, int w,
                      int classes) {
    return guard([&] {
        need(count > 0 && c > 0 && h > 0 && w > 0, "dataset dims must be positive");
        for (Engine* e : ctx->engines()) e->set_dataset(img, lab, count, c, h, w, classes, false);
    });
}

int pbkd_dataset_load_device(pbkd_ctx* ctx, const float* img, const int* lab, int count, int c, int h,
                             int w, int classes) {
    return guard([&] {
        need(count > 0 && c > 0 && h > 0 && w > 0, "dataset dims must be positive");
        ctx->eng->set_dataset(img, lab, count, c, h, w, classes, true);
    });
}

int pbkd_run(pbkd_ctx* ctx, const pbkd_task* tasks, int n_tasks, const int* tr, int n_tr, const int* ev,
             int n_ev, int flags, pbkd_results** out) {
    return guard([&] {
        const auto t0 = std::chrono::steady_clock::now();
        std::vector<pbkd::DistillTask> ts;
        for (int i = 0; i < n_tasks; ++i) ts.push_back(to_task(tasks[i]));
        RunOptions opt;
        opt.baseline_and_eval = (flags & PBKD_RUN_STEP_ONLY) == 0;
        opt.use_graphs = (flags & PBKD_RUN_NO_GRAPH) == 0;
        opt.profile = (flags & PBKD_RUN_PROFILE) != 0;
        auto r = std::make_unique<pbkd_results>();
        r->res = ctx->eng->run(ts, std::vector<int>(tr, tr + n_tr), std::vector<int>(ev, ev + n_ev), opt);
        r->wall = now_s(t0);
        r->epoch_ms = ctx->eng->timing().epoch_ms_total;
        r->timing = ctx->eng->timing();
        *out = r.release();
    });
}

int pbkd_run_timing(const pbkd_results* r, double* timed_ms, int* timed_epochs, long long* launches,
                    double* epoch_ms, int cap, int* n_epochs) {
    return guard([&] {
        if (timed_ms) *timed_ms = r->timing.timed_ms;
        if (epoch_ms && cap < 0) {  // cap < 0: epoch_ms[0] receives the teacher part instead
            epoch_ms[0] = r->timing.teacher_ms;
            return;
        }
        if (timed_epochs) *timed_epochs = r->timing.timed_epochs;
        if (launches) *launches = r->timing.launches;
        if (n_epochs) *n_epochs = static_cast<int>(r->timing.epoch_ms.size());
        if (epoch_ms)
            for (int i = 0; i < std::min<int>(cap, static_cast<int>(r->timing.epoch_ms.size())); ++i)
                epoch_ms[i] = r->timing.epoch_ms[static_cast<size_t>(i)];
    });
}

int pbkd_run_timed(pbkd_ctx* ctx, const pbkd_task* tasks, int n_tasks, const int* tr, int n_tr, const int* ev,
                   int n_ev, int flags, int timed_from_epoch, pbkd_results** out) {
    return guard([&] {
        const auto t0 = std::chrono::steady_clock::now();
        std::vector<pbkd::DistillTask> ts;
        for (int i = 0; i < n_tasks; ++i) ts.push_back(to_task(tasks[i]));
        RunOptions opt;
        opt.baseline_and_eval = (flags & PBKD_RUN_STEP_ONLY) == 0;
        opt.use_graphs = (flags & PBKD_RUN_NO_GRAPH) == 0;
        opt.profile = (flags & PBKD_RUN_PROFILE) != 0;
        opt.timed_from_epoch = timed_from_epoch;
        auto r = std::make_unique<pbkd_results>();
        r->res = ctx->eng->run(ts, std::vector<int>(tr, tr + n_tr), std::vector<int>(ev, ev + n_ev), opt);
        r->wall = now_s(t0);
        r->epoch_ms = ctx->eng->timing().epoch_ms_total;
        r->timing = ctx->eng->timing();
        *out = r.release();
    });
}

int pbkd_bench_kernel(pbkd_ctx* ctx, int which, int batch, int iters, double* ms, double* bytes,
                      double* flops) {
    return guard([&] { ctx->eng->bench_kernel(which, batch, iters, ms, bytes, flops); });
}

int pbkd_nccl_unique_id(char* out128) {
    return guard([&] { nccl_unique_id(out128); });
}

int pbkd_ctx_set_comm(pbkd_ctx* ctx, const char* id128, int rank, int world) {
    return guard([&] {
        if (world < 1 || rank < 0 || rank >= world) throw std::invalid_argument("bad rank/world");
        ctx->eng->set_comm(id128, rank, world);
    });
}

int pbkd_run_sharded(pbkd_ctx* ctx, const pbkd_task* tasks, int n_tasks, const int* tr, int n_tr, const int* ev,
                     int n_ev, int flags, int timed_from_epoch, const int* g_blocks, const int* g_owner, int n_global,
                     int virtual_shards, const double* share, int n_share, pbkd_results** out) {
    return guard([&] {
        const auto t0 = std::chrono::steady_clock::now();
        std::vector<pbkd::DistillTask> ts;
        for (int i = 0; i < n_tasks; ++i) ts.push_back(to_task(tasks[i]));
        RunOptions opt;
        opt.baseline_and_eval = (flags & PBKD_RUN_STEP_ONLY) == 0;
        opt.use_graphs = (flags & PBKD_RUN_NO_GRAPH) == 0;
        opt.profile = (flags & PBKD_RUN_PROFILE) != 0;
        opt.timed_from_epoch = timed_from_epoch;
        for (int i = 0; i < n_global; ++i) opt.global_blocks.push_back({g_blocks[i], g_owner[i]});
        opt.virtual_shards = virtual_shards;
        if (share) opt.shard_share.assign(share, share + n_share);
        auto r = std::make_unique<pbkd_results>();
        r->res = ctx->eng->run(ts, std::vector<int>(tr, tr + n_tr), std::vector<int>(ev, ev + n_ev), opt);
        r->wall = now_s(t0);
        r->epoch_ms = ctx->eng->timing().epoch_ms_total;
        r->timing = ctx->eng->timing();
        *out = r.release();
    });
}

int pbkd_exchange_plan(const int* blocks, const int* owners, int nb, const long long* rows, int n_rows, int world,
                       int n_train, const double* share, int src, int dst, size_t* count, int* xj, int* xrow0,
                       int* xrows, int cap, int* n, int* shard_begin) {
    return guard([&] {
        need(world >= 1 && src >= 0 && src < world && dst >= 0 && dst < world, "bad src / dst / world");
        std::vector<double> sh = share ? std::vector<double>(share, share + world) : std::vector<double>();
        const BoundaryPlan p = make_boundary_plan(std::vector<int>(blocks, blocks + nb),
                                                  std::vector<int>(owners, owners + nb),
                                                  std::vector<long long>(rows, rows + n_rows), world, n_train, sh);
        const std::vector<BoundaryPlan::Xfer> xs = p.transfers(src, dst);
        *count = p.count(src, dst);
        *n = static_cast<int>(xs.size());
        for (int i = 0; i < std::min(cap, *n); ++i) {
            xj[i] = xs[static_cast<size_t>(i)].j;
            xrow0[i] = xs[static_cast<size_t>(i)].row0;
            xrows[i] = xs[static_cast<size_t>(i)].rows;
        }
        for (int s2 = 0; s2 <= world; ++s2) shard_begin[s2] = p.shard_begin[static_cast<size_t>(s2)];
    });
}

int pbkd_run_parallel(pbkd_ctx* ctx, const pbkd_task* tasks, int n_tasks, const int* tr, int n_tr,
                      const int* ev, int n_ev, int workers, int policy, const int* plan_ids,
                      const int* plan_counts, int flags, pbkd_results** out) {
    return guard([&] {
        // plan validation (runtime.cpp:127-156)
        if (workers < 1) throw pbkd::SpecError("worker_count must be at least 1");
        need(policy >= 0 && policy <= 2, "policy out of range");
        std::map<int, int> by_id;
        for (int i = 0; i < n_tasks; ++i)
            if (!by_id.emplace(tasks[i].block_index, i).second)
                throw pbkd::SpecError("two tasks reference block " + std::to_string(tasks[i].block_index));
        std::vector<std::vector<int>> queues(static_cast<size_t>(workers));
        std::set<int> seen;
        int at = 0;
        for (int w = 0; w < workers; ++w)
            for (int j = 0; j < plan_counts[w]; ++j) {
                const int id = plan_ids[at++];
                if (!by_id.count(id)) throw pbkd::SpecError("plan references unknown task id " + std::to_string(id));
                if (!seen.insert(id).second) throw pbkd::SpecError("plan assigns task " + std::to_string(id) + " twice");
                queues[static_cast<size_t>(w)].push_back(id);
            }
        if (static_cast<int>(seen.size()) != n_tasks)
            throw pbkd::SpecError("plan covers " + std::to_string(seen.size()) + " of " + std::to_string(n_tasks) +
                                  " tasks");
        const auto t0 = std::chrono::steady_clock::now();
        auto r = std::make_unique<pbkd_results>();
        // sync point 1: dispatch
        for (int w = 0; w < workers; ++w)
            for (int id : queues[static_cast<size_t>(w)]) r->trace.push_back({now_s(t0), w, id, 0});
        // every worker of this process maps onto this context's GPU; tasks the
        // engine rejects become failed results (runtime.cpp:212-220)
        std::vector<pbkd::DistillTask> ok;
        std::map<int, TaskOutcome> outcome;
        std::map<int, int> worker_of;
        for (int w = 0; w < workers; ++w)
            for (int id : queues[static_cast<size_t>(w)]) worker_of[id] = w;
        // per-task validation inside the per-task try (train_block throws,
        // run_parallel turns it into a failed result: runtime.cpp:212-220)
        const std::vector<int> trv(tr, tr + n_tr), evv(ev, ev + n_ev);
        for (int i = 0; i < n_tasks; ++i) {
            pbkd::DistillTask t = to_task(tasks[i]);
            try {
                ctx->eng->validate(t);
                ctx->eng->check_split(trv, evv);
                ok.push_back(t);
            } catch (const std::exception& e) {
                outcome[t.block_index] = failed_outcome(t, e.what());
                r->trace.push_back({now_s(t0), worker_of[t.block_index], t.block_index, 1});
                r->trace.push_back({now_s(t0), worker_of[t.block_index], t.block_index, 2});
            }
        }
        for (const pbkd::DistillTask& t : ok) r->trace.push_back({now_s(t0), worker_of[t.block_index], t.block_index, 1});
        RunOptions opt;
        opt.baseline_and_eval = (flags & PBKD_RUN_STEP_ONLY) == 0;
        opt.use_graphs = (flags & PBKD_RUN_NO_GRAPH) == 0;
        opt.profile = (flags & PBKD_RUN_PROFILE) != 0;
        if (!ok.empty() && !ctx->multi) {
            // a single-GPU context: every worker's tasks train on this GPU,
            // grouped (results do not depend on the grouping)
            std::vector<TaskOutcome> res = ctx->eng->run(ok, trv, evv, opt);
            for (TaskOutcome& o : res) outcome[o.block_index] = std::move(o);
            r->epoch_ms = ctx->eng->timing().epoch_ms_total;
            r->timing = ctx->eng->timing();
            for (const pbkd::DistillTask& t : ok)
                r->trace.push_back({now_s(t0), worker_of[t.block_index], t.block_index, 2});
        } else if (!ok.empty()) {
            // a context over a GPU list: worker w runs on GPU w % G, one host
            // thread per GPU (runtime.cpp:226-233); the GPUs share the teacher
            // forward (sample shards) and exchange boundary rows once over the
            // NCCL clique; every block trains on its own GPU with no
            // cross-block synchronisation
            const std::vector<Engine*> engs = ctx->engines();
            const int G = static_cast<int>(engs.size());
            std::map<int, pbkd::DistillTask> task_of;
            for (const pbkd::DistillTask& t : ok) task_of[t.block_index] = t;
            std::vector<std::deque<int>> gq(static_cast<size_t>(G));
            for (int w = 0; w < workers; ++w)
                for (int id : queues[static_cast<size_t>(w)])
                    if (task_of.count(id)) gq[static_cast<size_t>(w % G)].push_back(id);
            if (policy == static_cast<int>(pbkd::SchedulePolicy::WorkStealing)) {
                // runtime.cpp:178-206 at dispatch granularity: an idle GPU takes
                // the tail of the queue with the most remaining teacher MACs
                std::vector<int> ids;
                for (const auto& kv : task_of) ids.push_back(kv.first);
                const auto wts = pbkd::mac_proxy_weights(ctx->eng->teacher(), ids);
                std::map<int, double> wt;
                for (const pbkd::TaskWeight& x : wts) wt[x.task_id] = x.weight;
                for (int g = 0; g < G; ++g) {
                    if (!gq[static_cast<size_t>(g)].empty()) continue;
                    int victim = -1;
                    double most = 0.0;
                    for (int v = 0; v < G; ++v) {
                        if (gq[static_cast<size_t>(v)].size() < 2) continue;
                        double sum = 0.0;
                        for (int id : gq[static_cast<size_t>(v)]) sum += wt[id];
                        if (sum > most) most = sum, victim = v;
                    }
                    if (victim < 0) break;
                    const int id = gq[static_cast<size_t>(victim)].back();
                    gq[static_cast<size_t>(victim)].pop_back();
                    gq[static_cast<size_t>(g)].push_back(id);
                    worker_of[id] = g;
                    r->trace.push_back({now_s(t0), g, id, 3});
                }
            }
            std::vector<std::pair<int, int>> global;
            for (int g = 0; g < G; ++g)
                for (int id : gq[static_cast<size_t>(g)]) global.push_back({id, g});
            std::vector<std::vector<TaskOutcome>> res(static_cast<size_t>(G));
            std::vector<std::string> err(static_cast<size_t>(G));
            std::vector<std::thread> th;
            for (int g = 0; g < G; ++g)
                th.emplace_back([&, g] {
                    try {
                        std::vector<pbkd::DistillTask> mine;
                        for (int id : gq[static_cast<size_t>(g)]) mine.push_back(task_of[id]);
                        RunOptions o = opt;
                        o.global_blocks = global;
                        res[static_cast<size_t>(g)] = engs[static_cast<size_t>(g)]->run(mine, trv, evv, o);
                    } catch (const std::exception& e) {
                        err[static_cast<size_t>(g)] = e.what();
                    }
                });
            for (std::thread& x : th) x.join();
            for (int g = 0; g < G; ++g)
                if (!err[static_cast<size_t>(g)].empty())
                    throw std::runtime_error("GPU " + std::to_string(g) + ": " + err[static_cast<size_t>(g)]);
            for (auto& v : res)
                for (TaskOutcome& o : v) outcome[o.block_index] = std::move(o);
            r->timing = ctx->eng->timing();
            for (Engine* e : engs) r->epoch_ms = std::max(r->epoch_ms, e->timing().epoch_ms_total);
            for (const pbkd::DistillTask& t : ok)
                r->trace.push_back({now_s(t0), worker_of[t.block_index], t.block_index, 2});
        }
        // sync point 2: gather in task-id order
        for (auto& kv : outcome) r->res.push_back(std::move(kv.second));
        r->trace.push_back({now_s(t0), 0, -1, 4});
        r->wall = r->trace.back().timestamp_s;
        *out = r.release();
    });
}

int pbkd_run_count(const pbkd_results* r) { return r ? static_cast<int>(r->res.size()) : 0; }

int pbkd_run_profile_count(const pbkd_results* r) { return r ? static_cast<int>(r->timing.prof.size()) : 0; }

int pbkd_run_profile_entry(const pbkd_results* r, int i, char* name, size_t cap, int* launches, double* ms,
                           double* bytes, double* flops) {
    return guard([&] {
        need(i >= 0 && i < static_cast<int>(r->timing.prof.size()), "profile entry out of range");
        auto it = r->timing.prof.begin();
        std::advance(it, i);
        if (name && cap) {
            std::strncpy(name, it->first.c_str(), cap - 1);
            name[cap - 1] = 0;
        }
        *launches = it->second.launches;
        *ms = it->second.ms;
        *bytes = it->second.bytes;
        *flops = it->second.flops;
    });
}

int pbkd_run_info(const pbkd_results* r, int i, pbkd_result_info* info) {
    return guard([&] {
        const TaskOutcome& o = r->res.at(static_cast<size_t>(i));
        std::memset(info, 0, sizeof(*info));
        info->block_index = o.block_index;
        info->failed = o.failed ? 1 : 0;
        std::strncpy(info->kind, o.kind.c_str(), sizeof(info->kind) - 1);
        std::strncpy(info->failure, o.failure.c_str(), sizeof(info->failure) - 1);
        info->n_loss = static_cast<int>(o.loss_history.size());
        info->n_eval = static_cast<int>(o.eval_history.size());
        info->n_steps = static_cast<long long>(o.step_losses.size());
        info->n_block_floats = o.final_block.size();
        info->has_best = o.best_block.empty() ? 0 : 1;
        info->final_local_loss = o.final_local_loss;
        info->best_eval = o.best_eval;
        info->wall_time_s = o.wall_time_s;
    });
}

int pbkd_run_loss_history(const pbkd_results* r, int i, double* out, int cap) {
    return guard([&] {
        const auto& v = r->res.at(static_cast<size_t>(i)).loss_history;
        if (static_cast<int>(v.size()) > cap) throw std::length_error("buffer too small");
        std::copy(v.begin(), v.end(), out);
    });
}

int pbkd_run_eval_history(const pbkd_results* r, int i, int* epochs, double* acc, int cap) {
    return guard([&] {
        const auto& v = r->res.at(static_cast<size_t>(i)).eval_history;
        if (static_cast<int>(v.size()) > cap) throw std::length_error("buffer too small");
        for (size_t k = 0; k < v.size(); ++k) {
            epochs[k] = v[k].epoch;
            acc[k] = v[k].accuracy;
        }
    });
}

int pbkd_run_block(const pbkd_results* r, int i, int which, float* out, size_t cap) {
    return guard([&] {
        const TaskOutcome& o = r->res.at(static_cast<size_t>(i));
        const std::vector<float>& v = which == 0 ? o.best_block : o.final_block;
        if (v.size() > cap) throw std::length_error("buffer too small");
        std::copy(v.begin(), v.end(), out);
    });
}

int pbkd_run_step_losses(const pbkd_results* r, int i, float* out, long long cap) {
    return guard([&] {
        const auto& v = r->res.at(static_cast<size_t>(i)).step_losses;
        if (static_cast<long long>(v.size()) > cap) throw std::length_error("buffer too small");
        std::copy(v.begin(), v.end(), out);
    });
}

int pbkd_run_trace(const pbkd_results* r, pbkd_trace_event* out, int cap, int* n) {
    return guard([&] {
        *n = static_cast<int>(r->trace.size());
        for (int k = 0; k < std::min(cap, *n); ++k) out[k] = r->trace[static_cast<size_t>(k)];
    });
}

double pbkd_run_wall_time(const pbkd_results* r) { return r ? r->wall : 0.0; }
double pbkd_run_epoch_ms(const pbkd_results* r) { return r ? r->epoch_ms : 0.0; }
void pbkd_run_free(pbkd_results* r) { delete r; }

int pbkd_prefix_infer(pbkd_ctx* ctx, const float* x, int n, int k, int inclusive, float* out, size_t cap,
                      int* shape) {
    return guard([&] {
        const pbkd::Network& net = ctx->eng->teacher();
        pbkd::Tensor t(n, net.in_c, net.in_h, net.in_w);
        std::copy(x, x + t.size(), t.data.begin());
        pbkd::Tensor y = ctx->eng->prefix_infer(t, k, inclusive != 0);
        if (y.size() > cap) throw std::length_error("buffer too small");
        std::copy(y.data.begin(), y.data.end(), out);
        shape[0] = y.n, shape[1] = y.c, shape[2] = y.h, shape[3] = y.w;
    });
}

static pbkd::Block block_from_flat(int kind, int cin, int cout, int stride, const float* w) {
    pbkd::ReplacementBlock rb = pbkd::build_candidate(static_cast<pbkd::CandidateKind>(kind), cin, cout, stride, 0);
    size_t at = 0;
    pbkd::for_each_block_array(rb.block, [&](const std::string&, pbkd::Tensor& t) {
        std::copy(w + at, w + at + t.data.size(), t.data.begin());
        at += t.data.size();
    });
    return rb.block;
}

int pbkd_candidate_infer(pbkd_ctx* ctx, int kind, int cin, int cout, int stride, const float* bw,
                         const float* x, int n, int h, int w, float* out, size_t cap) {
    return guard([&] {
        pbkd::Block b = block_from_flat(kind, cin, cout, stride, bw);
        pbkd::Tensor t(n, cin, h, w);
        std::copy(x, x + t.size(), t.data.begin());
        pbkd::Tensor y = ctx->eng->candidate_infer(b, t);
        if (y.size() > cap) throw std::length_error("buffer too small");
        std::copy(y.data.begin(), y.data.end(), out);
    });
}

int pbkd_eval_with_student(pbkd_ctx* ctx, int k, int kind, const float* sw, const int* ev, int n_ev,
                           int batch_size, double* acc) {
    return guard([&] {
        if (batch_size < 1) throw pbkd::SpecError("batch_size must be at least 1");
        const pbkd::Network& net = ctx->eng->teacher();
        if (k < 1 || k > static_cast<int>(net.blocks.size()))
            throw pbkd::SpecError("block index " + std::to_string(k) + " out of range");
        const pbkd::Block& tb = net.blocks[static_cast<size_t>(k) - 1];
        pbkd::Block b = block_from_flat(kind, tb.in_channels, tb.out_channels, tb.stride, sw);
        *acc = ctx->eng->eval_with_student(k, b, std::vector<int>(ev, ev + n_ev));
    });
}

uint64_t pbkd_mix_seed(uint64_t a, uint64_t b) { return pbkd::mix_seed(a, b); }

int pbkd_stratified_split(const int* labels, int n, double frac, uint64_t seed, int* tr, int* ntr, int* ev,
                          int* nev) {
    return guard([&] {
        pbkd::Dataset d;
        d.labels.assign(labels, labels + n);
        pbkd::SplitIndices s = pbkd::stratified_split(d, frac, seed);
        std::copy(s.train_idx.begin(), s.train_idx.end(), tr);
        std::copy(s.eval_idx.begin(), s.eval_idx.end(), ev);
        *ntr = static_cast<int>(s.train_idx.size());
        *nev = static_cast<int>(s.eval_idx.size());
    });
}

int pbkd_epoch_order(const int* tr, int n, uint64_t seed, int epoch, int* out) {
    return guard([&] {
        const std::vector<int> o = pbkd::epoch_order(std::vector<int>(tr, tr + n), seed, epoch);
        std::copy(o.begin(), o.end(), out);
    });
}

int pbkd_build_candidate(int kind, int cin, int cout, int stride, uint64_t seed, float* out, size_t cap,
                         size_t* n) {
    return guard([&] {
        need(kind >= 0 && kind <= 3, "candidate kind out of range");
        pbkd::ReplacementBlock rb = pbkd::build_candidate(static_cast<pbkd::CandidateKind>(kind), cin, cout, stride, seed);
        size_t at = 0;
        pbkd::for_each_block_array(rb.block, [&](const std::string&, pbkd::Tensor& t) {
            if (out) {
                if (at + t.data.size() > cap) throw std::length_error("buffer too small");
                std::copy(t.data.begin(), t.data.end(), out + at);
            }
            at += t.data.size();
        });
        if (n) *n = at;
    });
}

static void plan_out(const pbkd::SchedulePlan& p, int* ids, int* counts) {
    int at = 0;
    for (size_t w = 0; w < p.assignments.size(); ++w) {
        counts[w] = static_cast<int>(p.assignments[w].size());
        for (int id : p.assignments[w]) ids[at++] = id;
    }
}

int pbkd_round_robin(const int* ids, int n, int workers, int* out_ids, int* out_counts) {
    return guard([&] { plan_out(pbkd::round_robin(std::vector<int>(ids, ids + n), workers), out_ids, out_counts); });
}

int pbkd_wfd_bin_pack(const int* ids, const double* w, int n, int workers, int* out_ids, int* out_counts,
                      double* mk) {
    return guard([&] {
        std::vector<pbkd::TaskWeight> tw;
        for (int i = 0; i < n; ++i) tw.push_back({ids[i], w[i]});
        pbkd::SchedulePlan p = pbkd::wfd_bin_pack(tw, workers);
        plan_out(p, out_ids, out_counts);
        if (mk) *mk = p.predicted_makespan;
    });
}

int pbkd_makespan(const int* plan_ids, const int* plan_counts, int workers, const int* ids, const double* w,
                  int n, double* out) {
    return guard([&] {
        pbkd::SchedulePlan p;
        p.worker_count = workers;
        p.assignments.resize(static_cast<size_t>(workers));
        int at = 0;
        for (int k = 0; k < workers; ++k)
            for (int j = 0; j < plan_counts[k]; ++j) p.assignments[static_cast<size_t>(k)].push_back(plan_ids[at++]);
        std::vector<pbkd::TaskWeight> tw;
        for (int i = 0; i < n; ++i) tw.push_back({ids[i], w[i]});
        *out = pbkd::makespan(p, tw);
    });
}

int pbkd_mac_proxy_weights(const char* spec, const int* blocks, int n, double* out) {
    return guard([&] {
        pbkd::Network net = spec_net(spec);
        const std::vector<pbkd::TaskWeight> w = pbkd::mac_proxy_weights(net, std::vector<int>(blocks, blocks + n));
        for (int i = 0; i < n; ++i) out[i] = w[static_cast<size_t>(i)].weight;
    });
}

// -------------------------------------------------------- kernel level --
int pbkd_k_dw_fwd(pbkd_ctx* ctx, const float* x, const float* w, float* y, int n, int h, int wd, int c,
                  int stride, int pad) {
    return guard([&] {
        DwFwdOp o{};
        o.x = x;
        o.w = w;
        o.y = y;
        o.n = n;
        o.h = h;
        o.wd = wd;
        o.c = c;
        o.ho = (h + 2 * pad - 3) / stride + 1;
        o.wo = (wd + 2 * pad - 3) / stride + 1;
        o.stride = stride;
        o.pad = pad;
        dw_fwd_finalize(o);
        launch_one(ctx->eng->stream(), launch_dw_fwd, o, ctas_dw_fwd(o));
    });
}

int pbkd_k_dw_bwd(pbkd_ctx* ctx, const float* gy, const float* p, const float* w, const float* mean,
                  const float* inv, const float* gamma, const float* beta, float* gyp, float* gk, float* sg,
                  float* sgx, int n, int h, int wd, int c) {
    return guard([&] {
        if (c % 4 != 0 && c > kThreads) throw std::invalid_argument("dw_bwd: unsupported channel count");
        const long long rows = static_cast<long long>(n) * h * wd;
        DwBwdOp o{};
        o.gy = gy;
        o.xp = p;
        o.w = w;
        o.gyprev = gyp;
        o.mean = mean;
        o.inv = inv;
        o.gamma = gamma;
        o.beta = beta;
        o.n = n;
        o.h = h;
        o.wd = wd;
        o.c = c;
        dw_bwd_finalize(o);
        Scratch pgk(static_cast<size_t>(o.ctas) * 9 * c), psg(static_cast<size_t>(o.ctas) * c),
            psgx(static_cast<size_t>(o.ctas) * c);
        o.part_gk = pgk.p;
        o.part_sg = psg.p;
        o.part_sgx = psgx.p;
        cudaStream_t st = ctx->eng->stream();
        launch_one(st, launch_dw_bwd, o, ctas_dw_bwd(o));
        ReduceOp r{};
        r.part = pgk.p, r.out = gk, r.parts = o.ctas, r.width = 9 * c;
        launch_one(st, launch_reduce, r, ctas_reduce(r));
        r.part = psg.p, r.out = sg, r.width = c;
        launch_one(st, launch_reduce, r, ctas_reduce(r));
        r.part = psgx.p, r.out = sgx;
        launch_one(st, launch_reduce, r, ctas_reduce(r));
    });
}

int pbkd_k_dw_gk(pbkd_ctx* ctx, const float* gy, const float* x, float* gk, int n, int h, int wd, int c,
                 int stride, int pad) {
    return guard([&] {
        if (c % 4 != 0 && c > kThreads) throw std::invalid_argument("dw_gk: unsupported channel count");
        DwGkOp o{};
        o.gy = gy;
        o.x = x;
        o.n = n;
        o.h = h;
        o.wd = wd;
        o.c = c;
        o.ho = (h + 2 * pad - 3) / stride + 1;
        o.wo = (wd + 2 * pad - 3) / stride + 1;
        o.stride = stride;
        o.pad = pad;
        const long long rows = static_cast<long long>(n) * o.ho * o.wo;
        dw_gk_finalize(o);
        Scratch pgk(static_cast<size_t>(o.ctas) * 9 * c);
        o.part_gk = pgk.p;
        cudaStream_t st = ctx->eng->stream();
        launch_one(st, launch_dw_gk, o, ctas_dw_gk(o));
        ReduceOp r{};
        r.part = pgk.p, r.out = gk, r.parts = o.ctas, r.width = 9 * c;
        launch_one(st, launch_reduce, r, ctas_reduce(r));
    });
}

// PBKD_GEMM_PRESPLIT=1 (tests): hand the GEMMs pre-split tf32 planes of
// their operands, exercising the TMA kernel's no-conversion paths (K-major
// and MN-major); results must be bitwise those of the converting paths.
struct Planes {
    std::unique_ptr<Scratch> hi, lo;
    const float* h = nullptr;
    const float* l = nullptr;
    Planes(const float* x, size_t n, cudaStream_t st) {
        static const bool on = [] {
            const char* e = std::getenv("PBKD_GEMM_PRESPLIT");
            return e && e[0] == '1';
        }();
        if (!on || !x) return;
        hi = std::make_unique<Scratch>(n);
        lo = std::make_unique<Scratch>(n);
        launch_tf32_split(x, static_cast<long long>(n), hi->p, lo->p, st);
        h = hi->p;
        l = lo->p;
    }
};

int pbkd_k_pw_fwd(pbkd_ctx* ctx, const float* x, const float* w, float* y, int rows, int cin, int cout,
                  float* col_sum, float* col_sq) {
    return guard([&] {
        cudaStream_t st = ctx->eng->stream();
        Planes px(x, static_cast<size_t>(rows) * cin, st), pw(w, static_cast<size_t>(cout) * cin, st);
        GemmOp g{};
        g.M = rows, g.N = cout, g.K = cin;
        g.A = x, g.lda = cin, g.a_kmajor = 1;
        g.B = w, g.ldb = cin, g.b_kmajor = 1;
        g.a_hi = px.h, g.a_lo = px.l, g.a_ts_req = 1, g.b_hi = pw.h, g.b_lo = pw.l;
        g.C = y, g.ldc = cout;
        g.ksplit = 1;
        gemm_finalize(g);
        if (col_sum || col_sq) {
            Scratch p0(static_cast<size_t>(g.tiles_m) * cout), p1(static_cast<size_t>(g.tiles_m) * cout);
            g.epi = 1, g.part0 = p0.p, g.part1 = p1.p;
            launch_gemm_one(st, g);
            ReduceOp r{};
            r.parts = g.tiles_m, r.width = cout;
            if (col_sum) {
                r.part = p0.p, r.out = col_sum;
                launch_one(st, launch_reduce, r, ctas_reduce(r));
            }
            if (col_sq) {
                r.part = p1.p, r.out = col_sq;
                launch_one(st, launch_reduce, r, ctas_reduce(r));
            }
        } else {
            launch_gemm_one(st, g);
        }
    });
}

int pbkd_k_pw_bwd(pbkd_ctx* ctx, const float* x, const float* w, const float* gy, float* gx, float* gw,
                  int rows, int cin, int cout) {
    return guard([&] {
        cudaStream_t st = ctx->eng->stream();
        Planes px(x, static_cast<size_t>(rows) * cin, st), pw(w, static_cast<size_t>(cout) * cin, st),
            pg(gy, static_cast<size_t>(rows) * cout, st);
        if (gx) {
            GemmOp g{};
            g.M = rows, g.N = cin, g.K = cout;
            g.A = gy, g.lda = cout, g.a_kmajor = 1;
            g.B = w, g.ldb = cin, g.b_kmajor = 0;
            g.a_hi = pg.h, g.a_lo = pg.l, g.a_ts_req = 1, g.b_hi = pw.h, g.b_lo = pw.l;
            g.C = gx, g.ldc = cin;
            g.ksplit = 1;
            gemm_finalize(g);
            launch_gemm_one(st, g);
        }
        if (gw) {
            const int splits = std::max(1, std::min(64, ceil_div(rows, 512)));
            Scratch part(static_cast<size_t>(splits) * cout * cin);
            GemmOp g{};
            g.M = cout, g.N = cin, g.K = rows;
            g.A = gy, g.lda = cout, g.a_kmajor = 0;
            g.B = x, g.ldb = cin, g.b_kmajor = 0;
            g.a_hi = pg.h, g.a_lo = pg.l, g.a_ts_req = 1, g.b_hi = px.h, g.b_lo = px.l;
            g.ldc = cin;
            g.epi = 2;
            g.ksplit = splits;
            g.C = part.p;
            gemm_finalize(g);
            launch_gemm_one(st, g);
            ReduceOp r{};
            r.part = part.p, r.out = gw, r.parts = g.ksplit, r.width = cout * cin;
            launch_one(st, launch_reduce, r, ctas_reduce(r));
        }
    });
}

int pbkd_k_sgd(pbkd_ctx* ctx, float* w, const float* g, float* v, size_t n, float lr, float m) {
    return guard([&] {
        if (!(lr > 0.0f)) throw std::invalid_argument("sgd_step: lr must be > 0");
        if (m < 0.0f || m >= 1.0f) throw std::invalid_argument("sgd_step: momentum must be in [0,1)");
        SgdOp o{};
        o.w = w, o.v = v, o.g = g, o.n = static_cast<long long>(n), o.lr = lr, o.mom = m;
        launch_one(ctx->eng->stream(), launch_sgd, o, ctas_sgd(o.n));
    });
}

int pbkd_sgd_host(float* w, const float* g, float* v, size_t n, float lr, float m) {
    return guard([&] {
        if (!(lr > 0.0f)) throw std::invalid_argument("sgd_step: lr must be > 0");
        if (m < 0.0f || m >= 1.0f) throw std::invalid_argument("sgd_step: momentum must be in [0,1)");
        if (n == 0) return;
        Scratch dw(n), dg(n), dv(n);
        PBKD_CUDA(cudaMemcpy(dw.p, w, n * 4, cudaMemcpyHostToDevice));
        PBKD_CUDA(cudaMemcpy(dg.p, g, n * 4, cudaMemcpyHostToDevice));
        PBKD_CUDA(cudaMemcpy(dv.p, v, n * 4, cudaMemcpyHostToDevice));
        SgdOp o{};
        o.w = dw.p, o.v = dv.p, o.g = dg.p, o.n = static_cast<long long>(n), o.lr = lr, o.mom = m;
        launch_one(cudaStream_t(0), launch_sgd, o, ctas_sgd(o.n));
        PBKD_CUDA(cudaMemcpy(w, dw.p, n * 4, cudaMemcpyDeviceToHost));
        PBKD_CUDA(cudaMemcpy(v, dv.p, n * 4, cudaMemcpyDeviceToHost));
    });
}

}  // extern "C"
