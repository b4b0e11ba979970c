// engine.cu -- per-GPU distillation engine (see engine.hpp).
#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cctype>
#include <cstdio>
#include <thread>
#include <typeinfo>
#include <cstdlib>
#include <cstring>
#include <map>
#include <queue>
#include <set>
#include <numeric>
#include <sstream>

#include "comm.hpp"
#include "engine.hpp"
#include "nettrain.hpp"
#include "ops.cuh"
#include "pbkd/dataset.hpp"
#include "pbkd/replacement.hpp"

namespace pbkd_gpu {

using pbkd::Block;
using pbkd::DistillTask;
using pbkd::LayerKind;
using pbkd::Network;
using pbkd::SpecError;
using pbkd::Tensor;

namespace {


// PBKD_TRACE=1: host wall time of each phase of run() on stderr (synchronises
// the stream at every mark, so only for diagnosis).
struct PhaseTrace {
    bool on = std::getenv("PBKD_TRACE") != nullptr;
    cudaStream_t st = nullptr;
    std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
    void mark(const char* what) {
        if (!on) return;
        cudaStreamSynchronize(st);
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[pbkd] %-28s %9.3f ms\n", what,
                     std::chrono::duration<double, std::milli>(now - t).count());
        t = now;
    }
};

// ------------------------------------------------------------ device memory
// Buffers come from the device's stream-ordered memory pool on the engine
// stream (release threshold: keep everything), so the per-run allocations of
// activation streams and workspaces are pool hits after the first run instead
// of cudaMalloc/cudaFree round trips.  g_alloc_stream is set by every Engine
// entry point (thread-local: one engine per thread at a time).
thread_local cudaStream_t g_alloc_stream = nullptr;

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    cudaStream_t s = nullptr;
    DevBuf() = default;
    explicit DevBuf(size_t n) { alloc(n); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    DevBuf(DevBuf&& o) noexcept : p(o.p), bytes(o.bytes), s(o.s) { o.p = nullptr, o.bytes = 0; }
    DevBuf& operator=(DevBuf&& o) noexcept {
        release();
        p = o.p, bytes = o.bytes, s = o.s;
        o.p = nullptr, o.bytes = 0;
        return *this;
    }
    ~DevBuf() { release(); }
    void alloc(size_t n) {
        release();
        bytes = std::max<size_t>(n, 16);
        s = g_alloc_stream;
        PBKD_CUDA(cudaMallocAsync(&p, bytes, s));
    }
    void release() {
        if (p) cudaFreeAsync(p, s);
        p = nullptr;
        bytes = 0;
    }
    float* f() const { return static_cast<float*>(p); }
    int* i() const { return static_cast<int*>(p); }
    double* d() const { return static_cast<double*>(p); }
};

template <class T>
DevBuf upload(const std::vector<T>& v, cudaStream_t st) {
    DevBuf b(v.size() * sizeof(T));
    if (!v.empty()) PBKD_CUDA(cudaMemcpyAsync(b.p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, st));
    return b;
}

// The forward GEMM takes the raw dw output through TMEM (PBKD_FWD_TS=0:
// pre-split planes written by the dw forward).
bool fwd_ts_on() {
    static const bool on = [] {
        const char* e = std::getenv("PBKD_FWD_TS");
        return !(e && e[0] == '0') && gemm_ts_enabled();
    }();
    return on;
}

// ------------------------------------------------------- algorithmic work
// Compulsory fp32 bytes and flops of one op: what the kernel must
// move / compute at minimum, not what it does move (pre-split operand planes,
// halo re-reads and partial sums are overheads against these).
using Work = std::pair<double, double>;
double el(long long a, long long b = 1, long long c = 1, long long d = 1) {
    return static_cast<double>(a) * static_cast<double>(b) * static_cast<double>(c) * static_cast<double>(d);
}
Work op_work(const DwFwdOp& o) {
    return {4.0 * (el(o.n, o.h, o.wd, o.c) + el(o.n, o.ho, o.wo, o.c)), 18.0 * el(o.n, o.ho, o.wo, o.c)};
}
Work op_work(const DwBwdOp& o) { return {12.0 * el(o.n, o.h, o.wd, o.c), 36.0 * el(o.n, o.h, o.wd, o.c)}; }
Work op_work(const DwGkOp& o) {
    return {4.0 * (el(o.n, o.h, o.wd, o.c) + el(o.n, o.ho, o.wo, o.c)), 18.0 * el(o.n, o.ho, o.wo, o.c)};
}
Work op_work(const ReduceOp& o) { return {4.0 * (el(o.parts, o.width) + o.width), el(o.parts, o.width)}; }
Work op_work(const BnStatOp& o) { return {8.0 * el(o.tiles, o.c), 2.0 * el(o.tiles, o.c)}; }
Work op_work(const LossOp& o) { return {8.0 * el(o.rows, o.c), 12.0 * el(o.rows, o.c)}; }
Work op_work(const BnBwdFinOp& o) { return {8.0 * el(o.ctas, o.c), 2.0 * el(o.ctas, o.c)}; }
Work op_work(const BnBwdApplyOp& o) { return {12.0 * static_cast<double>(o.total), 12.0 * static_cast<double>(o.total)}; }
Work op_work(const SgdOp& o) { return {20.0 * static_cast<double>(o.n), 4.0 * static_cast<double>(o.n)}; }
Work op_work(const ScatterOp& o) { return {8.0 * el(o.rows, o.width), 0.0}; }
Work op_work(const GemmOp& o) {
    const double a = o.conv ? el(o.M / (o.oh * o.ow), o.ih, o.iw, o.ic) : el(o.M, o.K);
    return {4.0 * (a + el(o.K, o.N) + el(o.M, o.N)), 2.0 * el(o.M, o.N, o.K)};
}

// Knockout profiling (diagnosis only): PBKD_KNOCKOUT=<name>[,<name>...] drops
// those launch classes (op names as in the profile, or gemm_fwd / gemm_dgrad /
// gemm_wgrad / gemm_conv) from the recorded programs and ignores the failure
// flags, so the epoch time shows each class's critical-path contribution
// (tools/gpu_knockout.sh).  Results are meaningless in this mode.
const std::vector<std::string>& knockouts() {
    static const std::vector<std::string> v = [] {
        std::vector<std::string> out;
        const char* e = std::getenv("PBKD_KNOCKOUT");
        std::string cur;
        for (const char* c = e ? e : "";; ++c) {
            if (*c == ',' || *c == 0) {
                if (!cur.empty()) out.push_back(cur);
                cur.clear();
                if (*c == 0) break;
            } else {
                cur += *c;
            }
        }
        return out;
    }();
    return v;
}
bool knocked_out(const std::string& name) {
    for (const std::string& k : knockouts())
        if (name.rfind(k, 0) == 0) return true;
    return false;
}

// Slot -> tile map of a grouped TMA GEMM launch (see Program::gemm_class);
// empty: keep the round robin (PBKD_GEMM_LPT=0, one tile per CTA, or more
// tiles per CTA than the kernel's tile table holds).
std::vector<int> lpt_slots(const std::vector<GemmOp>& ops, int total, int cls) {
    static const int mode = [] {  // 0 off, 1 every TMA launch, 2 all but split-K (wgrad) launches
        const char* e = std::getenv("PBKD_GEMM_LPT");
        return e ? std::atoi(e) : 0;
    }();
    if (mode == 0 || cls % kGemmClassKind < kGemmClassTma) return {};
    if (mode == 2 && std::all_of(ops.begin(), ops.end(), [](const GemmOp& o) { return o.epi == 2; })) return {};
    const int G = gemm_tma_grid(total);
    if (G >= total) return {};
    struct Tile {
        double cost;
        int id;
    };
    std::vector<Tile> tiles;
    tiles.reserve(static_cast<size_t>(total));
    for (const GemmOp& o : ops) {
        const int n = std::max(1, ctas_gemm(o)), mn = std::max(1, o.tiles_m * o.tiles_n);
        for (int l = 0; l < n; ++l) {
            const int k0 = (l / mn) * o.kchunk, kend = std::min(o.K, k0 + o.kchunk);
            const int nch = std::max(1, (kend - k0 + 31) / 32);
            tiles.push_back({nch + 1.5, o.cta_begin + l});
        }
    }
    std::stable_sort(tiles.begin(), tiles.end(), [](const Tile& a, const Tile& b) { return a.cost > b.cost; });
    using Load = std::pair<double, int>;  // (load, cta): ties to the lower CTA
    std::priority_queue<Load, std::vector<Load>, std::greater<Load>> heap;
    for (int b = 0; b < G; ++b) heap.push({0.0, b});
    std::vector<std::vector<int>> lists(static_cast<size_t>(G));
    for (const Tile& t : tiles) {
        Load l = heap.top();
        heap.pop();
        lists[static_cast<size_t>(l.second)].push_back(t.id);
        l.first += t.cost;
        heap.push(l);
    }
    size_t per = 0;
    for (const auto& v : lists) per = std::max(per, v.size());
    if (per > 64) return {};  // kMaxTiles of the kernels
    std::vector<int> perm(static_cast<size_t>(G) * per, -1);
    for (int b = 0; b < G; ++b)
        for (size_t j = 0; j < lists[static_cast<size_t>(b)].size(); ++j)
            perm[static_cast<size_t>(b) + j * static_cast<size_t>(G)] = lists[static_cast<size_t>(b)][j];
    return perm;
}

// ----------------------------------------------------------------- program
// A recorded sequence of launches.  Grouped ops keep their descriptor arrays
// in one device slab; the whole program can be captured into a CUDA graph.
class Program {
public:
    template <class Op>
    void grouped(void (*launch)(const Op*, int, int, cudaStream_t), std::vector<Op> ops,
                 const std::function<int(const Op&)>& ctas) {
        if (ops.empty() || knocked_out(op_name(typeid(Op).name()))) return;
        int total = 0;
        for (Op& o : ops) {
            o.cta_begin = total;
            total += std::max(1, ctas(o));
        }
        const size_t off = (host_.size() + 63) & ~size_t(63);
        host_.resize(off + ops.size() * sizeof(Op));
        std::memcpy(host_.data() + off, ops.data(), ops.size() * sizeof(Op));
        const int nd = static_cast<int>(ops.size());
        steps_.push_back([launch, off, nd, total](cudaStream_t st, const uint8_t* slab) {
            launch(reinterpret_cast<const Op*>(slab + off), nd, total, st);
        });
        names_.push_back(op_name(typeid(Op).name()));
        KernelStat w;
        for (const Op& o : ops) {
            const auto bf = op_work(o);
            w.bytes += bf.first, w.flops += bf.second;
        }
        work_.push_back(w);
    }
    // tcgen05 GEMMs: one launch per kernel / N-tile class (the tile is a
    // template parameter), all tasks of that class grouped in it; several
    // classes run as a parallel section (independent outputs)
    void gemm(std::vector<GemmOp> all) {
        std::vector<int> classes;
        for (const GemmOp& o : all) classes.push_back(gemm_bn_class(o));
        std::sort(classes.begin(), classes.end());
        classes.erase(std::unique(classes.begin(), classes.end()), classes.end());
        std::vector<Program*> dst(classes.size(), this);
        if (classes.size() > 1) dst = par(static_cast<int>(classes.size()));
        for (size_t ci = 0; ci < classes.size(); ++ci) {
            std::vector<GemmOp> ops;
            for (const GemmOp& o : all)
                if (gemm_bn_class(o) == classes[ci]) ops.push_back(o);
            dst[ci]->gemm_class(classes[ci], std::move(ops));
        }
    }
    void gemm_class(int cls, std::vector<GemmOp> ops) {
        if (ops.empty()) return;
        // Longest-processing-time order: a persistent CTA takes tiles t,
        // t+grid, ... of the launch, so ops whose tiles carry the most K
        // chunks go first and start at t=0 on distinct CTAs instead of
        // landing last behind the short tiles (the launch's critical path).
        // Tile results do not depend on which CTA computes them.
        std::stable_sort(ops.begin(), ops.end(), [](const GemmOp& a, const GemmOp& b) { return a.kchunk > b.kchunk; });
        const char* kind = ops[0].conv ? "conv" : ops[0].epi == 2 ? "wgrad" : ops[0].epi == 1 ? "fwd" : "dgrad";
        const std::string cname = std::string("gemm_") + kind +
                                  (cls % kGemmClassKind >= 3 * kGemmClassTma   ? "_ts"
                                   : cls % kGemmClassKind >= 2 * kGemmClassTma ? "_pre"
                                   : cls % kGemmClassKind >= kGemmClassTma   ? "_tma"
                                                                             : "_reg") +
                                  std::to_string(cls % kGemmClassTma);
        if (knocked_out(cname)) return;
        int total = 0;
        for (GemmOp& o : ops) {
            o.cta_begin = total;
            total += std::max(1, ctas_gemm(o));
        }
        const size_t off = (host_.size() + 63) & ~size_t(63);
        host_.resize(off + ops.size() * sizeof(GemmOp));
        std::memcpy(host_.data() + off, ops.data(), ops.size() * sizeof(GemmOp));
        const int nd = static_cast<int>(ops.size());
        // Optional balanced persistent schedule (PBKD_GEMM_LPT=1/2): tiles in
        // longest-first order, each to the least-loaded CTA (cost = K chunks +
        // an epilogue), as a slot -> tile map.  The round robin leaves the
        // grouped launches' busiest CTA ~40% above the mean and LPT cuts the
        // isolated launch 8%, yet the graph epoch runs 1% slower with it (the
        // staggered CTA exits of the round robin let the next, programmatically
        // launched kernel's CTAs become resident early): off by default.
        // Tile results do not depend on the CTA that computes them.
        const std::vector<int> perm = lpt_slots(ops, total, cls);
        size_t poff = 0;
        int slots = total;
        if (!perm.empty()) {
            poff = (host_.size() + 15) & ~size_t(15);
            host_.resize(poff + perm.size() * sizeof(int));
            std::memcpy(host_.data() + poff, perm.data(), perm.size() * sizeof(int));
            slots = static_cast<int>(perm.size());
        }
        steps_.push_back([off, nd, slots, cls, poff](cudaStream_t st, const uint8_t* slab) {
            launch_gemm_bn(reinterpret_cast<const GemmOp*>(slab + off), nd, slots, cls, st,
                           poff ? reinterpret_cast<const int*>(slab + poff) : nullptr);
        });
        names_.push_back(cname);
        KernelStat w;
        for (const GemmOp& o : ops) {
            const auto bf = op_work(o);
            w.bytes += bf.first, w.flops += bf.second;
        }
        work_.push_back(w);
    }
    void raw(std::function<void(cudaStream_t)> f, const char* name = "raw", double bytes = 0.0) {
        steps_.push_back([f](cudaStream_t st, const uint8_t*) { f(st); });
        names_.push_back(name);
        KernelStat w;
        w.bytes = bytes;
        work_.push_back(w);
    }
    // Parallel section: n independent sub-programs (disjoint outputs).  In a
    // captured graph sub 0 runs on the parent stream and sub i on a side
    // stream (fork / join events), so they execute concurrently; eagerly they
    // run in order.  The caller fills the returned programs.
    std::vector<Program*> par(int n) {
        auto ps = std::make_unique<ParStep>();
        std::vector<Program*> out;
        for (int i = 0; i < n; ++i) {
            ps->subs.push_back(std::make_unique<Program>());
            out.push_back(ps->subs.back().get());
        }
        ParStep* raw_ps = ps.get();
        pars_.push_back(std::move(ps));
        steps_.push_back([this, raw_ps](cudaStream_t st, const uint8_t*) { run_par(*raw_ps, st); });
        names_.push_back("par");
        work_.push_back(KernelStat{});
        par_of_.resize(steps_.size(), nullptr);
        par_of_.back() = raw_ps;
        return out;
    }
    void finalize(cudaStream_t st) {
        slab_.alloc(std::max<size_t>(host_.size(), 64));
        if (!host_.empty())
            PBKD_CUDA(cudaMemcpyAsync(slab_.p, host_.data(), host_.size(), cudaMemcpyHostToDevice, st));
        for (auto& ps : pars_)
            for (auto& sub : ps->subs)
                if (!sub->finalized_) sub->finalize(st);
        PBKD_CUDA(cudaStreamSynchronize(st));
        finalized_ = true;
    }
    void run(cudaStream_t st) {
        if (!finalized_) finalize(st);
        for (auto& s : steps_) s(st, static_cast<const uint8_t*>(slab_.p));
    }
    // Eager run with a CUDA event after every launch; adds each launch's
    // device time and algorithmic work to prof[name] (parallel sections are
    // profiled launch by launch, in order).
    void run_profiled(cudaStream_t st, std::map<std::string, KernelStat>& prof) {
        if (!finalized_) finalize(st);
        std::vector<cudaEvent_t> ev(steps_.size() + 1);
        for (auto& e : ev) PBKD_CUDA(cudaEventCreate(&e));
        PBKD_CUDA(cudaEventRecord(ev[0], st));
        par_of_.resize(steps_.size(), nullptr);
        for (size_t i = 0; i < steps_.size(); ++i) {
            if (par_of_[i]) {
                for (auto& sub : par_of_[i]->subs) sub->run_profiled(st, prof);
            } else {
                steps_[i](st, static_cast<const uint8_t*>(slab_.p));
            }
            PBKD_CUDA(cudaEventRecord(ev[i + 1], st));
        }
        PBKD_CUDA(cudaEventSynchronize(ev.back()));
        for (size_t i = 0; i < steps_.size(); ++i) {
            if (par_of_[i]) continue;
            float ms = 0.0f;
            PBKD_CUDA(cudaEventElapsedTime(&ms, ev[i], ev[i + 1]));
            KernelStat& e = prof[names_[i]];
            e.launches += 1;
            e.ms += ms;
            e.bytes += work_[i].bytes;
            e.flops += work_[i].flops;
        }
        for (auto& e : ev) cudaEventDestroy(e);
    }
    void build_graph(cudaStream_t st, const std::vector<cudaStream_t>* side = nullptr) {
        if (!finalized_) finalize(st);
        cudaGraph_t g;
        set_side(side);
        PBKD_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
        for (auto& s : steps_) s(st, static_cast<const uint8_t*>(slab_.p));
        PBKD_CUDA(cudaStreamEndCapture(st, &g));
        set_side(nullptr);
        for (cudaEvent_t e : cap_events_) cudaEventDestroy(e);
        cap_events_.clear();
        PBKD_CUDA(cudaGraphInstantiate(&exec_, g, 0));
        PBKD_CUDA(cudaGraphDestroy(g));
    }
    void launch_graph(cudaStream_t st) { PBKD_CUDA(cudaGraphLaunch(exec_, st)); }
    // Eager run with the parallel sections on the side streams (fork / join
    // events, as in a captured graph): for programs that run only once, where
    // capturing and instantiating a graph would cost more than it saves.
    void run_concurrent(cudaStream_t st, const std::vector<cudaStream_t>* side) {
        if (!finalized_) finalize(st);
        set_side(side);
        for (auto& s : steps_) s(st, static_cast<const uint8_t*>(slab_.p));
        set_side(nullptr);
        // fork / join events of every nesting level (run_on also copies nested
        // handles one level up: destroy each handle once); recorded events may
        // be destroyed before they complete (released then)
        std::set<cudaEvent_t> evs;
        collect_events(evs);
        for (cudaEvent_t e : evs) cudaEventDestroy(e);
    }
    void collect_events(std::set<cudaEvent_t>& evs) {
        evs.insert(cap_events_.begin(), cap_events_.end());
        cap_events_.clear();
        for (auto& ps : pars_)
            for (auto& sub : ps->subs) sub->collect_events(evs);
    }
    bool has_graph() const { return exec_ != nullptr; }
    size_t launches() const {
        size_t n = 0;
        for (size_t i = 0; i < steps_.size(); ++i) {
            const ParStep* ps = i < par_of_.size() ? par_of_[i] : nullptr;
            if (!ps) ++n;
            else
                for (auto& sub : ps->subs) n += sub->launches();
        }
        return n;
    }
    ~Program() {
        if (exec_) cudaGraphExecDestroy(exec_);
    }

private:
    struct ParStep {
        std::vector<std::unique_ptr<Program>> subs;
    };
    // side streams while capturing (null: eager, sub-programs in order)
    void set_side(const std::vector<cudaStream_t>* side) {
        side_ = side;
        for (auto& ps : pars_)
            for (auto& sub : ps->subs) sub->set_side(side);
    }
    void run_par(ParStep& ps, cudaStream_t st) {
        if (!side_ || side_->empty() || ps.subs.size() < 2) {
            for (auto& sub : ps.subs) sub->run(st);
            return;
        }
        std::vector<cudaEvent_t> joins;
        for (size_t i = 1; i < ps.subs.size(); ++i) {
            cudaStream_t bs = (*side_)[(i - 1) % side_->size()];
            cudaEvent_t fork, join;
            PBKD_CUDA(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
            PBKD_CUDA(cudaEventCreateWithFlags(&join, cudaEventDisableTiming));
            cap_events_.push_back(fork), cap_events_.push_back(join);
            PBKD_CUDA(cudaEventRecord(fork, st));
            PBKD_CUDA(cudaStreamWaitEvent(bs, fork, 0));
            ps.subs[i]->run_on(bs);
            PBKD_CUDA(cudaEventRecord(join, bs));
            joins.push_back(join);
        }
        ps.subs[0]->run_on(st);
        for (cudaEvent_t j : joins) PBKD_CUDA(cudaStreamWaitEvent(st, j, 0));
    }
    void run_on(cudaStream_t st) {  // finalized already (capture time)
        for (auto& s : steps_) s(st, static_cast<const uint8_t*>(slab_.p));
        for (auto& ps : pars_)
            for (auto& sub : ps->subs)
                for (cudaEvent_t e : sub->cap_events_) cap_events_.push_back(e);
    }
    static std::string op_name(const char* mangled) {  // "N8pbkd_gpu7DwFwdOpE" -> "DwFwdOp"
        std::string m(mangled), out;
        size_t i = m.find("pbkd_gpu");
        i = i == std::string::npos ? 0 : i + 8;
        while (i < m.size() && std::isdigit(static_cast<unsigned char>(m[i]))) ++i;
        while (i < m.size() && m[i] != 'E') out += m[i++];
        return out.empty() ? m : out;
    }
    std::vector<uint8_t> host_;
    DevBuf slab_;
    std::vector<std::function<void(cudaStream_t, const uint8_t*)>> steps_;
    std::vector<std::string> names_;
    std::vector<KernelStat> work_;
    std::vector<std::unique_ptr<ParStep>> pars_;
    std::vector<ParStep*> par_of_;  // step index -> parallel section (or null)
    const std::vector<cudaStream_t>* side_ = nullptr;
    std::vector<cudaEvent_t> cap_events_;
    bool finalized_ = false;
    cudaGraphExec_t exec_ = nullptr;
};

void print_profile(const char* what, const std::map<std::string, KernelStat>& prof) {
    double tot = 0.0;
    for (auto& kv : prof) tot += kv.second.ms;
    std::vector<std::pair<double, std::string>> v;
    for (auto& kv : prof) v.push_back({kv.second.ms, kv.first});
    std::sort(v.rbegin(), v.rend());
    std::fprintf(stderr, "[pbkd-prof] %s: %.3f ms total (eager, events per launch)\n", what, tot);
    for (auto& [ms, name] : v) {
        const KernelStat& k = prof.at(name);
        std::fprintf(stderr, "[pbkd-prof]   %-22s %5d launches %9.3f ms %5.1f%%  avg %8.1f us  %7.0f GB/s %7.1f TF/s\n",
                     name.c_str(), k.launches, ms, 100.0 * ms / tot, 1e3 * ms / k.launches, k.bytes / ms / 1e6,
                     k.flops / ms / 1e9);
    }
}

// ------------------------------------------------------------- teacher dev
struct ConvDev {
    int cin = 0, cout = 0, k = 0, stride = 1, pad = 0;
    int kp = 0;          // weight row pitch: k*k*cin rounded up to 4 floats (16-byte TMA rows)
    DevBuf w;            // [cout][k*k][cin]
    DevBuf w_hi, w_lo;   // the same, pre-split into tf32 hi / lo (3xTF32 operands)
    DevBuf scale, shift; // inference batch-norm affine (ops.hpp:304-321)
};

struct TBlockDev {
    int kind = 0;  // 0 conv (3x3 or 1x1), 1 residual, 2 bottleneck, 3 stem (7x7 conv + max pool)
    int cin = 0, hin = 0, win = 0, cout = 0, hout = 0, wout = 0;
    int stride = 1;  // the block's stride (the student candidate's)
    ConvDev c1, c2, c3;
    bool has_proj = false;
    ConvDev proj;  // 1x1 stride projection, no affine
    int mid_h = 0, mid_w = 0;
    long long scratch = 0;  // largest intermediate tensor per sample (floats)
};

// dev_w: the layer's weights already on the device ([cout][cin][kk], the
// reference layout), e.g. inside the teacher's flat weight upload
ConvDev conv_upload(const pbkd::LayerParams& conv, const pbkd::LayerParams* bn, const float* dev_w, cudaStream_t st) {
    ConvDev d;
    d.cin = conv.in_channels;
    d.cout = conv.out_channels;
    d.k = conv.kernel;
    d.stride = conv.stride;
    d.pad = conv.padding;
    const int kk = d.k * d.k;
    d.kp = (kk * d.cin + 3) / 4 * 4;
    const size_t nw = static_cast<size_t>(d.cout) * d.kp;
    {  // relayout [cout][cin][kk] -> [cout][kk][cin] (rows of pitch kp) and tf32 split on the device
        d.w.alloc(nw * sizeof(float));
        d.w_hi.alloc(nw * sizeof(float));
        d.w_lo.alloc(nw * sizeof(float));
        if (d.kp != kk * d.cin)
            for (DevBuf* b : {&d.w, &d.w_hi, &d.w_lo}) PBKD_CUDA(cudaMemsetAsync(b->p, 0, nw * sizeof(float), st));
        launch_conv_weight_prep(dev_w, d.cout, d.cin, kk, d.kp, d.w.f(), d.w_hi.f(), d.w_lo.f(), st);
    }
    if (bn) {
        std::vector<float> sc(d.cout), sh(d.cout);
        for (int j = 0; j < d.cout; ++j) {  // ops.hpp:312-314, float arithmetic
            volatile float s = bn->moving_var.data[j] + static_cast<float>(1e-5);
            const float inv = 1.0f / std::sqrt(static_cast<float>(s));
            volatile float scale = bn->gamma.data[j] * inv;
            volatile float prod = bn->moving_mean.data[j] * scale;
            sc[j] = scale;
            sh[j] = bn->beta.data[j] - prod;
        }
        d.scale = upload(sc, st);
        d.shift = upload(sh, st);
    }
    return d;
}

// tf32 planes of an activation buffer (null: none)
struct Planes2 {
    float* hi = nullptr;
    float* lo = nullptr;
};

GemmOp conv_gemm(const ConvDev& c, const float* x, int n, int ih, int iw, float* y, bool affine,
                 const float* skip, bool relu_out, Planes2 xp = {}, Planes2 yp = {}) {
    GemmOp o{};
    if (gemm_ts_enabled()) {
        // A through tensor memory: the conv splits its raw fp32 input itself,
        // so neither input nor output planes are needed (PBKD_GEMM_TS=0: planes)
        o.a_ts_req = 1;
        xp = Planes2{}, yp = Planes2{};
    }
    o.a_hi = xp.hi, o.a_lo = xp.lo;  // input planes: the conv runs on pre-split A
    o.c_hi = yp.hi, o.c_lo = yp.lo;  // output planes for the next conv
    o.conv = 1;
    o.ih = ih;
    o.iw = iw;
    o.ic = c.cin;
    o.ksz = c.k;
    o.cstride = c.stride;
    o.cpad = c.pad;
    o.oh = (ih + 2 * c.pad - c.k) / c.stride + 1;
    o.ow = (iw + 2 * c.pad - c.k) / c.stride + 1;
    o.M = n * o.oh * o.ow;
    o.N = c.cout;
    o.K = c.k * c.k * c.cin;
    o.A = x;
    o.B = c.w.f();
    o.b_hi = c.w_hi.f();
    o.b_lo = c.w_lo.f();
    o.ldb = c.kp;
    o.b_kmajor = 1;
    o.C = y;
    o.ldc = c.cout;
    o.epi = 0;
    o.ksplit = 1;
    if (affine) {
        o.scale = c.scale.f();
        o.shift = c.shift.f();
    }
    o.skip = skip;
    o.relu = relu_out ? 1 : 0;
    gemm_finalize(o);
    return o;
}


// ------------------------------------------------------------- task state
struct UnitDims {
    int cin, hin, win, cout, ho, wo, stride;
};

struct TaskState {
    DistillTask task;
    int units = 2;
    UnitDims u[kMaxUnits];
    int k = 0;  // block index
    // in_row: one sample of the student's input.  The first unit of a block
    // whose input has a channel count that is not a multiple of 4 (the
    // network input, 3 channels) runs on zero-padded channels (u[0].cin, a
    // multiple of 4: 16-byte rows for the TMA GEMMs and depthwise tiles);
    // cin_ref is the real count (parameter layout of the results)
    int in_row = 0, out_row = 0, cin_ref = 0;
    long long total_steps = 0;
    std::vector<int> steps_in_epoch;  // [epochs+1], index 0 unused
    // parameters
    size_t nparams = 0, nstats = 0;
    size_t off_dw[kMaxUnits], off_pw[kMaxUnits], off_g[kMaxUnits], off_b[kMaxUnits];
    DevBuf params, grads, vel, mstats, snapshot;
    // pos: this epoch's order (slot -> train row); eval_in: the eval split's
    // boundary k-1 (once per run)
    DevBuf pos, eval_in;
    // the run's teacher boundaries k-1 / k for all training samples in train
    // order, read through pos
    const float* bx = nullptr;
    const float* bt = nullptr;
    int nsrc = 0;
    // workspace
    DevBuf d[kMaxUnits], p[kMaxUnits], gp, gd, gy;
    // tf32 hi / lo planes of the pointwise GEMM operands (3xTF32 split),
    // written by their producers when the TMA GEMM consumes them pre-split:
    // dw outputs (fwd A, wgrad B), BN-backward outputs (dgrad A, wgrad A),
    // parameters (pw weights: fwd B, dgrad B)
    // planes[u]: unit u's GEMMs (fwd, dgrad, wgrad) all take TMA pre-split
    // operands, so its dw output and BN gradient are written as planes only
    bool planes_d[kMaxUnits] = {false, false, false}, planes_w = false;
    DevBuf d_hi[kMaxUnits], d_lo[kMaxUnits], gp_hi, gp_lo, params_hi, params_lo;
    DevBuf cs0, cs1, psg, psgx, pgk, ploss, wsplit;
    DevBuf mean, inv, sg, sgx;  // [units][cout]
    DevBuf scale, shift;        // inference affine [units][cout]
    // bookkeeping
    DevBuf step_loss, epoch_loss, failed, best, take, eval_acc, baseline;
    // host copy of the initial parameters / moving stats (init_task_host)
    std::vector<float> host_params, host_stats;
    bool host_ready = false;
    int n_evals_planned = 0;
    std::vector<int> eval_epochs;
    float* w_dw(int u) const { return params.f() + off_dw[u]; }
    float* w_pw(int u) const { return params.f() + off_pw[u]; }
    float* w_g(int u) const { return params.f() + off_g[u]; }
    float* w_b(int u) const { return params.f() + off_b[u]; }
    float* g_dw(int u) const { return grads.f() + off_dw[u]; }
    float* g_pw(int u) const { return grads.f() + off_pw[u]; }
    float* g_g(int u) const { return grads.f() + off_g[u]; }
    float* g_b(int u) const { return grads.f() + off_b[u]; }
    float* mm(int uu) const { return mstats.f() + static_cast<size_t>(uu) * 2 * u[0].cout; }
    float* mv(int uu) const { return mstats.f() + (static_cast<size_t>(uu) * 2 + 1) * u[0].cout; }
    float* mean_u(int uu) const { return mean.f() + static_cast<size_t>(uu) * u[0].cout; }
    float* inv_u(int uu) const { return inv.f() + static_cast<size_t>(uu) * u[0].cout; }
    float* sg_u(int uu) const { return sg.f() + static_cast<size_t>(uu) * u[0].cout; }
    float* sgx_u(int uu) const { return sgx.f() + static_cast<size_t>(uu) * u[0].cout; }
    float* scale_u(int uu) const { return scale.f() + static_cast<size_t>(uu) * u[0].cout; }
    float* shift_u(int uu) const { return shift.f() + static_cast<size_t>(uu) * u[0].cout; }
};

// parameter segments start on 16-byte boundaries (float4 loads)
void pad4(std::vector<float>& v) {
    while (v.size() % 4) v.push_back(0.0f);
}

// channel count a student unit runs its input on (see TaskState::cin_ref)
int padded_channels(int c) { return c % 4 == 0 ? c : (c + 3) / 4 * 4; }

int split_rows() {  // rows per wgrad K split (diagnosis knob PBKD_SPLIT_ROWS)
    static const int r = [] {
        const char* e = std::getenv("PBKD_SPLIT_ROWS");
        return e ? std::max(32, std::atoi(e)) : 512;
    }();
    return r;
}
int split_max() {
    static const int r = [] {
        const char* e = std::getenv("PBKD_SPLIT_MAX");
        return e ? std::max(1, std::atoi(e)) : 64;
    }();
    return r;
}
int split_count(long long kdim) { return std::max(1, std::min<int>(split_max(), ceil_div(kdim, split_rows()))); }

}  // namespace

// ================================================================= Impl ====
struct Engine::Impl {
    int dev = 0;
    cudaStream_t st = nullptr;
    bool has_teacher = false;
    Network net;
    std::vector<TBlockDev> tblocks;
    // classifier
    DevBuf cls_kinds, cls_w, cls_b;
    int cls_layers = 0, cls_maxw = 0, cls_in_c = 0, cls_hw = 0;
    // dataset
    DevBuf images, labels, eval_labels;
    int count = 0, dc = 0, dh = 0, dw = 0, classes = 0;
    RunTiming timing;
    std::unique_ptr<NcclComm> comm;
    PhaseTrace trace;
    void* pinned = nullptr;  // readback staging (grows as needed)
    size_t pinned_bytes = 0;
    std::vector<cudaStream_t> side_streams;  // parallel sections of the epoch graphs
    // layer-by-layer executor (generic candidates, Combined objective,
    // fine-tuning, block-level API) and the teacher it runs: the flat teacher
    // weights stay resident; the DevNet is built on first use
    std::unique_ptr<NetExec> nx;
    DevBuf teacher_flat;
    std::unique_ptr<DevNet> tnet;
    std::vector<int> host_labels;

    explicit Impl(int device) : dev(device) {
        PBKD_CUDA(cudaSetDevice(dev));
        g_alloc_stream = st;
        PBKD_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        const char* ps = std::getenv("PBKD_SIDE_STREAMS");
        side_streams.resize(ps ? std::max(0, std::atoi(ps)) : 4);
        for (cudaStream_t& s2 : side_streams) PBKD_CUDA(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
        nx = std::make_unique<NetExec>(st);
        cudaMemPool_t pool;
        PBKD_CUDA(cudaDeviceGetDefaultMemPool(&pool, dev));
        uint64_t keep = ~uint64_t(0);
        PBKD_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
    }
    ~Impl() {
        cudaSetDevice(dev);
        g_alloc_stream = st;
        // device buffers are freed on st, so before the stream goes away
        tblocks.clear();
        tnet.reset();
        for (DevBuf* b : {&cls_kinds, &cls_w, &cls_b, &images, &labels, &eval_labels, &teacher_flat}) b->release();
        if (st) {
            cudaStreamSynchronize(st);
            cudaStreamDestroy(st);
        }
        for (cudaStream_t s2 : side_streams) cudaStreamDestroy(s2);
        if (pinned) cudaFreeHost(pinned);
        g_alloc_stream = nullptr;
    }

    int max_row() const {
        long long m = static_cast<long long>(net.in_c) * net.in_h * net.in_w;
        for (const TBlockDev& b : tblocks) m = std::max<long long>(m, static_cast<long long>(b.cout) * b.hout * b.wout);
        for (const TBlockDev& b : tblocks) m = std::max(m, b.scratch);
        return static_cast<int>(m);
    }

    // flat: the weights in for_each_array order (host; pinned memory makes the
    // single H2D copy asynchronous).  Null: taken from the network's tensors.
    void load_teacher(Network n_in, const float* flat = nullptr, size_t nflat = 0) {
        PBKD_CUDA(cudaSetDevice(dev));
        g_alloc_stream = st;
        net = std::move(n_in);
        Network& n = net;
        std::map<const pbkd::Tensor*, size_t> off;  // tensor -> offset in the flat array
        size_t total = 0;
        pbkd::for_each_array(n, [&](const std::string&, pbkd::Tensor& t) {
            off[&t] = total;
            total += t.data.size();
        });
        std::vector<float> packed;
        if (flat == nullptr) {
            packed.reserve(total);
            pbkd::for_each_array(n, [&](const std::string&, pbkd::Tensor& t) {
                packed.insert(packed.end(), t.data.begin(), t.data.end());
            });
            flat = packed.data();
        } else if (nflat != total) {
            throw std::invalid_argument("teacher weights: flat size does not match the network");
        }
        trace.st = st;
        trace.t = std::chrono::steady_clock::now();
        tnet.reset();
        teacher_flat.alloc(std::max<size_t>(total, 1) * sizeof(float));
        PBKD_CUDA(cudaMemcpyAsync(teacher_flat.p, flat, total * sizeof(float), cudaMemcpyHostToDevice, st));
        trace.mark("teacher: H2D copy");
        const float* dbase = teacher_flat.f();
        auto dev_of = [&](const pbkd::Tensor& t) { return dbase + off.at(&t); };
        tblocks.clear();
        int c = n.in_c, h = n.in_h, w = n.in_w;
        for (const Block& b : n.blocks) {
            TBlockDev d;
            d.cin = c;
            d.hin = h;
            d.win = w;
            d.cout = b.out_channels;
            if (b.spec_kind == "bottleneck") {  // SURVEY 8f-4 (model.cpp build_bottleneck)
                d.kind = 2;
                d.c1 = conv_upload(b.layers[0], &b.layers[1], dev_of(b.layers[0].weight), st);
                d.c2 = conv_upload(b.layers[3], &b.layers[4], dev_of(b.layers[3].weight), st);
                d.c3 = conv_upload(b.layers[6], &b.layers[7], dev_of(b.layers[6].weight), st);
                const pbkd::LayerParams& add = b.layers[8];
                if (!add.weight.data.empty()) {
                    d.has_proj = true;
                    pbkd::LayerParams pl = pbkd::make_conv_layer(LayerKind::Conv1x1, add.in_channels,
                                                                 add.out_channels, 1, add.stride, 0);
                    d.proj = conv_upload(pl, nullptr, dev_of(add.weight), st);
                }
                d.stride = d.c2.stride;
                d.hout = (h + 2 * d.c2.pad - 3) / d.c2.stride + 1;
                d.wout = (w + 2 * d.c2.pad - 3) / d.c2.stride + 1;
                d.mid_h = d.hout, d.mid_w = d.wout;
                d.scratch = static_cast<long long>(d.c1.cout) * h * w;  // the 1x1 reduce at input resolution
            } else if (b.spec_kind == "stem7x7") {
                d.kind = 3;
                d.c1 = conv_upload(b.layers[0], &b.layers[1], dev_of(b.layers[0].weight), st);
                d.stride = d.c1.stride;
                d.mid_h = (h + 2 * d.c1.pad - d.c1.k) / d.c1.stride + 1;
                d.mid_w = (w + 2 * d.c1.pad - d.c1.k) / d.c1.stride + 1;
                d.hout = (d.mid_h + 2 - 3) / 2 + 1;  // max pool 3x3 / 2, pad 1
                d.wout = (d.mid_w + 2 - 3) / 2 + 1;
                d.scratch = static_cast<long long>(d.cout) * d.mid_h * d.mid_w;
            } else if (b.spec_kind == "residual3x3") {
                d.kind = 1;
                d.c1 = conv_upload(b.layers[0], &b.layers[1], dev_of(b.layers[0].weight), st);
                d.c2 = conv_upload(b.layers[3], &b.layers[4], dev_of(b.layers[3].weight), st);
                const pbkd::LayerParams& add = b.layers[5];
                if (!add.weight.data.empty()) {
                    d.has_proj = true;
                    pbkd::LayerParams pl = pbkd::make_conv_layer(LayerKind::Conv1x1, add.in_channels,
                                                                 add.out_channels, 1, add.stride, 0);
                    d.proj = conv_upload(pl, nullptr, dev_of(add.weight), st);
                }
                d.mid_h = (h + 2 * d.c1.pad - 3) / d.c1.stride + 1;
                d.mid_w = (w + 2 * d.c1.pad - 3) / d.c1.stride + 1;
                d.hout = d.mid_h;
                d.wout = d.mid_w;
                d.stride = d.c1.stride;
                d.scratch = static_cast<long long>(d.cout) * d.mid_h * d.mid_w;
            } else {
                d.kind = 0;
                d.c1 = conv_upload(b.layers[0], &b.layers[1], dev_of(b.layers[0].weight), st);
                d.hout = (h + 2 * d.c1.pad - d.c1.k) / d.c1.stride + 1;
                d.wout = (w + 2 * d.c1.pad - d.c1.k) / d.c1.stride + 1;
                d.stride = d.c1.stride;
            }
            c = d.cout;
            h = d.hout;
            w = d.wout;
            tblocks.push_back(std::move(d));
        }
        trace.mark("teacher: blocks (prep)");
        cls_in_c = c;
        cls_hw = h * w;
        std::vector<int> kinds;
        std::vector<float> cw, cb;
        int width = c;
        cls_maxw = c;
        for (const pbkd::LayerParams& l : n.classifier.layers) {
            if (l.kind == LayerKind::GlobalAvgPool) {
                kinds.push_back(0);
                kinds.push_back(width);
            } else if (l.kind == LayerKind::ReLU) {
                kinds.push_back(1);
                kinds.push_back(width);
            } else {
                kinds.push_back(2);
                kinds.push_back(l.out_channels);
                cw.insert(cw.end(), l.weight.data.begin(), l.weight.data.end());
                cb.insert(cb.end(), l.bias.data.begin(), l.bias.data.end());
                width = l.out_channels;
                cls_maxw = std::max(cls_maxw, width);
            }
        }
        cls_layers = static_cast<int>(n.classifier.layers.size());
        cls_kinds = upload(kinds, st);
        cls_w = upload(cw, st);
        cls_b = upload(cb, st);
        PBKD_CUDA(cudaStreamSynchronize(st));
        has_teacher = true;
    }

    // Teacher block j (0-based) forward on n samples: x -> y.  scratch t1/sk.
    // tf32 planes registered for activation buffers (teacher ping / pong /
    // t1 of a run): convs reading such a buffer take pre-split A, convs
    // writing one also emit its planes
    std::map<const float*, Planes2> act_planes;
    Planes2 planes_for(const float* p) const {
        auto it = act_planes.find(p);
        return it == act_planes.end() ? Planes2{} : it->second;
    }

    void teacher_block(Program& P, int j, const float* x, float* y, int n, float* t1, float* sk) {
        const TBlockDev& b = tblocks[static_cast<size_t>(j)];
        const Planes2 xp = planes_for(x), yp = planes_for(y), tp = planes_for(t1), sp = planes_for(sk);
        if (b.kind == 0) {
            P.gemm({conv_gemm(b.c1, x, n, b.hin, b.win, y, true, nullptr, true, xp, yp)});
            return;
        }
        if (b.kind == 2) {  // bottleneck: t1 = reduce(x), sk = 3x3(t1), y = expand(sk) + skip
            P.gemm({conv_gemm(b.c1, x, n, b.hin, b.win, t1, true, nullptr, true, xp, tp)});
            P.gemm({conv_gemm(b.c2, t1, n, b.hin, b.win, sk, true, nullptr, true, tp, sp)});
            const float* skip = x;
            if (b.has_proj) {  // the projection lands in y; the expand conv adds it element-wise in place
                P.gemm({conv_gemm(b.proj, x, n, b.hin, b.win, y, false, nullptr, false, xp)});
                skip = y;
            }
            P.gemm({conv_gemm(b.c3, sk, n, b.hout, b.wout, y, true, skip, true, sp, yp)});
            return;
        }
        if (b.kind == 3) {  // stem: conv7x7 + BN + ReLU into t1, 3x3/2 max pool into y
            P.gemm({conv_gemm(b.c1, x, n, b.hin, b.win, t1, true, nullptr, true, xp)});
            const int c = b.cout, mh = b.mid_h, mw = b.mid_w;
            float* ph = gemm_ts_enabled() ? nullptr : yp.hi;  // planes only for pre-split consumers
            float* pl = gemm_ts_enabled() ? nullptr : yp.lo;
            P.raw([=](cudaStream_t s2) { launch_maxpool3x3(t1, y, ph, pl, n, mh, mw, c, s2); }, "MaxPoolOp");
            return;
        }
        P.gemm({conv_gemm(b.c1, x, n, b.hin, b.win, t1, true, nullptr, true, xp, tp)});
        const float* skip = x;
        if (b.has_proj) {
            P.gemm({conv_gemm(b.proj, x, n, b.hin, b.win, sk, false, nullptr, false, xp)});
            skip = sk;
        }
        P.gemm({conv_gemm(b.c2, t1, n, b.mid_h, b.mid_w, y, true, skip, true, tp, yp)});
    }

    void load_dataset(const float* img, const int* lab, int n, int c, int h, int w, int cls, bool on_dev) {
        PBKD_CUDA(cudaSetDevice(dev));
        g_alloc_stream = st;
        const size_t sz = static_cast<size_t>(n) * c * h * w;
        images.alloc(sz * sizeof(float));
        PBKD_CUDA(cudaMemcpyAsync(images.p, img, sz * sizeof(float),
                                  on_dev ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
        labels.alloc(static_cast<size_t>(n) * sizeof(int));
        PBKD_CUDA(cudaMemcpyAsync(labels.p, lab, static_cast<size_t>(n) * sizeof(int),
                                  cudaMemcpyHostToDevice, st));
        host_labels.assign(lab, lab + n);
        PBKD_CUDA(cudaStreamSynchronize(st));
        count = n;
        dc = c;
        dh = h;
        dw = w;
        classes = cls;
    }

    // ------------------------------------------------------------ tasks --
    void validate(const DistillTask& t) const {  // distill.cpp:86-100
        if (t.epochs < 1) throw SpecError("epochs must be at least 1");
        if (t.eval_every < 1) throw SpecError("eval_every must be at least 1");
        if (t.batch_size < 1) throw SpecError("batch_size must be at least 1");
        if (t.lambda_local < 0) throw SpecError("lambda_local must be non-negative");
        if (t.threshold < 0.0 || t.threshold > 1.0) throw SpecError("threshold must lie in [0,1]");
        if (t.max_steps < 0) throw SpecError("max_steps must be non-negative");
        // SgdState::step -> ops::sgd_step (ops.hpp:545-548) rejects these on the
        // first step; train_block propagates it (run_parallel: failed result)
        if (!(t.lr > 0.0f)) throw std::invalid_argument("sgd_step: lr must be > 0");
        if (t.momentum < 0.0f || t.momentum >= 1.0f)
            throw std::invalid_argument("sgd_step: momentum must be in [0,1)");
        const std::vector<int> ok = pbkd::identify_replaceable(net);
        if (!std::binary_search(ok.begin(), ok.end(), t.block_index))
            throw SpecError("block " + std::to_string(t.block_index) + " of '" + net.name +
                            "' is not replaceable");
        if (t.loss_mode == pbkd::LossMode::Combined && !net.has_classifier())
            throw SpecError("combined loss needs a network with a classifier");
    }

    // Tasks the grouped lockstep path does not take run layer by layer
    // (nettrain.cu): the Combined objective and the skip candidates.
    static bool generic_task(const DistillTask& t) {
        return t.loss_mode == pbkd::LossMode::Combined || t.kind == pbkd::CandidateKind::TwoLayerSkip ||
               t.kind == pbkd::CandidateKind::ThreeLayerSkip;
    }
    DevNet& teacher_net() {
        if (!tnet) tnet = std::make_unique<DevNet>(make_devnet(*nx, net, teacher_flat.f(), true));
        return *tnet;
    }
    DataView data_view() const {
        DataView d;
        d.images = images.f();
        d.labels = host_labels;
        d.count = count, d.c = dc, d.h = dh, d.w = dw, d.classes = classes;
        return d;
    }

    // task, block index, unit geometry (what init_task_host needs)
    void task_dims(TaskState& s, const DistillTask& t) const {
        s.task = t;
        s.k = t.block_index;
        const TBlockDev& tb = tblocks[static_cast<size_t>(s.k) - 1];
        s.units = (t.kind == pbkd::CandidateKind::ThreeLayer) ? 3 : 2;
        const int ho = (tb.hin - 1) / tb.stride + 1, wo = (tb.win - 1) / tb.stride + 1;
        s.cin_ref = tb.cin;
        const int cpad = padded_channels(tb.cin);
        for (int u = 0; u < s.units; ++u)
            s.u[u] = u == 0 ? UnitDims{cpad, tb.hin, tb.win, tb.cout, ho, wo, tb.stride}
                            : UnitDims{tb.cout, ho, wo, tb.cout, ho, wo, 1};
    }

    void init_task(TaskState& s, const DistillTask& t, int ntrain, int neval) {
        task_dims(s, t);
        const TBlockDev& tb = tblocks[static_cast<size_t>(s.k) - 1];
        const int ho = s.u[0].ho, wo = s.u[0].wo;
        if (ho != tb.hout || wo != tb.wout) throw SpecError("candidate output shape differs from teacher block");
        s.in_row = s.u[0].cin * tb.hin * tb.win;
        s.out_row = tb.cout * ho * wo;
        const int B = t.batch_size;
        const int spe = ceil_div(ntrain, B);
        long long total = static_cast<long long>(t.epochs) * spe;
        if (t.max_steps > 0) total = std::min<long long>(total, t.max_steps);
        s.total_steps = total;
        s.steps_in_epoch.assign(static_cast<size_t>(t.epochs) + 1, 0);
        for (int e = 1; e <= t.epochs; ++e)
            s.steps_in_epoch[e] = static_cast<int>(std::max<long long>(0, std::min<long long>(spe, total - static_cast<long long>(e - 1) * spe)));
        s.eval_epochs.clear();
        s.eval_epochs.push_back(0);
        for (int e = 1; e <= t.epochs; ++e)
            if (s.steps_in_epoch[e] > 0 && e % t.eval_every == 0) s.eval_epochs.push_back(e);
        s.n_evals_planned = static_cast<int>(s.eval_epochs.size());

        if (!s.host_ready) init_task_host(s);
        std::vector<float>& host = s.host_params;
        std::vector<float>& stats = s.host_stats;
        s.nparams = host.size();
        s.nstats = stats.size();
        s.params = upload(host, st);
        s.planes_w = false;
        for (int u = 0; u < s.units; ++u) s.planes_w = s.planes_w || gemm_presplit_ok(s.u[u].cin);
        if (s.planes_w) {
            s.params_hi.alloc(host.size() * sizeof(float));
            s.params_lo.alloc(host.size() * sizeof(float));
            launch_tf32_split(s.params.f(), static_cast<long long>(host.size()), s.params_hi.f(), s.params_lo.f(), st);
        }
        s.grads.alloc(s.nparams * sizeof(float));
        PBKD_CUDA(cudaMemsetAsync(s.grads.p, 0, s.nparams * sizeof(float), st));
        s.vel.alloc(s.nparams * sizeof(float));
        PBKD_CUDA(cudaMemsetAsync(s.vel.p, 0, s.nparams * sizeof(float), st));
        s.mstats = upload(stats, st);
        s.snapshot.alloc((s.nparams + s.nstats) * sizeof(float));
        init_task_device(s, B, ho, wo, tb, ntrain, neval, total, spe);
    }

    // Host half of init_task (no CUDA calls; run for all tasks in parallel):
    // the candidate's seeded init (build_candidate, bit-exact) in the device
    // parameter layout.
    static void init_task_host(TaskState& s) {
        const DistillTask& t = s.task;
        pbkd::ReplacementBlock cand = pbkd::build_candidate(t.kind, s.cin_ref, s.u[0].cout, s.u[0].stride,
                                                            pbkd::mix_seed(t.seed, 0));
        std::vector<float>& host = s.host_params;
        std::vector<float>& stats = s.host_stats;
        host.clear();
        stats.clear();
        size_t li = 0;
        for (int u = 0; u < s.units; ++u) {
            const pbkd::LayerParams& dwl = cand.block.layers[li];
            const pbkd::LayerParams& pwl = cand.block.layers[li + 1];
            const pbkd::LayerParams& bnl = cand.block.layers[li + 2];
            li += 4;
            const int ci = s.u[u].cin, cr = u == 0 ? s.cin_ref : ci, co = s.u[u].cout;
            pad4(host);
            s.off_dw[u] = host.size();
            for (int tap = 0; tap < 9; ++tap)
                for (int c = 0; c < ci; ++c) host.push_back(c < cr ? dwl.weight.data[static_cast<size_t>(c) * 9 + tap] : 0.0f);
            pad4(host);
            s.off_pw[u] = host.size();
            for (int o = 0; o < co; ++o)  // [co][ci], padded input channels 0
                for (int c = 0; c < ci; ++c) host.push_back(c < cr ? pwl.weight.data[static_cast<size_t>(o) * cr + c] : 0.0f);
            pad4(host);
            s.off_g[u] = host.size();
            host.insert(host.end(), bnl.gamma.data.begin(), bnl.gamma.data.end());
            pad4(host);
            s.off_b[u] = host.size();
            host.insert(host.end(), bnl.beta.data.begin(), bnl.beta.data.end());
            (void)co;
            stats.insert(stats.end(), bnl.moving_mean.data.begin(), bnl.moving_mean.data.end());
            stats.insert(stats.end(), bnl.moving_var.data.begin(), bnl.moving_var.data.end());
        }
        while (host.size() % 4) host.push_back(0.0f);  // vector-friendly padding (never trained)
        s.host_ready = true;
    }

    void init_task_device(TaskState& s, int B, int ho, int wo, const TBlockDev& tb, int ntrain, int neval,
                          long long total, int spe) {
        // epoch order and workspace
        s.pos.alloc(static_cast<size_t>(ntrain) * sizeof(int));
        s.eval_in.alloc(static_cast<size_t>(std::max(neval, 1)) * s.in_row * sizeof(float));
        if (s.cin_ref != s.u[0].cin)  // padded channels stay 0 (the sink writes the real ones)
            PBKD_CUDA(cudaMemsetAsync(s.eval_in.p, 0, static_cast<size_t>(std::max(neval, 1)) * s.in_row * sizeof(float), st));
        const long long M = static_cast<long long>(B) * ho * wo;
        const int cin = s.u[0].cin, cout = tb.cout, cmax = std::max(cin, cout);
        for (int u = 0; u < s.units; ++u) {
            s.d[u].alloc(static_cast<size_t>(M) * s.u[u].cin * sizeof(float));
            s.planes_d[u] = gemm_presplit_ok(s.u[u].cin) && gemm_presplit_ok(s.u[u].cout) && s.planes_w;
            if (s.planes_d[u] && !(fwd_ts_on() && gemm_bsplit_enabled())) {
                s.d_hi[u].alloc(static_cast<size_t>(M) * s.u[u].cin * sizeof(float));
                s.d_lo[u].alloc(static_cast<size_t>(M) * s.u[u].cin * sizeof(float));
            }
            s.p[u].alloc(static_cast<size_t>(M) * cout * sizeof(float));
        }
        s.gp.alloc(static_cast<size_t>(M) * cout * sizeof(float));
        // BN gradient planes only when the backward GEMMs take A pre-split
        // (PBKD_GEMM_TS=0); by default they split the raw gradient themselves
        if (s.planes_w && gemm_presplit_ok(cout) && !gemm_ts_enabled()) {
            s.gp_hi.alloc(static_cast<size_t>(M) * cout * sizeof(float));
            s.gp_lo.alloc(static_cast<size_t>(M) * cout * sizeof(float));
        }
        s.gd.alloc(static_cast<size_t>(M) * cmax * sizeof(float));
        s.gy.alloc(static_cast<size_t>(M) * cout * sizeof(float));
        const int tiles = ceil_div(M, 128);
        s.cs0.alloc(static_cast<size_t>(tiles) * cout * sizeof(float));
        s.cs1.alloc(static_cast<size_t>(tiles) * cout * sizeof(float));
        int pc = 1;
        for (int u = 0; u < s.units; ++u) {
            pc = std::max(pc, rows_part_ctas(M, s.u[u].cin));
            pc = std::max(pc, dw_tile(B, s.u[u].ho, s.u[u].wo, s.u[u].cin, s.u[u].stride, 2).tiles);
        }
        pc = std::max(pc, rows_part_ctas(M, cout));
        s.psg.alloc(static_cast<size_t>(pc) * cout * sizeof(float));
        s.psgx.alloc(static_cast<size_t>(pc) * cout * sizeof(float));
        s.pgk.alloc(static_cast<size_t>(pc) * 9 * cmax * sizeof(float));
        s.ploss.alloc(static_cast<size_t>(pc) * sizeof(float));
        s.wsplit.alloc(static_cast<size_t>(split_count(M)) * cout * cmax * sizeof(float));
        s.mean.alloc(static_cast<size_t>(s.units) * cout * sizeof(float));
        s.inv.alloc(static_cast<size_t>(s.units) * cout * sizeof(float));
        s.sg.alloc(static_cast<size_t>(s.units) * cout * sizeof(float));
        s.sgx.alloc(static_cast<size_t>(s.units) * cout * sizeof(float));
        s.scale.alloc(static_cast<size_t>(s.units) * cout * sizeof(float));
        s.shift.alloc(static_cast<size_t>(s.units) * cout * sizeof(float));
        s.step_loss.alloc(static_cast<size_t>(std::max<long long>(total, 1)) * sizeof(float));
        PBKD_CUDA(cudaMemsetAsync(s.step_loss.p, 0, static_cast<size_t>(std::max<long long>(total, 1)) * sizeof(float), st));
        s.epoch_loss.alloc(static_cast<size_t>(spe) * sizeof(float));
        s.failed.alloc(sizeof(int));
        PBKD_CUDA(cudaMemsetAsync(s.failed.p, 0, sizeof(int), st));
        s.best.alloc(sizeof(double));
        const double neg1 = -1.0;
        PBKD_CUDA(cudaMemcpyAsync(s.best.p, &neg1, sizeof(double), cudaMemcpyHostToDevice, st));
        s.take.alloc(sizeof(int));
        s.eval_acc.alloc(static_cast<size_t>(s.n_evals_planned) * sizeof(double));
        s.baseline.alloc(static_cast<size_t>(spe) * sizeof(double));
    }

    // ---------------------------------------------------------- step ops --
    void add_step(Program& P, std::vector<TaskState*>& act, int step, long long gstep_unused, int ntrain,
                  const std::vector<long long>& gsteps) {
        (void)gstep_unused;
        if (act.empty()) return;
        const int U = act[0]->units;
        struct Ctx {
            TaskState* s;
            int n;        // samples this step
            long long M;  // rows
            const float* x0;
            const float* t;
            const int* failed;
            long long gstep;
            const int* rows;  // boundary mode: batch slot -> train row
        };
        std::vector<Ctx> cx;
        for (size_t i = 0; i < act.size(); ++i) {
            TaskState* s = act[i];
            const int B = s->task.batch_size;
            const int n = std::min(B, ntrain - step * B);
            if (!s->bx) throw std::logic_error("student step recorded without teacher boundaries");
            Ctx c{s, n, static_cast<long long>(n) * s->u[0].ho * s->u[0].wo, s->bx, s->bt,
                  knockouts().empty() ? s->failed.i() : nullptr, gsteps[i],
                  s->pos.i() + static_cast<size_t>(step) * B};
            cx.push_back(c);
        }
        // ---- forward
        for (int u = 0; u < U; ++u) {
            std::vector<DwFwdOp> dws;
            std::vector<GemmOp> gms;
            std::vector<BnStatOp> bns;
            for (Ctx& c : cx) {
                TaskState& s = *c.s;
                const UnitDims& d = s.u[u];
                DwFwdOp o{};
                o.x = u == 0 ? c.x0 : s.p[u - 1].f();
                o.w = s.w_dw(u);
                o.y = s.d[u].f();
                // The forward GEMM takes the raw dw output through TMEM, and the
                // weight-gradient GEMM splits it as B in shared memory, so the dw
                // forward writes fp32 only.  With planes (PBKD_GEMM_BSPLIT=0) it
                // writes both; PBKD_FWD_TS=0: planes only, pre-split A.
                if (s.d_hi[u].p) o.y_hi = s.d_hi[u].f(), o.y_lo = s.d_lo[u].f(), o.y_both = fwd_ts_on() ? 1 : 0;
                o.n = c.n;
                o.h = d.hin;
                o.wd = d.win;
                o.c = d.cin;
                o.ho = d.ho;
                o.wo = d.wo;
                o.stride = d.stride;
                o.pad = 1;
                o.pro = u == 0 ? 0 : 1;
                if (u == 0 && c.rows) o.rows = c.rows, o.nsrc = s.nsrc;
                if (u > 0) {
                    o.pa = s.mean_u(u - 1);
                    o.pb = s.inv_u(u - 1);
                    o.pc = s.w_g(u - 1);
                    o.pd = s.w_b(u - 1);
                }
                o.failed = c.failed;
                dw_fwd_finalize(o);
                dws.push_back(o);
                GemmOp g{};
                g.M = static_cast<int>(c.M);
                g.N = d.cout;
                g.K = d.cin;
                g.A = s.d[u].f();
                if (s.d_hi[u].p) g.a_hi = s.d_hi[u].f(), g.a_lo = s.d_lo[u].f(), g.a_ts_req = o.y_both;
                else if (s.planes_d[u]) g.a_ts_req = 1;
                if (s.planes_w) g.b_hi = s.params_hi.f() + s.off_pw[u], g.b_lo = s.params_lo.f() + s.off_pw[u];
                g.lda = d.cin;
                g.a_kmajor = 1;
                g.B = s.w_pw(u);
                g.ldb = d.cin;
                g.b_kmajor = 1;
                g.C = s.p[u].f();
                g.ldc = d.cout;
                g.epi = 1;
                g.part0 = s.cs0.f();
                g.part1 = s.cs1.f();
                g.ksplit = 1;
                gemm_finalize(g);
                if (s.d_hi[u].p && !(g.a_presplit || g.a_tmem))
                    throw std::logic_error("pre-split dw output not consumed by the fwd GEMM");
                g.failed = c.failed;
                gms.push_back(g);
                BnStatOp b{};
                b.part_sum = s.cs0.f();
                b.part_sq = s.cs1.f();
                b.tiles = g.tiles_m;
                b.c = d.cout;
                b.m = c.M;
                b.mean = s.mean_u(u);
                b.inv = s.inv_u(u);
                b.mm = s.mm(u);
                b.mv = s.mv(u);
                b.update_moving = 1;
                b.failed = c.failed;
                bns.push_back(b);
            }
            P.grouped<DwFwdOp>(launch_dw_fwd, dws, ctas_dw_fwd);
            P.gemm(gms);
            P.grouped<BnStatOp>(launch_bn_stat, bns, [](const BnStatOp& o) { return ctas_cols(o.c); });
        }
        // ---- loss and last batch-norm backward sums
        {
            std::vector<LossOp> ls;
            std::vector<BnBwdFinOp> fs;
            for (Ctx& c : cx) {
                TaskState& s = *c.s;
                const int u = U - 1;
                const int cout = s.u[u].cout;
                LossOp o{};
                o.p = s.p[u].f();
                o.t = c.t;
                o.mean = s.mean_u(u);
                o.inv = s.inv_u(u);
                o.gamma = s.w_g(u);
                o.beta = s.w_b(u);
                o.part_sg = s.psg.f();
                o.part_sgx = s.psgx.f();
                o.part_loss = s.ploss.f();
                o.rows = static_cast<int>(c.M);
                o.c = cout;
                o.ctas = rows_part_ctas(c.M, cout);
                o.rows_per = rows_part_per(c.M, o.ctas);
                const size_t count = static_cast<size_t>(c.M) * cout;
                o.kmse = (1.0f * 2.0f) / static_cast<float>(count);
                o.failed = c.failed;
                if (c.rows) o.trows = c.rows, o.srow = s.out_row;
                ls.push_back(o);
                BnBwdFinOp f{};
                f.part_sg = s.psg.f();
                f.part_sgx = s.psgx.f();
                f.part_loss = s.ploss.f();
                f.ctas = o.ctas;
                f.c = cout;
                f.sg = s.sg_u(u);
                f.sgx = s.sgx_u(u);
                f.ggamma = s.g_g(u);
                f.gbeta = s.g_b(u);
                f.loss_out = s.epoch_loss.f() + step;
                f.count = static_cast<double>(count);
                f.failed = s.failed.i();
                fs.push_back(f);
            }
            std::vector<LossOp> narrow, wide;  // one CTA thread per 4 channels up to 1024 channels
            for (const LossOp& o : ls) (o.c <= (o.c % 4 == 0 ? 4 : 1) * kThreads ? narrow : wide).push_back(o);
            P.grouped<LossOp>(launch_loss, narrow, [](const LossOp& o) { return o.ctas; });
            P.grouped<LossOp>(launch_loss_wide, wide, [](const LossOp& o) { return o.ctas; });
            P.grouped<BnBwdFinOp>(launch_bn_bwd_fin, fs, [](const BnBwdFinOp& o) { return ctas_cols(o.c); });
        }
        // ---- backward
        for (int u = U - 1; u >= 0; --u) {
            std::vector<BnBwdApplyOp> aps;
            std::vector<GemmOp> dg, wg;
            std::vector<ReduceOp> wr, kr;
            std::vector<DwBwdOp> dbs;
            std::vector<DwGkOp> gks;
            for (Ctx& c : cx) {
                TaskState& s = *c.s;
                const UnitDims& d = s.u[u];
                BnBwdApplyOp a{};
                a.p = s.p[u].f();
                a.t = u == U - 1 ? c.t : nullptr;
                a.gin = u == U - 1 ? nullptr : s.gy.f();
                a.gout = s.gp.f();
                if (s.planes_d[u] && s.gp_hi.p) a.gout_hi = s.gp_hi.f(), a.gout_lo = s.gp_lo.f();
                a.mean = s.mean_u(u);
                a.inv = s.inv_u(u);
                a.gamma = s.w_g(u);
                a.beta = s.w_b(u);
                a.sg = s.sg_u(u);
                a.sgx = s.sgx_u(u);
                a.total = c.M * d.cout;
                a.c = d.cout;
                a.inv_m = 1.0f / static_cast<float>(c.M);
                a.kmse = (1.0f * 2.0f) / static_cast<float>(static_cast<size_t>(c.M) * d.cout);
                a.failed = c.failed;
                if (a.t && c.rows) a.trows = c.rows, a.srow = s.out_row;
                aps.push_back(a);
                // dgrad: gd[m][j] = sum_o gp[m][o] W[o][j]
                GemmOp g{};
                g.M = static_cast<int>(c.M);
                g.N = d.cin;
                g.K = d.cout;
                g.A = s.gp.f();
                if (s.planes_d[u]) {
                    if (s.gp_hi.p) g.a_hi = s.gp_hi.f(), g.a_lo = s.gp_lo.f();
                    else g.a_ts_req = 1;  // raw gradient split into TMEM by the GEMM
                }
                if (s.planes_w) g.b_hi = s.params_hi.f() + s.off_pw[u], g.b_lo = s.params_lo.f() + s.off_pw[u];
                g.lda = d.cout;
                g.a_kmajor = 1;
                g.B = s.w_pw(u);
                g.ldb = d.cin;
                g.b_kmajor = 0;
                g.C = s.gd.f();
                g.ldc = d.cin;
                g.epi = 0;
                g.ksplit = 1;
                gemm_finalize(g);
                if (s.planes_d[u] && !(g.a_presplit || g.a_tmem))
                    throw std::logic_error("BN gradient operand not consumed by dgrad");
                g.failed = c.failed;
                dg.push_back(g);
                // wgrad: gW[o][j] = sum_m gp[m][o] d[m][j]  (split-K over rows)
                GemmOp w{};
                w.M = d.cout;
                w.N = d.cin;
                w.K = static_cast<int>(c.M);
                w.A = s.gp.f();
                if (s.planes_d[u]) {
                    if (s.gp_hi.p) w.a_hi = s.gp_hi.f(), w.a_lo = s.gp_lo.f();
                    else w.a_ts_req = 1;
                }
                w.lda = d.cout;
                w.a_kmajor = 0;
                w.B = s.d[u].f();
                if (s.d_hi[u].p) w.b_hi = s.d_hi[u].f(), w.b_lo = s.d_lo[u].f();
                else if (s.planes_d[u]) w.b_split_req = 1;  // raw dw output split by the GEMM
                w.ldb = d.cin;
                w.b_kmajor = 0;
                w.ldc = d.cin;
                w.epi = 2;
                w.ksplit = split_count(c.M);
                // no split: the GEMM writes the gradient itself (C must be final
                // before gemm_finalize, which builds the TMA store map from it)
                w.C = w.ksplit == 1 ? s.g_pw(u) : s.wsplit.f();
                gemm_finalize(w);
                if (s.planes_d[u] && !((w.a_presplit || w.a_tmem) && (w.b_presplit || w.b_split)))
                    throw std::logic_error("pre-split operands not consumed by wgrad");
                w.failed = c.failed;
                if (w.ksplit > 1) {
                    ReduceOp r{};
                    r.part = s.wsplit.f();
                    r.out = s.g_pw(u);
                    r.parts = w.ksplit;
                    r.width = d.cout * d.cin;
                    r.failed = c.failed;
                    wr.push_back(r);
                }
                wg.push_back(w);
                if (u > 0) {
                    DwBwdOp b{};
                    b.gy = s.gd.f();
                    b.xp = s.p[u - 1].f();
                    b.w = s.w_dw(u);
                    b.gyprev = s.gy.f();
                    b.part_gk = s.pgk.f();
                    b.part_sg = s.psg.f();
                    b.part_sgx = s.psgx.f();
                    b.mean = s.mean_u(u - 1);
                    b.inv = s.inv_u(u - 1);
                    b.gamma = s.w_g(u - 1);
                    b.beta = s.w_b(u - 1);
                    b.n = c.n;
                    b.h = d.hin;
                    b.wd = d.win;
                    b.c = d.cin;
                    b.failed = c.failed;
                    dw_bwd_finalize(b);
                    dbs.push_back(b);
                    ReduceOp kk{};
                    kk.part = s.pgk.f();
                    kk.out = s.g_dw(u);
                    kk.parts = b.ctas;
                    kk.width = 9 * d.cin;
                    kk.failed = c.failed;
                    kr.push_back(kk);
                    // previous unit's BN-backward sums (ops.hpp:343-344: ggamma =
                    // sum(g * xhat), gbeta = sum(g)) in the same launch as the
                    // weight-gradient reduction
                    ReduceOp rg{};
                    rg.part = s.psg.f();
                    rg.out = s.sg_u(u - 1);
                    rg.out2 = s.g_b(u - 1);
                    rg.parts = b.ctas;
                    rg.width = d.cin;
                    rg.failed = c.failed;
                    kr.push_back(rg);
                    ReduceOp rx = rg;
                    rx.part = s.psgx.f();
                    rx.out = s.sgx_u(u - 1);
                    rx.out2 = s.g_g(u - 1);
                    kr.push_back(rx);
                } else {
                    DwGkOp b{};
                    b.gy = s.gd.f();
                    b.x = c.x0;
                    b.part_gk = s.pgk.f();
                    b.n = c.n;
                    b.h = d.hin;
                    b.wd = d.win;
                    b.c = d.cin;
                    b.ho = d.ho;
                    b.wo = d.wo;
                    b.stride = d.stride;
                    b.pad = 1;
                    b.failed = c.failed;
                    if (c.rows) b.rows = c.rows, b.nsrc = s.nsrc;
                    dw_gk_finalize(b);
                    gks.push_back(b);
                    ReduceOp kk{};
                    kk.part = s.pgk.f();
                    kk.out = s.g_dw(u);
                    kk.parts = b.ctas;
                    kk.width = 9 * d.cin;
                    kk.failed = c.failed;
                    kr.push_back(kk);
                }
            }
            auto red_ctas = ctas_reduce;
            P.grouped<BnBwdApplyOp>(launch_bn_bwd_apply, aps, [](const BnBwdApplyOp& o) { return ctas_elem(o.total); });
            // two independent branches: input gradient (dgrad -> dw backward
            // -> its reductions) and pointwise weight gradient (wgrad ->
            // split-K reduction); disjoint buffers, concurrent in the graph
            // (PBKD_BWD_MERGE=1: dgrad and wgrad GEMMs as one grouped launch
            // first, then the two reduction branches -- measured 1.4% slower
            // on the VGG-16 epoch: the depthwise backward then waits for the
            // wgrad tiles; off)
            static const bool bwd_merge = [] {
                const char* e = std::getenv("PBKD_BWD_MERGE");
                return e && e[0] == '1';
            }();
            if (bwd_merge) {
                std::vector<GemmOp> both = dg;
                both.insert(both.end(), wg.begin(), wg.end());
                P.gemm(both);
            }
            // PBKD_RED_MERGE=1: the two branches' partial-sum reductions as one
            // launch after the branches join
            static const bool red_merge = [] {
                const char* e = std::getenv("PBKD_RED_MERGE");
                return e && e[0] == '1';
            }();
            std::vector<Program*> br = P.par(2);
            Program& bx = *br[0];
            Program& bw = *br[1];
            if (!bwd_merge) bx.gemm(dg);
            if (u > 0) bx.grouped<DwBwdOp>(launch_dw_bwd, dbs, ctas_dw_bwd);
            else bx.grouped<DwGkOp>(launch_dw_gk, gks, ctas_dw_gk);
            if (!red_merge) bx.grouped<ReduceOp>(launch_reduce, kr, red_ctas);
            if (!bwd_merge) bw.gemm(wg);
            if (!red_merge) {
                bw.grouped<ReduceOp>(launch_reduce, wr, red_ctas);
            } else {
                std::vector<ReduceOp> all = kr;
                all.insert(all.end(), wr.begin(), wr.end());
                P.grouped<ReduceOp>(launch_reduce, all, red_ctas);
            }
        }
        // ---- optimizer
        std::vector<SgdOp> sg;
        for (Ctx& c : cx) {
            TaskState& s = *c.s;
            SgdOp o{};
            o.w = s.params.f();
            if (s.planes_w) o.w_hi = s.params_hi.f(), o.w_lo = s.params_lo.f();
            o.v = s.vel.f();
            o.g = s.grads.f();
            o.n = static_cast<long long>(s.nparams);
            o.lr = s.task.lr;
            o.mom = s.task.momentum;
            o.failed = c.failed;
            sg.push_back(o);
        }
        P.grouped<SgdOp>(launch_sgd, sg, [](const SgdOp& o) { return ctas_sgd(o.n); });
    }

    // Teacher pass over `n` samples (dataset indices at d_idx), scattering
    // boundary activations: for each task, boundary k-1 -> its input stream,
    // boundary k -> its target stream, rows placed at pos[t0 + i].
    struct Sink {
        int boundary;  // 0 = network input
        float* dst;
        const int* pos;
        int width;
        int cs = 0, cd = 0;  // channel padding of the destination rows (ScatterOp)
    };
    // Teacher boundaries: boundary j of training row t lives at bnd[j] + t *
    // bnd_row(j) (bnd[0] = the NHWC images, gathered for every row first).
    // The pass runs teacher blocks 1..kmax over training rows [r0, r1).
    int bnd_row(int j) const {
        if (j == 0) return net.in_c * net.in_h * net.in_w;
        const TBlockDev& b = tblocks[static_cast<size_t>(j) - 1];
        return b.cout * b.hout * b.wout;
    }
    // A teacher lane: the activation buffers one chain of teacher blocks
    // uses (their registered tf32 planes; t1 / sk: residual-block scratch).
    // Block j's output planes alternate between the pong / ping plane pairs.
    struct TLane {
        const float *ping, *pong;
        float *t1, *sk;
    };
    // Several lanes split the rows and run as a parallel section: a conv of
    // one lane fills the last-wave tail of the other lane's conv.
    void add_teacher_pass_bnd(Program& P, int r0, int r1, int kmax, const std::vector<float*>& bnd, int chunk,
                              const std::vector<TLane>& lanes) {
        const int n = r1 - r0;
        if (n <= 0 || kmax < 1) return;
        const int L = std::max(1, std::min(static_cast<int>(lanes.size()), n));
        std::vector<Program*> br = L > 1 ? P.par(L) : std::vector<Program*>{&P};
        for (int l = 0; l < L; ++l) {
            Program& Q = *br[static_cast<size_t>(l)];
            const TLane& ln = lanes[static_cast<size_t>(l)];
            const Planes2 pp = planes_for(ln.ping), qp = planes_for(ln.pong);
            const int b0 = r0 + static_cast<int>(static_cast<long long>(n) * l / L);
            const int b1 = r0 + static_cast<int>(static_cast<long long>(n) * (l + 1) / L);
            for (int t0 = b0; t0 < b1; t0 += chunk) {
                const int nc = std::min(chunk, b1 - t0);
                for (int j = 0; j < kmax; ++j) {
                    float* x = bnd[static_cast<size_t>(j)] + static_cast<size_t>(t0) * bnd_row(j);
                    float* y = bnd[static_cast<size_t>(j) + 1] + static_cast<size_t>(t0) * bnd_row(j + 1);
                    const Planes2 yp = (j % 2 == 0) ? qp : pp;
                    if (yp.hi) act_planes[y] = yp;
                    teacher_block(Q, j, x, y, nc, ln.t1, ln.sk);
                }
            }
        }
    }

    void add_teacher_pass(Program& P, const int* d_idx, int n, const std::vector<Sink>& sinks,
                          int chunk, float* ping, float* pong, float* t1, float* sk) {
        int kmax = 0;
        for (const Sink& s : sinks) kmax = std::max(kmax, s.boundary);
        const int in_c = net.in_c, in_h = net.in_h, in_w = net.in_w;
        const float* img = images.f();
        for (int t0 = 0; t0 < n; t0 += chunk) {
            const int nc = std::min(chunk, n - t0);
            const int* idx = d_idx + t0;
            P.raw([=](cudaStream_t s) { launch_gather_nhwc(img, idx, nc, in_c, in_h, in_w, ping, s); });
            float* cur = ping;
            float* nxt = pong;
            // boundary j's rows are scattered while teacher block j+1 runs
            // (both only read `cur`): a parallel section per boundary
            for (int j = 0; j <= kmax; ++j) {
                std::vector<ScatterOp> sc;
                for (const Sink& s : sinks)
                    if (s.boundary == j) sc.push_back(ScatterOp{cur, s.dst, s.pos + t0, nc, s.width, s.cs, s.cd, 0});
                auto scatter = [](Program& Q, std::vector<ScatterOp> ops) {
                    Q.grouped<ScatterOp>(launch_scatter, std::move(ops), [](const ScatterOp&) { return kScatterCtas; });
                };
                if (j == kmax) {
                    scatter(P, std::move(sc));
                    break;
                }
                if (sc.empty()) {
                    teacher_block(P, j, cur, nxt, nc, t1, sk);
                } else {
                    std::vector<Program*> br = P.par(2);
                    teacher_block(*br[0], j, cur, nxt, nc, t1, sk);
                    scatter(*br[1], std::move(sc));
                }
                std::swap(cur, nxt);
            }
        }
    }

    // Student inference over `rows_n` samples of x (task s), output into out.
    void add_student_infer(Program& P, TaskState& s, const float* x, int nsamp, float* bufa,
                           float* bufb, float* out) {
        const int U = s.units;
        for (int u = 0; u < U; ++u) {
            const UnitDims& d = s.u[u];
            const long long M = static_cast<long long>(nsamp) * d.ho * d.wo;
            float* scale = s.scale_u(u);
            float* shift = s.shift_u(u);
            float* g = s.w_g(u);
            float* b = s.w_b(u);
            float* mmv = s.mm(u);
            float* mvv = s.mv(u);
            const int cout = d.cout;
            P.raw([=](cudaStream_t st2) { launch_bn_infer_prep(g, b, mmv, mvv, cout, scale, shift, st2); });
            DwFwdOp o{};
            o.x = u == 0 ? x : bufb;
            o.w = s.w_dw(u);
            o.y = bufa;
            o.n = nsamp;
            o.h = d.hin;
            o.wd = d.win;
            o.c = d.cin;
            o.ho = d.ho;
            o.wo = d.wo;
            o.stride = d.stride;
            o.pad = 1;
            o.pro = u == 0 ? 0 : 2;
            if (u > 0) {
                o.pa = s.scale_u(u - 1);
                o.pb = s.shift_u(u - 1);
            }
            dw_fwd_finalize(o);
            P.grouped<DwFwdOp>(launch_dw_fwd, {o}, ctas_dw_fwd);
            GemmOp gm{};
            gm.M = static_cast<int>(M);
            gm.N = cout;
            gm.K = d.cin;
            gm.A = bufa;
            gm.lda = d.cin;
            gm.a_kmajor = 1;
            gm.B = s.w_pw(u);
            gm.ldb = d.cin;
            gm.b_kmajor = 1;
            gm.C = bufb;
            gm.ldc = cout;
            gm.ksplit = 1;
            gm.a_ts_req = 1;  // raw dw output split into TMEM by the GEMM
            if (s.planes_w && s.params_hi.p) gm.b_hi = s.params_hi.f() + s.off_pw[u], gm.b_lo = s.params_lo.f() + s.off_pw[u];
            gemm_finalize(gm);
            P.gemm({gm});
            if (u == U - 1) {
                const long long tot = M * cout;
                P.raw([=](cudaStream_t st2) { launch_bn_infer_relu(bufb, out, tot, cout, scale, shift, st2); });
            }
        }
    }

    std::vector<TaskOutcome> run(const std::vector<DistillTask>& tasks, const std::vector<int>& train_idx,
                                 const std::vector<int>& eval_idx, const RunOptions& opt);
    std::vector<TaskOutcome> run_grouped(const std::vector<DistillTask>& tasks, const std::vector<int>& train_idx,
                                         const std::vector<int>& eval_idx, const RunOptions& opt);

    // Teacher boundaries of one run (see run()): buffers, the exchange plan
    // and whether the one-time teacher pass has been issued.
    struct Boundaries {
        std::vector<DevBuf> bufs;
        std::vector<float*> bnd;  // bnd[j], j = 0..kmax, [ntrain][bnd_row(j)]
        // student inputs on zero-padded channels (TaskState::cin_ref): a copy
        // of boundary j with cd channels per pixel, made once the rows are in
        struct Pad {
            int j, cs, cd;
            DevBuf buf;
        };
        std::vector<Pad> pads;
        const int* iota = nullptr;  // 0..ntrain-1
        BoundaryPlan plan;
        int kmax = 0, me = 0, world = 1, chunk = 1;
        bool done = false;
        cudaEvent_t t0 = nullptr, t1 = nullptr;  // around the teacher pass + exchange
        ~Boundaries() {
            if (t0) cudaEventDestroy(t0);
            if (t1) cudaEventDestroy(t1);
        }
    };
    // Working buffers of the boundary pass: one TLane per teacher lane with
    // its registered tf32 planes (unregistered on destruction).
    struct TeacherWs {
        Impl& m;
        std::vector<std::array<DevBuf, 12>> bufs;
        std::vector<TLane> lanes;
        TeacherWs(Impl& im, size_t bytes, int nlanes) : m(im), bufs(static_cast<size_t>(nlanes)) {
            const bool tplanes = gemm_presplit_ok(32) && !gemm_ts_enabled();  // convs split raw inputs themselves otherwise
            for (auto& lb : bufs) {
                for (size_t i = 0; i < lb.size(); ++i)  // ping, pong, t1, sk (+ planes of each)
                    if (i < 4 || tplanes) lb[i].alloc(bytes);
                if (tplanes)
                    for (int i = 0; i < 4; ++i) m.act_planes[lb[static_cast<size_t>(i)].f()] = Planes2{lb[4 + 2 * i].f(), lb[5 + 2 * i].f()};
                lanes.push_back(TLane{lb[0].f(), lb[1].f(), lb[2].f(), lb[3].f()});
            }
        }
        ~TeacherWs() {
            for (auto& lb : bufs)
                for (int i = 0; i < 4; ++i) m.act_planes.erase(lb[static_cast<size_t>(i)].f());
        }
    };
    // The boundary pass of this rank (images of every training row into
    // boundary 0, teacher blocks 1..kmax over its shard -- every virtual
    // shard on one GPU) recorded into P.
    void record_boundary_pass(Program& P, Boundaries& b, const DevBuf& d_train, int ntrain, const TeacherWs& ws) {
        const float* img = images.f();
        const int* idx = d_train.i();
        float* x0 = b.bnd[0];
        const int in_c = net.in_c, in_h = net.in_h, in_w = net.in_w;
        P.raw([=](cudaStream_t s2) { launch_gather_nhwc(img, idx, ntrain, in_c, in_h, in_w, x0, s2); }, "GatherOp",
              8.0 * ntrain * in_c * in_h * in_w);
        const std::vector<int>& sb = b.plan.shard_begin;
        std::vector<const float*> added;
        for (int sh = 0; sh < b.plan.world; ++sh) {
            if (b.world > 1 && sh != b.me) continue;
            add_teacher_pass_bnd(P, sb[static_cast<size_t>(sh)], sb[static_cast<size_t>(sh) + 1], b.kmax, b.bnd,
                                 b.chunk, ws.lanes);
        }
        // the boundary rows' plane registrations were only needed while recording
        for (size_t j = 1; j < b.bnd.size(); ++j)
            for (auto it = act_planes.begin(); it != act_planes.end();) {
                const float* q = it->first;
                const bool in_j = q >= b.bnd[j] && q < b.bnd[j] + static_cast<size_t>(ntrain) * bnd_row(static_cast<int>(j));
                it = in_j ? act_planes.erase(it) : std::next(it);
            }
    }
    // Issues the one-time teacher pass (+ NCCL exchange) unless already done.
    void ensure_boundaries(Boundaries& b, const DevBuf& d_train, int ntrain, bool use_side) {
        if (b.done) return;
        b.done = true;
        PBKD_CUDA(cudaEventRecord(b.t0, st));
        {
            TeacherWs ws(*this, static_cast<size_t>(std::max(1, std::min(b.chunk, ntrain))) * max_row() * sizeof(float),
                         teacher_lanes());
            Program P;
            record_boundary_pass(P, b, d_train, ntrain, ws);
            if (use_side)
                P.run_concurrent(st, &side_streams);
            else
                P.run(st);
        }
        if (b.world > 1) comm->exchange(b.plan, b.bnd, st);  // boundary rows to the blocks that read them
        if (!b.pads.empty()) {
            Program P;
            std::vector<ScatterOp> ops;
            for (auto& p : b.pads)
                ops.push_back(ScatterOp{b.bnd[static_cast<size_t>(p.j)], p.buf.f(), b.iota, ntrain, bnd_row(p.j), p.cs,
                                        p.cd, 0});
            P.grouped<ScatterOp>(launch_scatter, std::move(ops), [](const ScatterOp&) { return kScatterCtas; });
            P.run(st);
        }
        PBKD_CUDA(cudaEventRecord(b.t1, st));
        trace.mark("run: teacher boundaries");
    }
    static int teacher_lanes() {  // PBKD_TEACHER_LANES, default 2
        const char* e = std::getenv("PBKD_TEACHER_LANES");
        return std::max(1, std::min(4, e ? std::atoi(e) : 2));
    }
    void run_group(std::vector<TaskState*>& ts, const std::vector<int>& train_idx,
                   const std::vector<int>& eval_idx, const RunOptions& opt, DevBuf& d_train,
                   DevBuf& d_eval, DevBuf& d_iota, Boundaries& bd, const std::function<void()>& prepare);
};

// =============================================================== run ======
std::vector<TaskOutcome> Engine::Impl::run(const std::vector<DistillTask>& tasks,
                                           const std::vector<int>& train_idx,
                                           const std::vector<int>& eval_idx, const RunOptions& opt) {
    std::vector<DistillTask> grouped;
    std::vector<size_t> where;
    for (size_t i = 0; i < tasks.size(); ++i)
        if (!generic_task(tasks[i])) grouped.push_back(tasks[i]), where.push_back(i);
    if (grouped.size() == tasks.size()) return run_grouped(tasks, train_idx, eval_idx, opt);
    PBKD_CUDA(cudaSetDevice(dev));
    g_alloc_stream = st;
    if (!has_teacher) throw std::logic_error("engine: no teacher loaded");
    if (count == 0) throw std::logic_error("engine: no dataset loaded");
    if (train_idx.empty()) throw SpecError("training split is empty");
    if (eval_idx.empty()) throw SpecError("evaluation split is empty");
    if (dc != net.in_c || dh != net.in_h || dw != net.in_w)
        throw pbkd::ShapeError("dataset image shape does not match the network input");
    for (const DistillTask& t : tasks) validate(t);
    std::vector<TaskOutcome> out(tasks.size());
    if (!grouped.empty()) {
        std::vector<TaskOutcome> g = run_grouped(grouped, train_idx, eval_idx, opt);
        for (size_t i = 0; i < g.size(); ++i) out[where[i]] = std::move(g[i]);
    }
    NetTrainer tr(*nx, data_view());
    for (size_t i = 0; i < tasks.size(); ++i)
        if (generic_task(tasks[i]))
            out[i] = tr.train_block(teacher_net(), net, tasks[i], train_idx, eval_idx, opt.baseline_and_eval);
    return out;
}

std::vector<TaskOutcome> Engine::Impl::run_grouped(const std::vector<DistillTask>& tasks,
                                                   const std::vector<int>& train_idx,
                                                   const std::vector<int>& eval_idx, const RunOptions& opt) {
    PBKD_CUDA(cudaSetDevice(dev));
        g_alloc_stream = st;
    trace.t = std::chrono::steady_clock::now();
    if (!has_teacher) throw std::logic_error("engine: no teacher loaded");
    if (count == 0) throw std::logic_error("engine: no dataset loaded");
    if (train_idx.empty()) throw SpecError("training split is empty");
    if (eval_idx.empty()) throw SpecError("evaluation split is empty");
    for (int i : train_idx)
        if (i < 0 || i >= count) throw std::out_of_range("gather_batch: index out of range");
    for (int i : eval_idx)
        if (i < 0 || i >= count) throw std::out_of_range("gather_batch: index out of range");
    if (dc != net.in_c || dh != net.in_h || dw != net.in_w)
        throw pbkd::ShapeError("dataset image shape does not match the network input");
    for (const DistillTask& t : tasks) validate(t);
    trace.st = st;
    const int ntrain = static_cast<int>(train_idx.size());
    const int neval = static_cast<int>(eval_idx.size());
    std::vector<std::unique_ptr<TaskState>> states;
    for (const DistillTask& t : tasks) {
        states.push_back(std::make_unique<TaskState>());
        task_dims(*states.back(), t);
    }
    // candidate inits (host RNG, bit-exact) for all tasks in parallel, in the
    // background: the first teacher pass runs on the GPU meanwhile
    struct Pool {
        std::vector<std::thread> th;
        ~Pool() {
            for (std::thread& t : th)
                if (t.joinable()) t.join();
        }
    } pool;
    for (auto& sp : states) pool.th.emplace_back([p = sp.get()] { init_task_host(*p); });
    bool prepared = false;
    const std::function<void()> prepare = [&] {
        if (prepared) return;
        for (std::thread& t : pool.th) t.join();
        trace.mark("run: candidate init (host, overlapped)");
        for (size_t i = 0; i < tasks.size(); ++i) init_task(*states[i], tasks[i], ntrain, neval);
        prepared = true;
        trace.mark("run: init tasks");
    };
    DevBuf d_train = upload(train_idx, st), d_eval = upload(eval_idx, st);
    std::vector<int> iota(static_cast<size_t>(std::max(ntrain, neval)));
    std::iota(iota.begin(), iota.end(), 0);
    DevBuf d_iota = upload(iota, st);
    // group by (batch size, units) -- lockstep requires equal step geometry
    std::map<std::pair<int, int>, std::vector<TaskState*>> groups;
    for (auto& s : states) groups[{s->task.batch_size, s->units}].push_back(s.get());
    timing = RunTiming{};

    // Teacher boundaries.  Inference-mode BN makes the teacher
    // per-sample and epoch-invariant (model.cpp:553-557), so every boundary
    // 0..kmax of the whole training split is computed ONCE per run and kept
    // in HBM in train order; the student kernels read their batches through
    // each block's epoch order (slot -> train row), so gather_batch /
    // make_batches (dataset.cpp:166-185, distill.cpp:22-30) become an index
    // array and nothing is scattered.  Multi-GPU: each rank computes the rows
    // of its shard of the training split and one grouped NCCL send/recv round
    // per run delivers the rows its blocks read (BoundaryPlan, comm.cpp).
    Boundaries bd;
    {
        const bool multi = comm && !opt.global_blocks.empty();
        bd.world = multi ? comm->world() : 1;
        bd.me = multi ? comm->rank() : 0;
        std::vector<std::pair<int, int>> gb = opt.global_blocks;
        if (gb.empty())
            for (auto& sp : states) gb.push_back({sp->k, bd.me});
        std::sort(gb.begin(), gb.end());
        std::vector<int> gblocks, gowners;
        for (const auto& [k, o] : gb) {
            if (k < 1 || k > static_cast<int>(tblocks.size()))
                throw SpecError("global block " + std::to_string(k) + " out of range");
            gblocks.push_back(k);
            gowners.push_back(o);
            bd.kmax = std::max(bd.kmax, k);
        }
        for (auto& sp : states)
            if (std::find(gb.begin(), gb.end(), std::make_pair(sp->k, bd.me)) == gb.end())
                throw std::logic_error("sharded run: local task not owned by this rank in global_blocks");
        std::vector<long long> rows;
        for (int j = 0; j <= bd.kmax; ++j) rows.push_back(bnd_row(j));
        const int nshards = bd.world > 1 ? bd.world : std::max(1, opt.virtual_shards);
        bd.plan = make_boundary_plan(gblocks, gowners, rows, nshards, ntrain, opt.shard_share);
        bd.chunk = std::max(1, std::min(ntrain, static_cast<int>((size_t(256) << 20) / (size_t(max_row()) * 4))));
        bd.bufs.resize(static_cast<size_t>(bd.kmax) + 1);
        for (int j = 0; j <= bd.kmax; ++j) {
            bd.bufs[static_cast<size_t>(j)].alloc(static_cast<size_t>(ntrain) * bnd_row(j) * sizeof(float));
            bd.bnd.push_back(bd.bufs[static_cast<size_t>(j)].f());
        }
        PBKD_CUDA(cudaEventCreate(&bd.t0));
        PBKD_CUDA(cudaEventCreate(&bd.t1));
        bd.iota = d_iota.i();
        for (auto& sp : states) {
            sp->bx = bd.bnd[static_cast<size_t>(sp->k) - 1];
            sp->bt = bd.bnd[static_cast<size_t>(sp->k)];
            sp->nsrc = ntrain;
            if (sp->cin_ref != sp->u[0].cin) {
                const int j = sp->k - 1;
                auto it = std::find_if(bd.pads.begin(), bd.pads.end(), [&](const Boundaries::Pad& p) { return p.j == j; });
                if (it == bd.pads.end()) {
                    Boundaries::Pad p{j, sp->cin_ref, sp->u[0].cin, DevBuf{}};
                    const UnitDims& d0 = sp->u[0];  // (in_row is set later, by init_task)
                    const size_t bytes = static_cast<size_t>(ntrain) * d0.cin * d0.hin * d0.win * sizeof(float);
                    p.buf.alloc(bytes);
                    PBKD_CUDA(cudaMemsetAsync(p.buf.p, 0, bytes, st));
                    bd.pads.push_back(std::move(p));
                    it = bd.pads.end() - 1;
                }
                sp->bx = it->buf.f();
            }
        }
    }
    for (auto& kv : groups) run_group(kv.second, train_idx, eval_idx, opt, d_train, d_eval, d_iota, bd, prepare);
    // a rank without local blocks still owes its shard to the others
    ensure_boundaries(bd, d_train, ntrain, true);
    prepare();
    {
        float ms = 0.0f;
        PBKD_CUDA(cudaEventSynchronize(bd.t1));
        PBKD_CUDA(cudaEventElapsedTime(&ms, bd.t0, bd.t1));
        timing.teacher_ms = ms;
    }
    if (opt.profile) {  // the boundary pass once more, per launch (idempotent: same rows)
        TeacherWs ws(*this, static_cast<size_t>(std::max(1, std::min(bd.chunk, ntrain))) * max_row() * sizeof(float), 1);
        Program P;
        record_boundary_pass(P, bd, d_train, ntrain, ws);
        P.run_profiled(st, timing.prof);
    }
    for (auto& sp : states) sp->bx = sp->bt = nullptr;

    trace.mark("run: groups done");
    // ---- read back and assemble train_block results: every task's arrays
    // in one batch of async copies into a persistent pinned buffer, one sync
    struct Rb {
        size_t losses, accs, base, best, fin, snap;
    };
    std::vector<Rb> rb(states.size());
    size_t rb_bytes = 0;
    auto take = [&](size_t n) {
        const size_t o = rb_bytes;
        rb_bytes += (n + 7) & ~size_t(7);
        return o;
    };
    for (size_t i = 0; i < states.size(); ++i) {
        TaskState& s = *states[i];
        const int spe = ceil_div(ntrain, s.task.batch_size);
        rb[i].losses = take(static_cast<size_t>(std::max<long long>(s.total_steps, 1)) * sizeof(float));
        rb[i].accs = take(static_cast<size_t>(s.n_evals_planned) * sizeof(double));
        rb[i].base = take(static_cast<size_t>(spe) * sizeof(double));
        rb[i].best = take(sizeof(double));
        rb[i].fin = take((s.nparams + s.nstats) * sizeof(float));
        rb[i].snap = take((s.nparams + s.nstats) * sizeof(float));
    }
    if (rb_bytes > pinned_bytes) {
        if (pinned) cudaFreeHost(pinned);
        PBKD_CUDA(cudaMallocHost(&pinned, rb_bytes));
        pinned_bytes = rb_bytes;
    }
    uint8_t* hb = static_cast<uint8_t*>(pinned);
    for (size_t i = 0; i < states.size(); ++i) {
        TaskState& s = *states[i];
        const int spe = ceil_div(ntrain, s.task.batch_size);
        auto cp = [&](size_t off, const void* src, size_t n) {
            if (n) PBKD_CUDA(cudaMemcpyAsync(hb + off, src, n, cudaMemcpyDeviceToHost, st));
        };
        cp(rb[i].losses, s.step_loss.p, static_cast<size_t>(std::max<long long>(s.total_steps, 1)) * sizeof(float));
        cp(rb[i].accs, s.eval_acc.p, static_cast<size_t>(s.n_evals_planned) * sizeof(double));
        cp(rb[i].base, s.baseline.p, static_cast<size_t>(spe) * sizeof(double));
        cp(rb[i].best, s.best.p, sizeof(double));
        cp(rb[i].fin, s.params.p, s.nparams * sizeof(float));
        cp(rb[i].fin + s.nparams * sizeof(float), s.mstats.p, s.nstats * sizeof(float));
        cp(rb[i].snap, s.snapshot.p, (s.nparams + s.nstats) * sizeof(float));
    }
    PBKD_CUDA(cudaStreamSynchronize(st));
    // per-task result assembly from the pinned buffer, tasks in parallel
    std::vector<TaskOutcome> out(states.size());
    auto assemble = [&](size_t si) {
        TaskState& s = *states[si];
        TaskOutcome& r = out[si];
        r.block_index = s.k;
        r.kind = pbkd::candidate_kind_name(s.task.kind);
        const int B = s.task.batch_size;
        const int spe = ceil_div(ntrain, B);
        const float* lp = reinterpret_cast<const float*>(hb + rb[si].losses);
        std::vector<float> losses(lp, lp + s.total_steps);
        const double* ap = reinterpret_cast<const double*>(hb + rb[si].accs);
        std::vector<double> accs(ap, ap + s.n_evals_planned);
        const double* bp = reinterpret_cast<const double*>(hb + rb[si].base);
        std::vector<double> base(bp, bp + spe);
        const double best = *reinterpret_cast<const double*>(hb + rb[si].best);
        const float* fp = reinterpret_cast<const float*>(hb + rb[si].fin);
        const float* sp = reinterpret_cast<const float*>(hb + rb[si].snap);
        // engine layout (dw tap-major, 16-byte padded segments) -> the
        // reference's for_each_block_array order, written in place
        auto to_ref_order = [&](const float* flat) {
            size_t n = 0;
            auto real_c = [&](int u) { return u == 0 ? s.cin_ref : s.u[u].cin; };
            for (int u = 0; u < s.units; ++u) n += static_cast<size_t>(real_c(u)) * (9 + s.u[u].cout) + 4 * s.u[u].cout;
            std::vector<float> o(n);
            float* w = o.data();
            for (int u = 0; u < s.units; ++u) {
                const int ci = s.u[u].cin, cr = real_c(u), co = s.u[u].cout;
                for (int c = 0; c < cr; ++c)
                    for (int tap = 0; tap < 9; ++tap) *w++ = flat[s.off_dw[u] + static_cast<size_t>(tap) * ci + c];
                for (int oc = 0; oc < co; ++oc)
                    w = std::copy(flat + s.off_pw[u] + static_cast<size_t>(oc) * ci,
                                  flat + s.off_pw[u] + static_cast<size_t>(oc) * ci + cr, w);
                w = std::copy(flat + s.off_g[u], flat + s.off_g[u] + co, w);
                w = std::copy(flat + s.off_b[u], flat + s.off_b[u] + co, w);
                const size_t st0 = s.nparams + static_cast<size_t>(u) * 2 * co;
                w = std::copy(flat + st0, flat + st0 + 2 * co, w);
            }
            return o;
        };
        r.final_block = to_ref_order(fp);
        r.step_losses = losses;
        if (opt.baseline_and_eval) {
            // distill.cpp:166-192: mean over batches of float batch losses
            double sum = 0.0;
            for (int b = 0; b < spe; ++b) {
                const int n = std::min(B, ntrain - b * B);
                const double cnt = static_cast<double>(static_cast<size_t>(n) * s.out_row);
                sum += static_cast<double>(static_cast<float>(base[b] / cnt));
            }
            r.loss_history.push_back(sum / spe);
            r.final_local_loss = sum / spe;
            r.eval_history.push_back({0, accs[0]});
        }
        long long g = 0;
        size_t ev = 1;
        for (int e = 1; e <= s.task.epochs; ++e) {
            const int n = s.steps_in_epoch[e];
            if (n == 0) break;
            double sum = 0.0;
            for (int b = 0; b < n; ++b) {
                const float l = losses[static_cast<size_t>(g + b)];
                if (!std::isfinite(l)) {  // distill.cpp:236-244
                    std::ostringstream msg;
                    msg << "block " << s.k << " diverged at epoch " << e << " batch " << b << " (loss "
                        << static_cast<double>(l) << ")";
                    r.failed = true;
                    r.failure = msg.str();
                    break;
                }
                sum += static_cast<double>(l);
            }
            if (r.failed) break;
            g += n;
            r.loss_history.push_back(sum / n);
            r.final_local_loss = sum / n;
            if (opt.baseline_and_eval && e % s.task.eval_every == 0 && ev < accs.size())
                r.eval_history.push_back({e, accs[ev++]});
        }
        if (opt.baseline_and_eval) {
            r.best_eval = best;
            r.best_block = to_ref_order(sp);
        }
        r.wall_time_s = timing.epoch_ms_total * 1e-3;
    };
    {
        std::vector<std::exception_ptr> err(states.size());
        auto guarded = [&](size_t si) {
            try {
                assemble(si);
            } catch (...) {
                err[si] = std::current_exception();
            }
        };
        std::vector<std::thread> th;
        for (size_t si = 1; si < states.size(); ++si) th.emplace_back(guarded, si);
        if (!states.empty()) guarded(0);
        for (std::thread& t : th) t.join();
        for (const std::exception_ptr& e : err)
            if (e) std::rethrow_exception(e);
    }
    trace.mark("run: readback");
    return out;
}

// acc_out[*slot] = accuracy, *slot += 1 (the slot advances on the device so
// the evaluation program can be replayed as a graph)
__global__ void eval_decide_kernel(const int* correct, int n_eval, double* best, int* take, double* acc_out,
                                   int* slot, const int* failed) {
    pdl_enter();
    const int k = (*slot)++;
    if (failed && *failed) {
        *take = 0;
        return;
    }
    const double acc = static_cast<double>(*correct) / static_cast<double>(n_eval);
    acc_out[k] = acc;
    if (acc > *best) {  // strict >, distill.cpp:160-163
        *best = acc;
        *take = 1;
    } else {
        *take = 0;
    }
}

__global__ void snapshot_kernel(float* dst, const float* params, size_t np, const float* stats,
                                size_t ns, const int* take) {
    pdl_enter();
    if (!*take) return;
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < np + ns;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        dst[i] = i < np ? params[i] : stats[i - np];
}

void Engine::Impl::run_group(std::vector<TaskState*>& ts, const std::vector<int>& train_idx,
                             const std::vector<int>& eval_idx, const RunOptions& opt, DevBuf& d_train,
                             DevBuf& d_eval, DevBuf& d_iota, Boundaries& bd,
                             const std::function<void()>& prepare) {
    const int ntrain = static_cast<int>(train_idx.size());
    const int neval = static_cast<int>(eval_idx.size());
    const int B = ts[0]->task.batch_size;
    const int spe = ceil_div(ntrain, B);
    const int mrow = max_row();
    const int chunk = std::max(1, std::min(ntrain, static_cast<int>((size_t(256) << 20) / (size_t(mrow) * 4))));
    const int ichunk = std::max(B, (chunk / B) * B);
    const size_t wsz = static_cast<size_t>(std::max(chunk, ichunk)) * mrow * sizeof(float);
    DevBuf ping(wsz), pong(wsz), t1(wsz), sk(wsz), ia(wsz), ib(wsz), io(wsz);
    // tf32 planes of the teacher's working buffers (pre-split conv operands)
    DevBuf plane_bufs[8];
    const bool tplanes = gemm_presplit_ok(32) && !gemm_ts_enabled();  // convs split raw inputs themselves otherwise
    if (tplanes) {
        float* bufs[4] = {ping.f(), pong.f(), t1.f(), sk.f()};
        for (int i = 0; i < 4; ++i) {
            plane_bufs[2 * i].alloc(wsz);
            plane_bufs[2 * i + 1].alloc(wsz);
            act_planes[bufs[i]] = Planes2{plane_bufs[2 * i].f(), plane_bufs[2 * i + 1].f()};
        }
    }
    struct PlaneReg {  // unregister when the buffers go away
        std::map<const float*, Planes2>& m;
        ~PlaneReg() { m.clear(); }
    } plane_reg{act_planes};
    // Evaluations and the epoch-0 baseline run the tasks as parallel sections
    // (one branch per stream: the main stream + the side streams); each branch
    // has its own workspace (student scratch, teacher-suffix buffers and their
    // planes), sized for the eval split (teacher suffix) or an inference chunk.
    const int nbr = std::max(1, std::min(static_cast<int>(ts.size()), 1 + static_cast<int>(side_streams.size())));
    const size_t esz = static_cast<size_t>(std::max(1, std::min(neval, ichunk))) * mrow * sizeof(float);
    struct BranchWs {
        DevBuf ia, ib, io, ping, pong, t1, sk, pl[8];
    };
    std::vector<BranchWs> bws(static_cast<size_t>(nbr));
    for (size_t b = 0; b < bws.size(); ++b) {
        BranchWs& w = bws[b];
        if (b == 0) continue;  // branch 0 uses the group's own buffers
        for (DevBuf* d : {&w.ia, &w.ib, &w.io}) d->alloc(wsz);
        for (DevBuf* d : {&w.ping, &w.pong, &w.t1, &w.sk}) d->alloc(esz);
        if (tplanes) {
            float* bufs[4] = {w.ping.f(), w.pong.f(), w.t1.f(), w.sk.f()};
            for (int i = 0; i < 4; ++i) {
                w.pl[2 * i].alloc(esz);
                w.pl[2 * i + 1].alloc(esz);
                act_planes[bufs[i]] = Planes2{w.pl[2 * i].f(), w.pl[2 * i + 1].f()};
            }
        }
    }
    struct WsPtrs {
        float *ia, *ib, *io, *ping, *pong, *t1, *sk;
    };
    auto branch_ws = [&](int b) {
        if (b == 0) return WsPtrs{ia.f(), ib.f(), io.f(), ping.f(), pong.f(), t1.f(), sk.f()};
        BranchWs& w = bws[static_cast<size_t>(b)];
        return WsPtrs{w.ia.f(), w.ib.f(), w.io.f(), w.ping.f(), w.pong.f(), w.t1.f(), w.sk.f()};
    };

    DevBuf correct(sizeof(int) * ts.size());
    int emax = 0;
    for (TaskState* s : ts) emax = std::max(emax, s->task.epochs);

    // Evaluation programs are identical from one eval to the next (the
    // eval_acc slot advances on the device), so each task set's program is
    // captured into a CUDA graph once and replayed.
    std::map<std::vector<TaskState*>, std::unique_ptr<Program>> eval_progs;
    std::map<std::vector<TaskState*>, int> eval_uses;
    std::vector<std::unique_ptr<Program>> eval_once;
    DevBuf eval_slots(sizeof(int) * ts.size());
    PBKD_CUDA(cudaMemsetAsync(eval_slots.p, 0, sizeof(int) * ts.size(), st));
    auto run_eval = [&](const std::vector<TaskState*>& which) {
        PBKD_CUDA(cudaMemsetAsync(correct.p, 0, sizeof(int) * ts.size(), st));
        auto found = eval_progs.find(which);
        if (found != eval_progs.end()) {
            found->second->launch_graph(st);
            return;
        }
        auto prog = std::make_unique<Program>();
        const int nb = std::min(nbr, static_cast<int>(which.size()));
        std::vector<Program*> br = nb > 1 ? prog->par(nb) : std::vector<Program*>{prog.get()};
        for (size_t i = 0; i < which.size(); ++i) {
            TaskState& s = *which[i];
            const int bi = static_cast<int>(i % static_cast<size_t>(nb));
            Program& P = *br[static_cast<size_t>(bi)];
            const WsPtrs W = branch_ws(bi);
            const size_t ti = static_cast<size_t>(std::find(ts.begin(), ts.end(), which[i]) - ts.begin());
            int* corr = correct.i() + ti;
            const int ech = bi == 0 ? ichunk : std::max(1, std::min(neval, ichunk));
            for (int e0 = 0; e0 < neval; e0 += ech) {
                const int ne = std::min(ech, neval - e0);
                add_student_infer(P, s, s.eval_in.f() + static_cast<size_t>(e0) * s.in_row, ne, W.ia, W.ib, W.io);
                float* cur = W.io;
                for (size_t j = static_cast<size_t>(s.k); j < tblocks.size(); ++j) {
                    float* nxt = cur == W.ping ? W.pong : W.ping;
                    teacher_block(P, static_cast<int>(j), cur, nxt, ne, W.t1, W.sk);
                    cur = nxt;
                }
                const int hw = cls_hw, cc = cls_in_c, nl = cls_layers, mw = cls_maxw;
                const int* kinds = cls_kinds.i();
                const float* w = cls_w.f();
                const float* b = cls_b.f();
                const int* labs = eval_labels.i() + e0;
                const float* xin = cur;
                P.raw([=](cudaStream_t s2) { launch_classifier_count(xin, ne, hw, cc, kinds, nl, w, b, mw, labs, corr, s2); });
            }
            double* accp = s.eval_acc.d();
            int* slotp = eval_slots.i() + ti;
            double* bestp = s.best.d();
            int* takep = s.take.i();
            const int* fl = s.failed.i();
            float* snapp = s.snapshot.f();
            const float* pp = s.params.f();
            const float* sp = s.mstats.f();
            const size_t np = s.nparams, ns = s.nstats;
            P.raw([=](cudaStream_t s2) {
                launch_k(eval_decide_kernel, dim3(1), dim3(1), 0, s2, corr, neval, bestp, takep, accp, slotp, fl);
                launch_k(snapshot_kernel, dim3(64), dim3(256), 0, s2, snapp, pp, np, sp, ns, takep);
            });
        }
        // a graph pays off once the same evaluation repeats a few times
        if (opt.use_graphs && ++eval_uses[which] >= 3) {
            prog->build_graph(st, &side_streams);
            prog->launch_graph(st);
            eval_progs.emplace(which, std::move(prog));
        } else {
            prog->run_concurrent(st, &side_streams);
            eval_once.push_back(std::move(prog));  // its slab lives until the run ends
        }
    };

    // ---- labels of the eval split (for the classifier count)
    {
        std::vector<int> lab(static_cast<size_t>(neval));
        std::vector<int> all(static_cast<size_t>(count));
        PBKD_CUDA(cudaMemcpy(all.data(), labels.p, all.size() * sizeof(int), cudaMemcpyDeviceToHost));
        for (int i = 0; i < neval; ++i) lab[static_cast<size_t>(i)] = all[static_cast<size_t>(eval_idx[static_cast<size_t>(i)])];
        eval_labels = upload(lab, st);
    }
    trace.mark("group: workspace + labels");

    // ---- epoch 0: baseline losses and first evaluation
    if (opt.baseline_and_eval) {
        ensure_boundaries(bd, d_train, ntrain, true);  // needs no task state: launch it first
        prepare();
        {  // eval-split prefix activations (once per run)
            Program P;
            std::vector<Sink> sk_eval;
            for (TaskState* s : ts) {
                const int c0 = s->u[0].cin, cr = s->cin_ref;
                const int wsrc = s->in_row / c0 * cr;  // the boundary's own row width
                sk_eval.push_back({s->k - 1, s->eval_in.f(), d_iota.i(), wsrc, cr != c0 ? cr : 0, cr != c0 ? c0 : 0});
            }
            add_teacher_pass(P, d_eval.i(), neval, sk_eval, chunk, ping.f(), pong.f(), t1.f(), sk.f());
            P.run(st);
        }
        {
            Program P;
            const int nb = std::min(nbr, static_cast<int>(ts.size()));
            std::vector<Program*> br = nb > 1 ? P.par(nb) : std::vector<Program*>{&P};
            for (size_t ti = 0; ti < ts.size(); ++ti) {
                TaskState* s = ts[ti];
                const int bi = static_cast<int>(ti % static_cast<size_t>(nb));
                Program& Q = *br[static_cast<size_t>(bi)];
                const WsPtrs W = branch_ws(bi);
                for (int r0 = 0; r0 < ntrain; r0 += ichunk) {
                    const int nr = std::min(ichunk, ntrain - r0);
                    add_student_infer(Q, *s, s->bx + static_cast<size_t>(r0) * s->in_row, nr, W.ia, W.ib, W.io);
                    const float* tg = s->bt + static_cast<size_t>(r0) * s->out_row;
                    const float* so = W.io;
                    const long long seg = static_cast<long long>(B) * s->out_row;
                    const long long tot = static_cast<long long>(nr) * s->out_row;
                    const int nseg = ceil_div(nr, B);
                    double* outp = s->baseline.d() + r0 / B;
                    Q.raw([=](cudaStream_t s2) { launch_mse_segments(so, tg, seg, tot, nseg, outp, s2); });
                }
            }
            P.run_concurrent(st, &side_streams);
        }
        trace.mark("group: epoch-0 baseline");
        run_eval(ts);
        trace.mark("group: epoch-0 eval");
    }

    // ---- training epochs
    prepare();
    cudaEvent_t e0, e1, t0, t1e;
    PBKD_CUDA(cudaEventCreate(&e0));
    PBKD_CUDA(cudaEventCreate(&e1));
    PBKD_CUDA(cudaEventCreate(&t0));
    PBKD_CUDA(cudaEventCreate(&t1e));
    bool timed_started = false;
    std::vector<long long> gbase(ts.size(), 0);
    auto epoch_key = [&](int e) {
        std::vector<int> key;
        for (TaskState* s : ts) key.push_back(e <= s->task.epochs ? s->steps_in_epoch[e] : 0);
        return key;
    };
    // Epoch programs (the student steps of one epoch), one per distinct key
    // (steps per task), recorded and captured BEFORE the first epoch runs so
    // no host capture time falls between device work.  A graph pays off only
    // for a program that runs more than once.
    std::map<std::vector<int>, std::unique_ptr<Program>> progs;
    std::map<std::vector<int>, int> key_uses;
    int last_epoch = 0;
    for (int e = 1; e <= emax; ++e) {
        const std::vector<int> key = epoch_key(e);
        if (std::all_of(key.begin(), key.end(), [](int v) { return v == 0; })) break;
        key_uses[key] += 1;
        last_epoch = e;
    }
    for (int e = 1; e <= last_epoch; ++e) {
        const std::vector<int> key = epoch_key(e);
        if (progs.count(key)) continue;
        auto prog = std::make_unique<Program>();
        for (int step = 0; step < spe; ++step) {
            std::vector<TaskState*> act;
            std::vector<long long> gs;
            for (size_t i = 0; i < ts.size(); ++i)
                if (step < key[i]) {
                    act.push_back(ts[i]);
                    gs.push_back(gbase[i] + step);
                }
            add_step(*prog, act, step, 0, ntrain, gs);
        }
        static const bool graph_single = [] {  // diagnosis: PBKD_GRAPH_SINGLE=1 captures single-use epochs too
            const char* e = std::getenv("PBKD_GRAPH_SINGLE");
            return e && e[0] == '1';
        }();
        if (opt.use_graphs && (key_uses[key] > 1 || graph_single)) prog->build_graph(st, &side_streams);
        progs.emplace(key, std::move(prog));
    }
    trace.mark("epoch: record programs / graphs");
    // host: epoch orders (bit-exact std::shuffle of the training rows: the
    // permutation std::shuffle applies depends only on the size and the
    // engine, so shuffling row numbers gives the slot -> train-row map even
    // when train_idx repeats a sample).  Computed for epoch e+1 while the GPU
    // runs epoch e.
    std::vector<int> rows_iota(static_cast<size_t>(ntrain));
    std::iota(rows_iota.begin(), rows_iota.end(), 0);
    auto make_ord = [&](int e, const std::vector<int>& key) {
        std::vector<std::vector<int>> out(ts.size());
        for (size_t i = 0; i < ts.size(); ++i)
            if (key[i] > 0) out[i] = pbkd::epoch_order(rows_iota, ts[i]->task.seed, e);
        return out;
    };
    std::vector<std::vector<int>> ord_next = last_epoch >= 1 ? make_ord(1, epoch_key(1)) : std::vector<std::vector<int>>{};
    // the timed window of a step-only run starting at epoch 1 includes the
    // run's one-time teacher pass (amortised over the epochs, not dropped)
    if (last_epoch >= 1 && opt.timed_from_epoch <= 1 && !bd.done) {
        PBKD_CUDA(cudaEventRecord(t0, st));
        timed_started = true;
    }
    ensure_boundaries(bd, d_train, ntrain, true);
    for (int e = 1; e <= last_epoch; ++e) {
        const std::vector<int> key = epoch_key(e);
        const bool timed = e >= opt.timed_from_epoch;
        if (timed && !timed_started) {
            PBKD_CUDA(cudaEventRecord(t0, st));
            timed_started = true;
        }
        std::vector<std::vector<int>> ord_now = std::move(ord_next);
        for (size_t i = 0; i < ts.size(); ++i)
            if (key[i] > 0)
                PBKD_CUDA(cudaMemcpyAsync(ts[i]->pos.p, ord_now[i].data(), ord_now[i].size() * sizeof(int),
                                          cudaMemcpyHostToDevice, st));
        Program& pr = *progs.at(key);
        PBKD_CUDA(cudaEventRecord(e0, st));
        if (pr.has_graph())
            pr.launch_graph(st);
        else
            pr.run_concurrent(st, &side_streams);
        PBKD_CUDA(cudaEventRecord(e1, st));
        trace.mark("epoch: launched (host)");
        for (size_t i = 0; i < ts.size(); ++i)  // epoch-local losses -> per-run history
            if (key[i] > 0)
                PBKD_CUDA(cudaMemcpyAsync(ts[i]->step_loss.f() + gbase[i], ts[i]->epoch_loss.p,
                                          static_cast<size_t>(key[i]) * sizeof(float), cudaMemcpyDeviceToDevice, st));
        if (timed) timing.launches += static_cast<long long>(pr.launches());
        if (e + 1 <= last_epoch) ord_next = make_ord(e + 1, epoch_key(e + 1));  // overlaps the GPU
        PBKD_CUDA(cudaEventSynchronize(e1));
        float ms = 0.0f;
        PBKD_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        timing.epoch_ms_total += ms;
        timing.epoch_ms.push_back(ms);
        timing.epochs += 1;
        if (timed) timing.timed_epochs += 1;
        for (size_t i = 0; i < ts.size(); ++i) {
            gbase[i] += key[i];
            timing.student_steps = std::max<long long>(timing.student_steps, gbase[i]);
        }
        if (opt.baseline_and_eval) {
            std::vector<TaskState*> which;
            for (size_t i = 0; i < ts.size(); ++i)
                if (key[i] > 0 && e % ts[i]->task.eval_every == 0) which.push_back(ts[i]);
            trace.mark("epoch: run");
            if (!which.empty()) run_eval(which);
            trace.mark("epoch: eval");
        }
    }
    if (timed_started) {
        PBKD_CUDA(cudaEventRecord(t1e, st));
        PBKD_CUDA(cudaEventSynchronize(t1e));
        float ms = 0.0f;
        PBKD_CUDA(cudaEventElapsedTime(&ms, t0, t1e));
        timing.timed_ms += ms;
        if (opt.timed_from_epoch <= 1) timing.timed_includes_teacher = true;
    }
    // outside the timed window: the last epoch's program once more, eagerly
    // with an event per launch, on a saved copy of the training state that
    // is restored afterwards (results are those of the real epochs)
    if (opt.profile && last_epoch >= 1) {
        struct Saved {
            DevBuf* dst;
            DevBuf copy;
        };
        std::vector<Saved> saved;
        for (TaskState* s : ts)
            for (DevBuf* b : {&s->params, &s->params_hi, &s->params_lo, &s->vel, &s->mstats, &s->failed, &s->grads}) {
                if (!b->p) continue;
                Saved sv{b, DevBuf(b->bytes)};
                PBKD_CUDA(cudaMemcpyAsync(sv.copy.p, b->p, b->bytes, cudaMemcpyDeviceToDevice, st));
                saved.push_back(std::move(sv));
            }
        progs.at(epoch_key(last_epoch))->run_profiled(st, timing.prof);
        for (Saved& sv : saved)
            PBKD_CUDA(cudaMemcpyAsync(sv.dst->p, sv.copy.p, sv.dst->bytes, cudaMemcpyDeviceToDevice, st));
    }
    cudaEventDestroy(t0);
    cudaEventDestroy(t1e);
    PBKD_CUDA(cudaStreamSynchronize(st));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
}

// ====================================================== kernel bench
__global__ void fill_kernel(float* p, size_t n, float v) {
    pdl_enter();
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x)
        p[i] = v * (1.0f + 0.001f * static_cast<float>(i % 97));
}

void Engine::bench_kernel(int which, int batch, int iters, double* ms, double* bytes, double* flops) {
    Impl& m = *impl_;
    PBKD_CUDA(cudaSetDevice(m.dev));
    g_alloc_stream = m.st;
    if (!m.has_teacher) throw std::logic_error("engine: no teacher loaded");
    // the teacher block with the most MACs
    size_t bi = 0;
    double best = -1;
    for (size_t j = 0; j < m.tblocks.size(); ++j) {
        const TBlockDev& b = m.tblocks[j];
        const double macs = static_cast<double>(b.hout) * b.wout * b.cout * b.cin * b.c1.k * b.c1.k;
        if (macs > best) best = macs, bi = j;
    }
    const TBlockDev& b = m.tblocks[bi];
    const int n = batch, c = b.cout, ho = b.hout, wo = b.wout;
    const long long M = static_cast<long long>(n) * ho * wo;
    const size_t big = static_cast<size_t>(std::max<long long>(M * std::max(c, b.cin) * 9LL, static_cast<long long>(n) * b.cin * b.hin * b.win));
    DevBuf x(big * 4), y(big * 4), z(big * 4), w(static_cast<size_t>(c) * std::max(c, b.cin) * 9 * 4 + 64),
        v(static_cast<size_t>(c) * 64 * 4 + 4096), parts(static_cast<size_t>(4096) * 9 * c * 4 + 4096);
    for (DevBuf* d : {&x, &y, &z, &w, &v})
        launch_k(fill_kernel, dim3(1024), dim3(256), 0, m.st, d->f(), d->bytes / 4, 0.37f);
    PBKD_LAUNCH_CHECK();
    Program P;
    double by = 0, fl = 0;
    if (which == 0) {
        const ConvDev& cv = b.c1;
        GemmOp o = conv_gemm(cv, x.f(), n, b.hin, b.win, y.f(), true, nullptr, true);
        P.gemm({o});
        fl = 2.0 * o.M * o.N * o.K;
        by = 4.0 * (static_cast<double>(n) * b.hin * b.win * b.cin + static_cast<double>(o.N) * o.K + static_cast<double>(o.M) * o.N);
    } else if (which == 1) {
        GemmOp g{};
        g.M = static_cast<int>(M), g.N = c, g.K = c;
        g.A = x.f(), g.lda = c, g.a_kmajor = 1, g.B = w.f(), g.ldb = c, g.b_kmajor = 1;
        g.C = y.f(), g.ldc = c, g.epi = 1, g.part0 = parts.f(), g.part1 = parts.f() + static_cast<size_t>(2048) * c;
        g.ksplit = 1;
        gemm_finalize(g);
        P.gemm({g});
        fl = 2.0 * M * c * c;
        by = 4.0 * (2.0 * M * c + static_cast<double>(c) * c);
    } else if (which == 2) {
        DwFwdOp o{};
        o.x = x.f(), o.w = w.f(), o.y = y.f(), o.n = n, o.h = ho, o.wd = wo, o.c = c, o.ho = ho, o.wo = wo;
        o.stride = 1, o.pad = 1, o.pro = 1, o.pa = v.f(), o.pb = v.f(), o.pc = v.f(), o.pd = v.f();
        dw_fwd_finalize(o);
        P.grouped<DwFwdOp>(launch_dw_fwd, {o}, ctas_dw_fwd);
        fl = 18.0 * M * c;
        by = 4.0 * (2.0 * M * c + 9.0 * c);
    } else if (which == 3) {
        DwBwdOp o{};
        o.gy = x.f(), o.xp = z.f(), o.w = w.f(), o.gyprev = y.f();
        o.mean = v.f(), o.inv = v.f(), o.gamma = v.f(), o.beta = v.f();
        o.n = n, o.h = ho, o.wd = wo, o.c = c;
        dw_bwd_finalize(o);
        o.part_gk = parts.f(), o.part_sg = parts.f(), o.part_sgx = parts.f();
        P.grouped<DwBwdOp>(launch_dw_bwd, {o}, ctas_dw_bwd);
        fl = 36.0 * M * c;
        by = 4.0 * (3.0 * M * c + 9.0 * c);
    } else {
        LossOp o{};
        o.p = x.f(), o.t = z.f(), o.mean = v.f(), o.inv = v.f(), o.gamma = v.f(), o.beta = v.f();
        o.rows = static_cast<int>(M), o.c = c, o.ctas = rows_part_ctas(M, c), o.rows_per = rows_part_per(M, o.ctas);
        o.part_sg = parts.f(), o.part_sgx = parts.f(), o.part_loss = parts.f(), o.kmse = 1e-6f;
        P.grouped<LossOp>(launch_loss, {o}, [](const LossOp& q) { return q.ctas; });
        fl = 8.0 * M * c;
        by = 4.0 * 2.0 * M * c;
    }
    P.finalize(m.st);
    for (int i = 0; i < 3; ++i) P.run(m.st);  // warm-up
    cudaEvent_t a, bev;
    PBKD_CUDA(cudaEventCreate(&a));
    PBKD_CUDA(cudaEventCreate(&bev));
    PBKD_CUDA(cudaStreamSynchronize(m.st));
    PBKD_CUDA(cudaEventRecord(a, m.st));
    for (int i = 0; i < iters; ++i) P.run(m.st);
    PBKD_CUDA(cudaEventRecord(bev, m.st));
    PBKD_CUDA(cudaEventSynchronize(bev));
    float t = 0.0f;
    PBKD_CUDA(cudaEventElapsedTime(&t, a, bev));
    cudaEventDestroy(a);
    cudaEventDestroy(bev);
    *ms = static_cast<double>(t) / iters;
    *bytes = by;
    *flops = fl;
}

// ====================================================== inference helpers
namespace {
Tensor nhwc_to_nchw(const std::vector<float>& v, int n, int c, int h, int w) {
    Tensor t(n, c, h, w);
    for (int i = 0; i < n; ++i)
        for (int y = 0; y < h; ++y)
            for (int x = 0; x < w; ++x)
                for (int ch = 0; ch < c; ++ch)
                    t.data[t.idx(i, ch, y, x)] = v[((static_cast<size_t>(i) * h + y) * w + x) * c + ch];
    return t;
}
std::vector<float> nchw_to_nhwc(const Tensor& t) {
    std::vector<float> v(t.size());
    for (int i = 0; i < t.n; ++i)
        for (int ch = 0; ch < t.c; ++ch)
            for (int y = 0; y < t.h; ++y)
                for (int x = 0; x < t.w; ++x)
                    v[((static_cast<size_t>(i) * t.h + y) * t.w + x) * t.c + ch] = t.data[t.idx(i, ch, y, x)];
    return v;
}
}  // namespace

Engine::Engine(int device) : impl_(std::make_unique<Impl>(device)) {}
Engine::~Engine() = default;
void Engine::set_teacher(const Network& net) { impl_->load_teacher(net); }
void Engine::set_teacher(Network&& net) { impl_->load_teacher(std::move(net)); }
void Engine::set_teacher(Network&& net, const float* flat, size_t n) { impl_->load_teacher(std::move(net), flat, n); }
const Network& Engine::teacher() const { return impl_->net; }
Network Engine::take_teacher() {
    impl_->has_teacher = false;
    impl_->tnet.reset();
    return std::move(impl_->net);
}
bool Engine::has_teacher() const { return impl_->has_teacher; }
void Engine::set_dataset(const float* img, const int* lab, int n, int c, int h, int w, int cls, bool on_dev) {
    impl_->load_dataset(img, lab, n, c, h, w, cls, on_dev);
}
std::vector<TaskOutcome> Engine::run(const std::vector<DistillTask>& t, const std::vector<int>& tr,
                                     const std::vector<int>& ev, const RunOptions& o) {
    return impl_->run(t, tr, ev, o);
}
const RunTiming& Engine::timing() const { return impl_->timing; }
NetExec& Engine::exec() {
    PBKD_CUDA(cudaSetDevice(impl_->dev));
    g_alloc_stream = impl_->st;
    return *impl_->nx;
}
NetTrainer Engine::trainer() {
    exec();
    if (impl_->count == 0) throw std::logic_error("engine: no dataset loaded");
    return NetTrainer(*impl_->nx, impl_->data_view());
}
DevNet& Engine::teacher_net() {
    exec();
    if (!impl_->has_teacher) throw std::logic_error("engine: no teacher loaded");
    return impl_->teacher_net();
}
void Engine::validate(const DistillTask& t) const {
    if (!impl_->has_teacher) throw std::logic_error("engine: no teacher loaded");
    impl_->validate(t);
}
void Engine::check_split(const std::vector<int>& tr, const std::vector<int>& ev) const {
    if (tr.empty()) throw SpecError("training split is empty");
    if (ev.empty()) throw SpecError("evaluation split is empty");
    for (const std::vector<int>* v : {&tr, &ev})
        for (int i : *v)
            if (i < 0 || i >= impl_->count) throw std::out_of_range("gather_batch: index out of range");
}
int Engine::device() const { return impl_->dev; }
void Engine::set_comm(const char* id, int rank, int world) {
    PBKD_CUDA(cudaSetDevice(impl_->dev));
    g_alloc_stream = impl_->st;
    impl_->comm.reset();
    if (world > 1) impl_->comm = std::make_unique<NcclComm>(id, rank, world);
}
void Engine::set_comm(std::unique_ptr<NcclComm> c) {
    PBKD_CUDA(cudaSetDevice(impl_->dev));
    g_alloc_stream = impl_->st;
    impl_->comm = std::move(c);
}
int Engine::comm_rank() const { return impl_->comm ? impl_->comm->rank() : 0; }
int Engine::comm_world() const { return impl_->comm ? impl_->comm->world() : 1; }
cudaStream_t Engine::stream() const { return impl_->st; }

Tensor Engine::prefix_infer(const Tensor& x, int k, bool inclusive) {
    Impl& m = *impl_;
    PBKD_CUDA(cudaSetDevice(m.dev));
    g_alloc_stream = m.st;
    if (!m.has_teacher) throw std::logic_error("engine: no teacher loaded");
    const int nb = static_cast<int>(m.tblocks.size());
    if (k < 1 || k > nb) throw std::out_of_range("prefix_infer: k=" + std::to_string(k) + " out of range");
    if (x.c != m.net.in_c || x.h != m.net.in_h || x.w != m.net.in_w)
        throw pbkd::ShapeError("prefix_infer: input shape " + x.shape_str() + " does not match the network");
    const int take = inclusive ? k : k - 1;
    if (take == 0) return x;
    const size_t wsz = static_cast<size_t>(x.n) * m.max_row() * sizeof(float);
    DevBuf a(wsz), b(wsz), t1(wsz), sk(wsz);
    const std::vector<float> in = nchw_to_nhwc(x);
    PBKD_CUDA(cudaMemcpy(a.p, in.data(), in.size() * sizeof(float), cudaMemcpyHostToDevice));
    Program P;
    float* cur = a.f();
    float* nxt = b.f();
    for (int j = 0; j < take; ++j) {
        m.teacher_block(P, j, cur, nxt, x.n, t1.f(), sk.f());
        std::swap(cur, nxt);
    }
    P.run(m.st);
    PBKD_CUDA(cudaStreamSynchronize(m.st));
    const TBlockDev& lb = m.tblocks[static_cast<size_t>(take) - 1];
    std::vector<float> out(static_cast<size_t>(x.n) * lb.cout * lb.hout * lb.wout);
    PBKD_CUDA(cudaMemcpy(out.data(), cur, out.size() * sizeof(float), cudaMemcpyDeviceToHost));
    return nhwc_to_nchw(out, x.n, lb.cout, lb.hout, lb.wout);
}

int candidate_units(const Block& b) {
    int u = 0;
    for (const pbkd::LayerParams& l : b.layers)
        if (l.kind == LayerKind::DepthwiseConv3x3) ++u;
    return u;
}

Tensor Engine::candidate_infer(const Block& cand, const Tensor& x) {
    Impl& m = *impl_;
    PBKD_CUDA(cudaSetDevice(m.dev));
    g_alloc_stream = m.st;
    for (const pbkd::LayerParams& l : cand.layers)
        if (l.kind == LayerKind::Add) throw SpecError("skip candidates are not implemented on the GPU path");
    const int U = candidate_units(cand);
    if (U < 1 || U > kMaxUnits) throw SpecError("not a depthwise-separable candidate block");
    TaskState s;
    s.units = U;
    const int ho = (x.h - 1) / cand.stride + 1, wo = (x.w - 1) / cand.stride + 1;
    std::vector<float> host, stats;
    size_t li = 0;
    for (int u = 0; u < U; ++u) {
        const pbkd::LayerParams& dwl = cand.layers[li];
        const pbkd::LayerParams& pwl = cand.layers[li + 1];
        const pbkd::LayerParams& bnl = cand.layers[li + 2];
        li += 4;
        const int ci = dwl.in_channels, co = pwl.out_channels;
        s.u[u] = u == 0 ? UnitDims{ci, x.h, x.w, co, ho, wo, cand.stride} : UnitDims{ci, ho, wo, co, ho, wo, 1};
        pad4(host);
            s.off_dw[u] = host.size();
        for (int tap = 0; tap < 9; ++tap)
            for (int c = 0; c < ci; ++c) host.push_back(dwl.weight.data[static_cast<size_t>(c) * 9 + tap]);
        pad4(host);
            s.off_pw[u] = host.size();
        host.insert(host.end(), pwl.weight.data.begin(), pwl.weight.data.end());
        pad4(host);
            s.off_g[u] = host.size();
        host.insert(host.end(), bnl.gamma.data.begin(), bnl.gamma.data.end());
        pad4(host);
            s.off_b[u] = host.size();
        host.insert(host.end(), bnl.beta.data.begin(), bnl.beta.data.end());
        stats.insert(stats.end(), bnl.moving_mean.data.begin(), bnl.moving_mean.data.end());
        stats.insert(stats.end(), bnl.moving_var.data.begin(), bnl.moving_var.data.end());
    }
    if (x.c != s.u[0].cin) throw pbkd::ShapeError("candidate input channels do not match");
    s.params = upload(host, m.st);
    s.mstats = upload(stats, m.st);
    const int cout = s.u[0].cout;
    s.scale.alloc(static_cast<size_t>(U) * cout * sizeof(float));
    s.shift.alloc(static_cast<size_t>(U) * cout * sizeof(float));
    const int row = std::max(x.c * x.h * x.w, std::max(cout, x.c) * ho * wo);
    const size_t wsz = static_cast<size_t>(x.n) * row * sizeof(float);
    DevBuf in(wsz), a(wsz), b(wsz), o(wsz);
    const std::vector<float> xin = nchw_to_nhwc(x);
    PBKD_CUDA(cudaMemcpy(in.p, xin.data(), xin.size() * sizeof(float), cudaMemcpyHostToDevice));
    Program P;
    m.add_student_infer(P, s, in.f(), x.n, a.f(), b.f(), o.f());
    P.run(m.st);
    PBKD_CUDA(cudaStreamSynchronize(m.st));
    std::vector<float> out(static_cast<size_t>(x.n) * cout * ho * wo);
    PBKD_CUDA(cudaMemcpy(out.data(), o.p, out.size() * sizeof(float), cudaMemcpyDeviceToHost));
    return nhwc_to_nchw(out, x.n, cout, ho, wo);
}

double Engine::eval_with_student(int block_index, const Block& student, const std::vector<int>& eval_idx) {
    Impl& m = *impl_;
    PBKD_CUDA(cudaSetDevice(m.dev));
    g_alloc_stream = m.st;
    if (eval_idx.empty()) throw SpecError("evaluation split is empty");
    if (block_index < 1 || block_index > static_cast<int>(m.tblocks.size()))
        throw SpecError("block index " + std::to_string(block_index) + " out of range");
    // prefix on host tensors, student, suffix + classifier on device
    std::vector<int> lab;
    pbkd::Dataset d;  // labels only
    std::vector<int> all(static_cast<size_t>(m.count));
    PBKD_CUDA(cudaMemcpy(all.data(), m.labels.p, all.size() * sizeof(int), cudaMemcpyDeviceToHost));
    std::vector<float> img(static_cast<size_t>(m.count) * m.dc * m.dh * m.dw);
    PBKD_CUDA(cudaMemcpy(img.data(), m.images.p, img.size() * sizeof(float), cudaMemcpyDeviceToHost));
    d.c = m.dc;
    d.h = m.dh;
    d.w = m.dw;
    d.images = img;
    d.labels = all;
    const Tensor xb = pbkd::gather_batch(d, eval_idx);
    const Tensor a = prefix_infer(xb, block_index, false);
    const Tensor so = candidate_infer(student, a);
    // suffix
    const int n = xb.n;
    const size_t wsz = static_cast<size_t>(n) * m.max_row() * sizeof(float);
    DevBuf p0(wsz), p1(wsz), t1(wsz), sk(wsz);
    const std::vector<float> sv = nchw_to_nhwc(so);
    PBKD_CUDA(cudaMemcpy(p0.p, sv.data(), sv.size() * sizeof(float), cudaMemcpyHostToDevice));
    Program P;
    float* cur = p0.f();
    float* nxt = p1.f();
    for (size_t j = static_cast<size_t>(block_index); j < m.tblocks.size(); ++j) {
        m.teacher_block(P, static_cast<int>(j), cur, nxt, n, t1.f(), sk.f());
        std::swap(cur, nxt);
    }
    for (int i : eval_idx) lab.push_back(all[static_cast<size_t>(i)]);
    DevBuf dl = upload(lab, m.st);
    DevBuf corr(sizeof(int));
    PBKD_CUDA(cudaMemsetAsync(corr.p, 0, sizeof(int), m.st));
    const float* xin = cur;
    P.raw([&, xin](cudaStream_t s2) {
        launch_classifier_count(xin, n, m.cls_hw, m.cls_in_c, m.cls_kinds.i(), m.cls_layers, m.cls_w.f(),
                                m.cls_b.f(), m.cls_maxw, dl.i(), corr.i(), s2);
    });
    P.run(m.st);
    int c = 0;
    PBKD_CUDA(cudaMemcpyAsync(&c, corr.p, sizeof(int), cudaMemcpyDeviceToHost, m.st));
    PBKD_CUDA(cudaStreamSynchronize(m.st));
    return static_cast<double>(c) / static_cast<double>(eval_idx.size());
}

}  // namespace pbkd_gpu
