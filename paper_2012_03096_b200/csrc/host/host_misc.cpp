// Host-side, bit-exact pieces of the hot path that stay on the CPU:
// candidate construction (replacement.cpp:11-82), activation indexing
// (dataset.cpp:136-185, distill.cpp:22-30,198-200) and block assignment
// (scheduler.cpp:43-102, pipeline.cpp:65-85).  Same libstdc++ engines and
// distributions as the reference, so seeds produce identical bits.
#include <algorithm>
#include <cmath>
#include <set>

#include "pbkd/dataset.hpp"
#include "pbkd/distill.hpp"
#include "pbkd/replacement.hpp"
#include "pbkd/scheduler.hpp"

namespace pbkd {

// ------------------------------------------------------------ candidates --
const char* candidate_kind_name(CandidateKind k) {
    switch (k) {
        case CandidateKind::TwoLayer: return "two_layer";
        case CandidateKind::ThreeLayer: return "three_layer";
        case CandidateKind::TwoLayerSkip: return "two_layer_skip";
        case CandidateKind::ThreeLayerSkip: return "three_layer_skip";
    }
    return "unknown";
}

CandidateKind candidate_kind_from_name(const std::string& name) {
    for (CandidateKind k : kAllCandidates)
        if (name == candidate_kind_name(k)) return k;
    throw SpecError("unknown replacement candidate '" + name + "'");
}

ReplacementBlock build_candidate(CandidateKind kind, int c_in, int c_out, int stride, uint64_t seed) {
    if (c_in < 1 || c_out < 1)
        throw std::invalid_argument("build_candidate: channel counts must be >= 1");
    if (stride != 1 && stride != 2)
        throw std::invalid_argument("build_candidate: stride must be 1 or 2");
    ReplacementBlock r;
    r.kind = kind;
    Block& b = r.block;
    b.name = "replacement";
    b.spec_kind = candidate_kind_name(kind);
    b.in_channels = c_in;
    b.out_channels = c_out;
    b.stride = stride;
    b.padding = 1;
    const bool skip = kind == CandidateKind::TwoLayerSkip || kind == CandidateKind::ThreeLayerSkip;
    const int units = (kind == CandidateKind::ThreeLayer || kind == CandidateKind::ThreeLayerSkip) ? 3 : 2;
    for (int u = 0; u < units; ++u) {
        const int ci = u == 0 ? c_in : c_out;
        b.layers.push_back(make_conv_layer(LayerKind::DepthwiseConv3x3, ci, ci, 3, u == 0 ? stride : 1, 1));
        b.layers.push_back(make_conv_layer(LayerKind::PointwiseConv, ci, c_out, 1, 1, 0));
        b.layers.push_back(make_batchnorm_layer(c_out));
        if (!(skip && u == units - 1)) b.layers.push_back(make_relu_layer(c_out));
    }
    if (skip) {
        b.layers.push_back(make_add_layer(c_in, c_out, stride));
        b.layers.push_back(make_relu_layer(c_out));
    }
    std::mt19937_64 rng(seed);
    init_block_weights(b, rng);
    return r;
}

ReplacementBlock default_replacement(int c_in, int c_out, int stride, uint64_t seed) {
    return build_candidate(CandidateKind::TwoLayer, c_in, c_out, stride, seed);
}

bool is_replacement_block(const Block& b) {
    for (CandidateKind k : kAllCandidates)
        if (b.spec_kind == candidate_kind_name(k)) return true;
    return false;
}

// ---------------------------------------------------------------- dataset --
SplitIndices stratified_split(const Dataset& d, double frac, uint64_t seed) {
    if (d.count() == 0) throw std::invalid_argument("stratified_split: dataset is empty");
    if (!(frac > 0.0 && frac < 1.0))
        throw std::invalid_argument("stratified_split: eval_fraction must be in (0,1)");
    std::vector<std::vector<int>> per_class;
    for (int i = 0; i < d.count(); ++i) {
        const int lab = d.labels[static_cast<size_t>(i)];
        if (lab >= static_cast<int>(per_class.size())) per_class.resize(static_cast<size_t>(lab) + 1);
        per_class[static_cast<size_t>(lab)].push_back(i);
    }
    SplitIndices s;
    for (size_t cls = 0; cls < per_class.size(); ++cls) {
        std::vector<int>& m = per_class[cls];
        if (m.empty()) continue;
        std::mt19937_64 rng(mix_seed(seed, cls));
        std::shuffle(m.begin(), m.end(), rng);
        if (m.size() < 2)
            throw std::invalid_argument("stratified_split: class " + std::to_string(cls) +
                                        " has fewer than 2 samples");
        size_t take = static_cast<size_t>(std::lround(frac * static_cast<double>(m.size())));
        take = std::clamp<size_t>(take, 1, m.size() - 1);
        s.eval_idx.insert(s.eval_idx.end(), m.begin(), m.begin() + static_cast<long>(take));
        s.train_idx.insert(s.train_idx.end(), m.begin() + static_cast<long>(take), m.end());
    }
    std::sort(s.eval_idx.begin(), s.eval_idx.end());
    std::sort(s.train_idx.begin(), s.train_idx.end());
    return s;
}

Tensor gather_batch(const Dataset& d, std::span<const int> idx) {
    if (idx.empty()) throw std::invalid_argument("gather_batch: empty index list");
    Tensor b(static_cast<int>(idx.size()), d.c, d.h, d.w);
    const size_t sz = d.image_size();
    for (size_t i = 0; i < idx.size(); ++i) {
        if (idx[i] < 0 || idx[i] >= d.count()) throw std::out_of_range("gather_batch: index out of range");
        std::copy_n(d.images.begin() + static_cast<long>(static_cast<size_t>(idx[i]) * sz), sz,
                    b.data.begin() + static_cast<long>(i * sz));
    }
    return b;
}

std::vector<int> gather_labels(const Dataset& d, std::span<const int> idx) {
    std::vector<int> out;
    out.reserve(idx.size());
    for (int i : idx) out.push_back(d.labels.at(static_cast<size_t>(i)));
    return out;
}

std::vector<int> epoch_order(const std::vector<int>& train_idx, uint64_t task_seed, int epoch) {
    std::vector<int> order = train_idx;
    std::mt19937_64 rng(mix_seed(task_seed, static_cast<uint64_t>(epoch)));
    std::shuffle(order.begin(), order.end(), rng);
    return order;
}

// -------------------------------------------------------------- scheduler --
namespace {
void check_weights(const std::vector<TaskWeight>& ws) {
    std::set<int> seen;
    for (const TaskWeight& t : ws) {
        if (!(t.weight > 0))
            throw SpecError("task " + std::to_string(t.task_id) + " has non-positive weight");
        if (!seen.insert(t.task_id).second) throw SpecError("duplicate task id " + std::to_string(t.task_id));
    }
}
}  // namespace

const char* schedule_policy_name(SchedulePolicy p) {
    switch (p) {
        case SchedulePolicy::RoundRobin: return "round_robin";
        case SchedulePolicy::WFD: return "wfd";
        case SchedulePolicy::WorkStealing: return "work_stealing";
    }
    return "unknown";
}

SchedulePolicy schedule_policy_from_name(const std::string& name) {
    if (name == "round_robin") return SchedulePolicy::RoundRobin;
    if (name == "wfd") return SchedulePolicy::WFD;
    if (name == "work_stealing") return SchedulePolicy::WorkStealing;
    throw SpecError("unknown scheduling policy '" + name + "'");
}

SchedulePlan round_robin(const std::vector<int>& ids, int workers) {
    if (workers < 1) throw SpecError("worker_count must be at least 1");
    std::set<int> seen;
    for (int id : ids)
        if (!seen.insert(id).second) throw SpecError("duplicate task id " + std::to_string(id));
    SchedulePlan p;
    p.worker_count = workers;
    p.policy = SchedulePolicy::RoundRobin;
    p.assignments.assign(static_cast<size_t>(workers), {});
    for (size_t i = 0; i < ids.size(); ++i) p.assignments[i % static_cast<size_t>(workers)].push_back(ids[i]);
    return p;
}

SchedulePlan wfd_bin_pack(const std::vector<TaskWeight>& weights, int workers) {
    if (workers < 1) throw SpecError("worker_count must be at least 1");
    check_weights(weights);
    std::vector<TaskWeight> order = weights;
    // heaviest first, equal weights by ascending id; least-loaded bin, lowest index on ties
    std::stable_sort(order.begin(), order.end(), [](const TaskWeight& a, const TaskWeight& b) {
        return a.weight != b.weight ? a.weight > b.weight : a.task_id < b.task_id;
    });
    SchedulePlan p;
    p.worker_count = workers;
    p.policy = SchedulePolicy::WFD;
    p.assignments.assign(static_cast<size_t>(workers), {});
    std::vector<double> load(static_cast<size_t>(workers), 0.0);
    for (const TaskWeight& t : order) {
        size_t bin = 0;
        for (size_t w = 1; w < load.size(); ++w)
            if (load[w] < load[bin]) bin = w;
        p.assignments[bin].push_back(t.task_id);
        load[bin] += t.weight;
    }
    p.predicted_makespan = *std::max_element(load.begin(), load.end());
    return p;
}

double makespan(const SchedulePlan& plan, const std::vector<TaskWeight>& weights) {
    double worst = 0.0;
    for (const std::vector<int>& q : plan.assignments) {
        double s = 0.0;
        for (int id : q) {
            auto it = std::find_if(weights.begin(), weights.end(),
                                   [id](const TaskWeight& t) { return t.task_id == id; });
            if (it == weights.end()) throw SpecError("task " + std::to_string(id) + " in the plan has no weight");
            s += it->weight;
        }
        worst = std::max(worst, s);
    }
    return worst;
}

std::vector<TaskWeight> mac_proxy_weights(const Network& net, const std::vector<int>& blocks) {
    const CostTable table = count_macs_params(net);
    std::vector<TaskWeight> out;
    for (int k : blocks) {
        const std::string pre = net.blocks.at(static_cast<size_t>(k) - 1).name + "/";
        double macs = 0;
        for (const CostRow& r : table.rows)
            if (r.layer.rfind(pre, 0) == 0) macs += static_cast<double>(r.macs);
        out.push_back({k, macs * 1e-6});
    }
    return out;
}

// ------------------------------------------------------------- loss names --
const char* loss_mode_name(LossMode m) { return m == LossMode::LocalOnly ? "local_only" : "combined"; }

LossMode loss_mode_from_name(const std::string& name) {
    if (name == "local_only" || name == "local") return LossMode::LocalOnly;
    if (name == "combined") return LossMode::Combined;
    throw SpecError("unknown loss mode '" + name + "'");
}

}  // namespace pbkd
