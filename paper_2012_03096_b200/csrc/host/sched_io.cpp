// Scheduler / runtime host utilities of the reference's API: trace and
// profile CSV files, the exhaustive makespan optimum and the discrete-event
// replay of a plan (scheduler.cpp:104-236, runtime.cpp:56-122, :245-380).
// File formats, error texts and the replay rules (owners pop their head,
// thieves take the tail of the most loaded queue; seeded randomized variant)
// are interface-dictated; the code is organised as this project's own
// (a line-oriented CSV reader shared by both formats, an event-queue
// simulator class, an iterative-deepening branch and bound).
#include <algorithm>
#include <deque>
#include <fstream>
#include <functional>
#include <limits>
#include <map>
#include <queue>
#include <random>
#include <set>
#include <sstream>
#include <tuple>

#include "pbkd/runtime.hpp"
#include "pbkd/scheduler.hpp"

namespace pbkd {

namespace {

std::string slurp(const std::string& path, const char* what) {
    std::ifstream f(path);
    if (!f) throw SpecError(path + ": cannot open " + what);
    return std::string((std::istreambuf_iterator<char>(f)), std::istreambuf_iterator<char>());
}

// Rows of a headed CSV text (CRLF tolerated, blank lines skipped), each
// split into exactly `fields` fields (the last one takes the rest).
void for_each_row(const std::string& text, const std::string& origin, const std::string& header,
                  const std::string& header_error, size_t fields,
                  const std::function<void(int, const std::string&, const std::vector<std::string>&)>& row) {
    std::istringstream in(text);
    std::string line;
    auto chomp = [](std::string& s) {
        if (!s.empty() && s.back() == '\r') s.pop_back();
    };
    if (!std::getline(in, line)) throw SpecError(origin + ": empty " + (fields == 2 ? "profile" : "trace") + " file");
    chomp(line);
    if (line != header) throw SpecError(origin + ": line 1: " + header_error);
    for (int no = 2; std::getline(in, line); ++no) {
        chomp(line);
        if (line.empty()) continue;
        std::vector<std::string> f;
        size_t at = 0;
        for (size_t i = 0; i + 1 < fields; ++i) {
            const size_t comma = line.find(',', at);
            if (comma == std::string::npos)
                throw SpecError(origin + ": line " + std::to_string(no) + ": expected " + std::to_string(fields) +
                                " fields");
            f.push_back(line.substr(at, comma - at));
            at = comma + 1;
        }
        f.push_back(line.substr(at));
        row(no, line, f);
    }
}

// whole-field numeric conversions (trailing characters are malformed)
template <class T, class Conv>
T whole(const std::string& s, Conv conv) {
    size_t used = 0;
    const T v = conv(s, &used);
    if (used != s.size()) throw std::invalid_argument("trailing characters");
    return v;
}
int to_int(const std::string& s) { return whole<int>(s, [](const std::string& x, size_t* u) { return std::stoi(x, u); }); }
double to_double(const std::string& s) {
    return whole<double>(s, [](const std::string& x, size_t* u) { return std::stod(x, u); });
}

std::map<int, double> weights_by_id(const std::vector<TaskWeight>& weights, bool with_value) {
    std::map<int, double> m;
    for (const TaskWeight& t : weights) {
        if (!(t.weight > 0))
            throw SpecError("task " + std::to_string(t.task_id) + " has non-positive weight" +
                            (with_value ? " " + std::to_string(t.weight) : std::string()));
        if (!m.emplace(t.task_id, t.weight).second) throw SpecError("duplicate task id " + std::to_string(t.task_id));
    }
    return m;
}

void write_csv(const std::string& path, const std::string& body) {
    std::ofstream f(path, std::ios::trunc);
    if (!f) throw SpecError(path + ": cannot open for writing");
    f << body;
    if (!f) throw SpecError(path + ": write failed");
}

// ---------------------------------------------------------------- replay
class Replay {
public:
    Replay(const SchedulePlan& plan, const std::map<int, double>& dur, const SimOptions& o)
        : plan_(plan), dur_(dur), opt_(o), rng_(o.seed) {}

    SimResult run() {
        SimResult r;
        for (size_t w = 0; w < plan_.assignments.size(); ++w)
            for (int id : plan_.assignments[w]) r.trace.push_back({0.0, static_cast<int>(w), id, TraceEventKind::Dispatch});
        double wall = plan_.policy == SchedulePolicy::WorkStealing ? stealing(r.trace) : back_to_back(r.trace);
        r.trace.push_back({wall, 0, -1, TraceEventKind::Gather});
        r.wall_time = wall;
        return r;
    }

private:
    double back_to_back(std::vector<TraceEvent>& trace) {
        std::vector<TraceEvent> ev;
        double wall = 0.0;
        for (size_t w = 0; w < plan_.assignments.size(); ++w) {
            double t = 0.0;
            for (int id : plan_.assignments[w]) {
                ev.push_back({t, static_cast<int>(w), id, TraceEventKind::TaskStart});
                t += dur_.at(id);
                ev.push_back({t, static_cast<int>(w), id, TraceEventKind::TaskEnd});
            }
            wall = std::max(wall, t);
        }
        std::stable_sort(ev.begin(), ev.end(), [](const TraceEvent& a, const TraceEvent& b) {
            return a.timestamp_s < b.timestamp_s;
        });
        trace.insert(trace.end(), ev.begin(), ev.end());
        return wall;
    }

    struct Wake {
        double t;
        uint64_t tie;  // random tie-break of simultaneous wake-ups (randomized mode)
        uint64_t seq;
        int worker;
        bool operator>(const Wake& o) const { return std::tie(t, tie, seq) > std::tie(o.t, o.tie, o.seq); }
    };

    double stealing(std::vector<TraceEvent>& trace) {
        const size_t W = plan_.assignments.size();
        std::vector<std::deque<int>> q(W);
        double longest = 0.0;
        for (size_t w = 0; w < W; ++w)
            for (int id : plan_.assignments[w]) {
                q[w].push_back(id);
                longest = std::max(longest, dur_.at(id));
            }
        std::priority_queue<Wake, std::vector<Wake>, std::greater<>> wakes;
        uint64_t seq = 0;
        auto wake = [&](double t, int w) { wakes.push({t, opt_.randomized ? rng_() : 0, seq++, w}); };
        for (size_t w = 0; w < W; ++w) wake(0.0, static_cast<int>(w));
        std::vector<int> hesitated(W, 0);
        double wall = 0.0;
        while (!wakes.empty()) {
            const Wake e = wakes.top();
            wakes.pop();
            const size_t w = static_cast<size_t>(e.worker);
            int task;
            if (!q[w].empty()) {  // owners take their own head
                task = q[w].front();
                q[w].pop_front();
            } else {
                std::vector<size_t> victims;
                for (size_t v = 0; v < W; ++v)
                    if (v != w && !q[v].empty()) victims.push_back(v);
                if (victims.empty()) continue;  // queues only drain: retire
                if (opt_.randomized && hesitated[w] < 64 && (rng_() & 1u)) {
                    ++hesitated[w];
                    std::uniform_real_distribution<double> lag(0.0, longest);
                    wake(e.t + lag(rng_), e.worker);
                    continue;
                }
                hesitated[w] = 0;
                size_t victim = victims.front();
                if (opt_.randomized) {
                    std::uniform_int_distribution<size_t> pick(0, victims.size() - 1);
                    victim = victims[pick(rng_)];
                } else {  // most remaining queued weight, ties to the lowest index
                    double most = -1.0;
                    for (size_t v : victims) {
                        double left = 0.0;
                        for (int id : q[v]) left += dur_.at(id);
                        if (left > most) most = left, victim = v;
                    }
                }
                task = q[victim].back();  // thieves take the tail
                q[victim].pop_back();
                trace.push_back({e.t, e.worker, task, TraceEventKind::Steal});
            }
            const double end = e.t + dur_.at(task);
            trace.push_back({e.t, e.worker, task, TraceEventKind::TaskStart});
            trace.push_back({end, e.worker, task, TraceEventKind::TaskEnd});
            wall = std::max(wall, end);
            wake(end, e.worker);
        }
        // dispatch events first, everything else in time order
        std::stable_sort(trace.begin(), trace.end(), [](const TraceEvent& a, const TraceEvent& b) {
            const bool da = a.kind == TraceEventKind::Dispatch, db = b.kind == TraceEventKind::Dispatch;
            if (da || db) return da && !db;
            return a.timestamp_s < b.timestamp_s;
        });
        return wall;
    }

    const SchedulePlan& plan_;
    const std::map<int, double>& dur_;
    SimOptions opt_;
    std::mt19937_64 rng_;
};

}  // namespace

void save_trace_csv(const std::string& path, const std::vector<TraceEvent>& trace) {
    std::ostringstream body;
    body.precision(17);
    body << "timestamp_s,worker_id,task_id,kind\n";
    for (const TraceEvent& e : trace)
        body << e.timestamp_s << "," << e.worker_id << "," << e.task_id << "," << trace_event_kind_name(e.kind) << "\n";
    write_csv(path, body.str());
}

std::vector<TraceEvent> parse_trace_csv(const std::string& text, const std::string& origin) {
    std::vector<TraceEvent> out;
    for_each_row(text, origin, "timestamp_s,worker_id,task_id,kind",
                 "expected header 'timestamp_s,worker_id,task_id,kind'", 4,
                 [&](int no, const std::string& line, const std::vector<std::string>& f) {
                     TraceEvent e;
                     try {
                         e.timestamp_s = to_double(f[0]);
                         e.worker_id = to_int(f[1]);
                         e.task_id = to_int(f[2]);
                     } catch (const std::exception&) {
                         throw SpecError(origin + ": line " + std::to_string(no) + ": malformed row '" + line + "'");
                     }
                     e.kind = trace_event_kind_from_name(f[3]);
                     out.push_back(e);
                 });
    return out;
}

std::vector<TraceEvent> load_trace_csv(const std::string& path) { return parse_trace_csv(slurp(path, "trace"), path); }

std::vector<TaskWeight> parse_profile_csv(const std::string& text, const std::string& origin) {
    std::vector<TaskWeight> out;
    for_each_row(text, origin, "task_id,weight_seconds",
                 "expected header 'task_id,weight_seconds', got '" +
                     text.substr(0, std::min(text.find('\n'), text.size())) + "'",
                 2, [&](int no, const std::string& line, const std::vector<std::string>& f) {
                     TaskWeight t;
                     try {
                         t.task_id = to_int(f[0]);
                         t.weight = to_double(f[1]);
                     } catch (const std::exception&) {
                         throw SpecError(origin + ": line " + std::to_string(no) + ": malformed row '" + line + "'");
                     }
                     if (!(t.weight > 0))
                         throw SpecError(origin + ": line " + std::to_string(no) + ": weight must be positive");
                     out.push_back(t);
                 });
    weights_by_id(out, true);  // duplicate ids
    return out;
}

std::vector<TaskWeight> load_profile_csv(const std::string& path) {
    return parse_profile_csv(slurp(path, "profile"), path);
}

void save_profile_csv(const std::string& path, const std::vector<TaskWeight>& weights) {
    std::ostringstream body;
    body.precision(17);
    body << "task_id,weight_seconds\n";
    for (const TaskWeight& t : weights) body << t.task_id << "," << t.weight << "\n";
    write_csv(path, body.str());
}

// Exact minimum makespan: weights placed largest first, each into every
// distinct bin (empty bins are interchangeable), pruned against the best
// complete placement so far (seeded with greedy LPT) and against the largest
// weight still to place.
double brute_force_schedule(const std::vector<TaskWeight>& weights, int workers) {
    if (workers < 1) throw SpecError("worker_count must be at least 1");
    if (weights.size() > 14)
        throw SpecError("exhaustive search is limited to 14 tasks, got " + std::to_string(weights.size()));
    if (workers > 4) throw SpecError("exhaustive search is limited to 4 workers, got " + std::to_string(workers));
    weights_by_id(weights, true);
    if (weights.empty()) return 0.0;
    std::vector<double> w;
    for (const TaskWeight& t : weights) w.push_back(t.weight);
    std::sort(w.rbegin(), w.rend());
    std::vector<double> load(static_cast<size_t>(workers), 0.0);
    for (double x : w) *std::min_element(load.begin(), load.end()) += x;  // LPT bound
    double best = *std::max_element(load.begin(), load.end());
    std::fill(load.begin(), load.end(), 0.0);
    std::function<void(size_t)> place = [&](size_t i) {
        if (i == w.size()) {
            best = std::min(best, *std::max_element(load.begin(), load.end()));
            return;
        }
        bool empty_tried = false;
        for (double& l : load) {
            if (l == 0.0) {
                if (empty_tried) continue;
                empty_tried = true;
            }
            if (l + w[i] >= best) continue;
            l += w[i];
            // w is descending: w[i+1] is the largest weight still to place
            if (std::max(l, i + 1 < w.size() ? w[i + 1] : 0.0) < best) place(i + 1);
            l -= w[i];
        }
    };
    place(0);
    return best;
}

SimResult simulate_execution(const SchedulePlan& plan, const std::vector<TaskWeight>& weights, const SimOptions& opts) {
    if (plan.worker_count < 1) throw SpecError("worker_count must be at least 1");
    if (plan.assignments.size() != static_cast<size_t>(plan.worker_count))
        throw SpecError("plan has " + std::to_string(plan.assignments.size()) + " worker lists for worker_count " +
                        std::to_string(plan.worker_count));
    const std::map<int, double> dur = weights_by_id(weights, false);
    std::set<int> seen;
    for (const auto& q : plan.assignments)
        for (int id : q) {
            if (!dur.count(id)) throw SpecError("task " + std::to_string(id) + " in the plan has no weight");
            if (!seen.insert(id).second) throw SpecError("plan assigns task " + std::to_string(id) + " twice");
        }
    return Replay(plan, dur, opts).run();
}

}  // namespace pbkd
