// nettrain.cu -- whole-network / generic-candidate training loops (nettrain.hpp).
#include <algorithm>
#include <chrono>
#include <cmath>
#include <numeric>
#include <random>
#include <sstream>

#include "nettrain.hpp"
#include "pbkd/replacement.hpp"

namespace pbkd_gpu {

using pbkd::Block;
using pbkd::Network;

namespace {

size_t block_floats(const Block& b) {
    size_t n = 0;
    pbkd::for_each_block_array(const_cast<Block&>(b), [&](const std::string&, pbkd::Tensor& t) { n += t.data.size(); });
    return n;
}

// std::shuffle over positions 0..n-1 with the reference's engine: the
// permutation depends only on n and the engine (distill.cpp:198-200)
std::vector<int> shuffled_positions(int n, uint64_t seed, int epoch) {
    std::vector<int> pos(static_cast<size_t>(n));
    std::iota(pos.begin(), pos.end(), 0);
    std::mt19937_64 rng(pbkd::mix_seed(seed, static_cast<uint64_t>(epoch)));
    std::shuffle(pos.begin(), pos.end(), rng);
    return pos;
}

std::vector<std::vector<int>> batches_of(const std::vector<int>& v, int b) {  // distill.cpp:22-30
    std::vector<std::vector<int>> out;
    for (size_t at = 0; at < v.size(); at += static_cast<size_t>(b))
        out.emplace_back(v.begin() + static_cast<long>(at), v.begin() + static_cast<long>(std::min(v.size(), at + b)));
    return out;
}

std::vector<float> block_to_host(NetExec& X, const DevBlock& b) {
    std::vector<float> v(static_cast<size_t>(b.n));
    X.arrays_to_host(b, v.data());
    return v;
}

}  // namespace

DevNet make_devnet(NetExec& X, const Network& net, const float* flat, bool on_dev) {
    DevNet d;
    size_t off = 0;
    for (const Block& b : net.blocks) {
        d.blocks.push_back(X.make_block(b, flat ? flat + off : nullptr, on_dev));
        d.replacement.push_back(pbkd::is_replacement_block(b));
        off += block_floats(b);
    }
    d.has_cls = net.has_classifier();
    if (d.has_cls) d.cls = X.make_block(net.classifier, flat ? flat + off : nullptr, on_dev);
    return d;
}

void devnet_to_host(NetExec& X, const DevNet& d, float* flat) {
    size_t off = 0;
    for (const DevBlock& b : d.blocks) {
        X.arrays_to_host(b, flat + off);
        off += static_cast<size_t>(b.n);
    }
    if (d.has_cls) X.arrays_to_host(d.cls, flat + off);
}

DTensor NetTrainer::images(const std::vector<int>& idx) {
    for (int i : idx)
        if (i < 0 || i >= d_.count) throw std::out_of_range("gather_batch: index out of range");
    DTensor di = X_.upload_ints(idx);
    return X_.gather(d_.images, reinterpret_cast<const int*>(di.p), static_cast<int>(idx.size()), d_.c, d_.h, d_.w);
}

DTensor NetTrainer::labels(const std::vector<int>& idx) {
    std::vector<int> l;
    l.reserve(idx.size());
    for (int i : idx) l.push_back(d_.labels.at(static_cast<size_t>(i)));
    return X_.upload_ints(l);
}

DTensor NetTrainer::infer(DevNet& net, DTensor x, size_t from, bool head) {
    for (size_t i = from; i < net.blocks.size(); ++i) x = X_.forward(net.blocks[i], x, false, nullptr);
    if (head && net.has_cls) x = X_.forward(net.cls, x, false, nullptr);
    return x;
}

// distill.cpp:286-295 (batch-independent: inference is per sample)
double NetTrainer::evaluate(DevNet& net, const std::vector<int>& idx, int batch) {
    if (idx.empty()) throw pbkd::SpecError("evaluation split is empty");
    if (batch < 1) throw pbkd::SpecError("batch_size must be at least 1");
    long long correct = 0;
    for (const auto& b : batches_of(idx, std::max(batch, 256))) {
        DTensor lab = labels(b);
        correct += X_.count_correct(infer(net, images(b), 0, true), reinterpret_cast<const int*>(lab.p));
    }
    return static_cast<double>(correct) / static_cast<double>(idx.size());
}

FitResult NetTrainer::fit(DevNet& net, const std::vector<int>& train, const std::vector<int>& eval, int epochs,
                          bool freeze, float lr, float momentum, int batch, uint64_t seed, bool teacher_mode) {
    if (epochs < 0) throw pbkd::SpecError("epochs must be non-negative");
    if (batch < 1) throw pbkd::SpecError("batch_size must be at least 1");
    if (train.empty()) throw pbkd::SpecError("training split is empty");
    if (!net.has_cls) throw pbkd::SpecError(teacher_mode ? "training needs a classifier head"
                                                         : "fine-tuning needs a classifier head");
    FitResult fr;
    fr.initial_eval = evaluate(net, eval, batch);
    fr.final_eval = fr.initial_eval;
    fr.eval_history.push_back({0, fr.initial_eval});
    // train mask (distill.cpp:346-359): frozen blocks run inference-mode BN
    const size_t nb = net.blocks.size();
    std::vector<bool> trains(nb, true);
    bool any = !freeze;
    if (freeze)
        for (size_t i = 0; i < nb; ++i) any |= (trains[i] = net.replacement[i]);
    if (epochs == 0 || !any) return fr;  // nothing to train is a no-op
    const bool train_cls = !freeze;
    for (int epoch = 1; epoch <= epochs; ++epoch) {
        const std::vector<int> pos = shuffled_positions(static_cast<int>(train.size()), seed, epoch);
        std::vector<int> order;
        order.reserve(pos.size());
        for (int p : pos) order.push_back(train[static_cast<size_t>(p)]);
        double loss_sum = 0.0;
        int done = 0;
        for (const auto& b : batches_of(order, batch)) {
            DTensor lab = labels(b);
            const int* ld = reinterpret_cast<const int*>(lab.p);
            std::vector<BlockCacheDev> caches(nb);
            BlockCacheDev ccache;
            DTensor cur = images(b);
            for (size_t i = 0; i < nb; ++i) cur = X_.forward(net.blocks[i], cur, trains[i], &caches[i]);
            DTensor logits = X_.forward(net.cls, cur, true, &ccache);
            DTensor probs;
            const double ce = X_.softmax_ce(logits, ld, &probs);
            if (!std::isfinite(ce))
                throw std::runtime_error(std::string(teacher_mode ? "teacher training" : "fine-tuning") +
                                         " diverged at epoch " + std::to_string(epoch));
            DTensor glog = X_.alloc(logits.n, logits.c, 1, 1, true);
            X_.softmax_ce_bwd(probs, ld, 1.0f, glog);
            for (size_t i = 0; i < nb; ++i)
                if (trains[i]) X_.zero_grads(net.blocks[i]);
            if (train_cls) X_.zero_grads(net.cls);
            // network_backward (model.cpp:671-686)
            DTensor g = X_.backward(net.cls, ccache, glog, nb > 0, train_cls);
            for (size_t i = nb; i-- > 0;) g = X_.backward(net.blocks[i], caches[i], g, i > 0, trains[i]);
            for (size_t i = 0; i < nb; ++i)
                if (trains[i]) X_.sgd(net.blocks[i], lr, momentum);
            if (train_cls) X_.sgd(net.cls, lr, momentum);
            loss_sum += ce;
            ++done;
        }
        fr.loss_history.push_back(loss_sum / done);
        const double acc = evaluate(net, eval, batch);
        fr.eval_history.push_back({epoch, acc});
        fr.final_eval = acc;
    }
    return fr;
}

TaskOutcome NetTrainer::train_block(DevNet& teacher, const Network& shape, const pbkd::DistillTask& t,
                                    const std::vector<int>& train, const std::vector<int>& eval, bool with_eval) {
    const auto t0 = std::chrono::steady_clock::now();
    auto elapsed = [&] { return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(); };
    TaskOutcome res;
    res.block_index = t.block_index;
    res.kind = pbkd::candidate_kind_name(t.kind);
    res.best_eval = -1.0;
    const int k = t.block_index;
    const Block& tb = shape.blocks.at(static_cast<size_t>(k) - 1);
    pbkd::ReplacementBlock cand =
        pbkd::build_candidate(t.kind, tb.in_channels, tb.out_channels, tb.stride, pbkd::mix_seed(t.seed, 0));
    DevBlock student = X_.make_block(cand.block);
    const bool combined = t.loss_mode == pbkd::LossMode::Combined;
    const int ntr = static_cast<int>(train.size());

    // teacher boundaries k-1 and k of the training split (train order) and
    // boundary k-1 of the evaluation split: inference-mode BN is per sample,
    // so computing them once equals prefix_infer + block_infer per batch
    auto boundary = [&](const std::vector<int>& idx, size_t upto, DTensor* before) {
        DTensor out;
        const int chunk = 256;
        for (int at = 0; at < static_cast<int>(idx.size()); at += chunk) {
            const std::vector<int> part(idx.begin() + at, idx.begin() + std::min<size_t>(idx.size(), at + chunk));
            DTensor cur = images(part);
            for (size_t j = 0; j < upto; ++j) {
                if (j + 1 == upto && before) {
                    if (!*before) *before = X_.alloc(static_cast<int>(idx.size()), cur.c, cur.h, cur.w);
                    X_.put_samples(*before, at, cur);
                }
                cur = X_.forward(teacher.blocks[j], cur, false, nullptr);
            }
            if (upto == 0 && before) {
                if (!*before) *before = X_.alloc(static_cast<int>(idx.size()), cur.c, cur.h, cur.w);
                X_.put_samples(*before, at, cur);
            }
            if (!out) out = X_.alloc(static_cast<int>(idx.size()), cur.c, cur.h, cur.w);
            X_.put_samples(out, at, cur);
        }
        return out;
    };
    DTensor a_train;
    DTensor t_train = boundary(train, static_cast<size_t>(k), &a_train);
    DTensor a_eval;
    if (with_eval) a_eval = boundary(eval, static_cast<size_t>(k) - 1, nullptr);

    // Combined objective: logits of the frozen remainder (distill.cpp:65-84)
    auto remainder = [&](DTensor s, std::vector<BlockCacheDev>* caches, BlockCacheDev* cc) {
        const size_t nb = teacher.blocks.size();
        if (caches) caches->assign(nb - static_cast<size_t>(k), BlockCacheDev{});
        for (size_t bi = static_cast<size_t>(k); bi < nb; ++bi)
            s = X_.forward(teacher.blocks[bi], s, false, caches ? &(*caches)[bi - k] : nullptr);
        return X_.forward(teacher.cls, s, false, cc);
    };
    auto record_eval = [&](int epoch) {
        long long correct = 0;
        for (int at = 0; at < static_cast<int>(eval.size()); at += 256) {
            const int n = std::min<int>(256, static_cast<int>(eval.size()) - at);
            DTensor cur = X_.forward(student, X_.slice_samples(a_eval, at, n), false, nullptr);
            DTensor logits = infer(teacher, cur, static_cast<size_t>(k), true);
            DTensor lab = labels(std::vector<int>(eval.begin() + at, eval.begin() + at + n));
            correct += X_.count_correct(logits, reinterpret_cast<const int*>(lab.p));
        }
        const double acc = static_cast<double>(correct) / static_cast<double>(eval.size());
        res.eval_history.push_back({epoch, acc});
        if (acc > res.best_eval) {
            res.best_eval = acc;
            res.best_block = block_to_host(X_, student);
        }
    };

    if (with_eval) {  // epoch-0 objective of the untouched student (distill.cpp:166-192)
        double obj_sum = 0.0, local_sum = 0.0;
        int nbat = 0;
        for (int at = 0; at < ntr; at += t.batch_size, ++nbat) {
            const int n = std::min(t.batch_size, ntr - at);
            DTensor tt = X_.slice_samples(t_train, at, n);
            DTensor so = X_.forward(student, X_.slice_samples(a_train, at, n), false, nullptr);
            const double local = X_.mse(so, tt);
            double obj = local;
            if (combined) {
                DTensor lab = labels(std::vector<int>(train.begin() + at, train.begin() + at + n));
                const double ce = X_.softmax_ce(remainder(so, nullptr, nullptr), reinterpret_cast<const int*>(lab.p),
                                                nullptr);
                obj = static_cast<double>(t.lambda_local) * local + ce;
            }
            obj_sum += obj;
            local_sum += local;
        }
        res.loss_history.push_back(obj_sum / nbat);
        res.final_local_loss = local_sum / nbat;
        record_eval(0);
    }

    long long steps = 0;
    bool cap = false;
    for (int epoch = 1; epoch <= t.epochs && !cap; ++epoch) {
        const std::vector<int> pos = shuffled_positions(ntr, t.seed, epoch);
        double obj_sum = 0.0, local_sum = 0.0;
        int done = 0;
        for (const auto& b : batches_of(pos, t.batch_size)) {
            if (t.max_steps > 0 && steps >= t.max_steps) {
                cap = true;
                break;
            }
            const int n = static_cast<int>(b.size());
            DTensor dpos = X_.upload_ints(b);
            const int* pd = reinterpret_cast<const int*>(dpos.p);
            DTensor a = X_.take_samples(a_train, pd, n), tt = X_.take_samples(t_train, pd, n);
            BlockCacheDev cache;
            DTensor so = X_.forward(student, a, true, &cache);
            const double local = X_.mse_step(so, tt);  // the grouped path's step-loss order
            DTensor gs = X_.alloc(so.n, so.c, so.h, so.w, true);
            double obj = local;
            if (!combined) {
                X_.mse_bwd(so, tt, 1.0f, gs);
            } else {
                if (t.lambda_local > 0) X_.mse_bwd(so, tt, t.lambda_local, gs);
                std::vector<int> rows;
                for (int p : b) rows.push_back(train[static_cast<size_t>(p)]);
                DTensor lab = labels(rows);
                const int* ld = reinterpret_cast<const int*>(lab.p);
                std::vector<BlockCacheDev> caches;
                BlockCacheDev cc;
                DTensor logits = remainder(so, &caches, &cc);
                DTensor probs;
                const double ce = X_.softmax_ce(logits, ld, &probs);
                DTensor glog = X_.alloc(logits.n, logits.c, 1, 1, true);
                X_.softmax_ce_bwd(probs, ld, 1.0f, glog);
                // remainder_backward (distill.cpp:74-84): no parameter gradients
                DTensor g = X_.backward(teacher.cls, cc, glog, true, false);
                for (size_t bi = teacher.blocks.size(); bi-- > static_cast<size_t>(k);)
                    g = X_.backward(teacher.blocks[bi], caches[bi - k], g, true, false);
                X_.axpy(gs, g);
                obj = static_cast<double>(t.lambda_local) * local + ce;
            }
            res.step_losses.push_back(static_cast<float>(obj));
            if (!std::isfinite(obj)) {  // distill.cpp:236-244: reported, not thrown
                std::ostringstream msg;
                msg << "block " << k << " diverged at epoch " << epoch << " batch " << done << " (loss " << obj << ")";
                res.failed = true;
                res.failure = msg.str();
                res.final_block = block_to_host(X_, student);
                res.wall_time_s = elapsed();
                return res;
            }
            X_.zero_grads(student);
            X_.backward(student, cache, gs, false, true);
            X_.sgd(student, t.lr, t.momentum);
            obj_sum += obj;
            local_sum += local;
            ++done;
            ++steps;
        }
        if (done == 0) break;  // the cap landed on an epoch boundary
        res.loss_history.push_back(obj_sum / done);
        res.final_local_loss = local_sum / done;
        if (with_eval && epoch % t.eval_every == 0) record_eval(epoch);
    }
    res.final_block = block_to_host(X_, student);
    res.wall_time_s = elapsed();
    return res;
}

}  // namespace pbkd_gpu
