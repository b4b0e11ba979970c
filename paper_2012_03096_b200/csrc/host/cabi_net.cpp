// cabi_net.cpp -- extern "C" block- and network-level entry points
// (include/pbkd_b200.h, "block / network level") over the layer-by-layer
// executor (csrc/netexec.cu) and trainer (csrc/nettrain.cu).
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "pbkd_b200.h"
#include "ctx.hpp"
#include "../common.cuh"
#include "../engine.hpp"
#include "../netexec.hpp"
#include "../nettrain.hpp"
#include "pbkd/model.hpp"
#include "pbkd/replacement.hpp"
#include "pbkd/weights_io.hpp"

using namespace pbkd_gpu;
using pbkd::LayerKind;



struct pbkd_block_cache {
    BlockCacheDev c;
    int n = 0, ch = 0, h = 0, w = 0;  // the block input's shape
    size_t n_layers = 0;
};

namespace {

// same error mapping as cabi.cpp (thread-local message + kind)
int fail(const std::exception& e, int kind);

template <class F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const pbkd::ShapeError& e) {
        return fail(e, PBKD_ERR_SHAPE);
    } catch (const pbkd_gpu::CudaError& e) {
        return fail(e, PBKD_ERR_CUDA);
    } catch (const std::out_of_range& e) {
        return fail(e, PBKD_ERR_RANGE);
    } catch (const std::invalid_argument& e) {
        return fail(e, PBKD_ERR_SPEC);
    } catch (const std::logic_error& e) {
        return fail(e, PBKD_ERR_LOGIC);
    } catch (const std::exception& e) {
        return fail(e, PBKD_ERR_OTHER);
    }
}

pbkd::LayerParams layer_of(const pbkd_layer_desc& d) {
    if (d.kind < 0 || d.kind > static_cast<int>(LayerKind::MaxPool3x3)) throw pbkd::SpecError("layer kind out of range");
    const auto kind = static_cast<LayerKind>(d.kind);
    switch (kind) {
        case LayerKind::Conv3x3:
        case LayerKind::Conv1x1:
        case LayerKind::Conv7x7:
            return pbkd::make_conv_layer(kind, d.in_channels, d.out_channels, d.kernel, d.stride, d.padding);
        case LayerKind::MaxPool3x3: return pbkd::make_maxpool_layer(d.in_channels);
        case LayerKind::DepthwiseConv3x3:
            return pbkd::make_conv_layer(kind, d.in_channels, d.in_channels, 3, d.stride, d.padding);
        case LayerKind::PointwiseConv:
            return pbkd::make_conv_layer(kind, d.in_channels, d.out_channels, 1, d.stride, 0);
        case LayerKind::BatchNorm: return pbkd::make_batchnorm_layer(d.in_channels);
        case LayerKind::ReLU: return pbkd::make_relu_layer(d.in_channels);
        case LayerKind::GlobalAvgPool: return pbkd::make_gap_layer(d.in_channels);
        case LayerKind::Dense: {
            pbkd::LayerParams l = pbkd::make_dense_layer(d.in_channels, d.out_channels);
            if (!d.has_bias) l.bias = pbkd::Tensor();
            return l;
        }
        case LayerKind::Add: {
            pbkd::LayerParams l = pbkd::make_add_layer(d.in_channels, d.out_channels, d.stride);
            if (static_cast<bool>(d.has_weight) != !l.weight.data.empty())
                throw pbkd::SpecError("add layer: projection flag does not match its shape");
            return l;
        }
    }
    throw pbkd::SpecError("layer kind out of range");
}

pbkd::Block block_of(const pbkd_layer_desc* L, int n, const char* spec_kind = "") {
    if (n < 0 || (n > 0 && !L)) throw pbkd::SpecError("block layer list is null");
    pbkd::Block b;
    b.spec_kind = spec_kind ? spec_kind : "";
    for (int i = 0; i < n; ++i) b.layers.push_back(layer_of(L[i]));
    if (n > 0) {
        b.in_channels = L[0].in_channels;
        b.out_channels = L[n - 1].out_channels;
        b.stride = L[0].stride;
    }
    return b;
}

size_t floats_of(pbkd::Block& b) {
    size_t k = 0;
    pbkd::for_each_block_array(b, [&](const std::string&, pbkd::Tensor& t) { k += t.data.size(); });
    return k;
}

pbkd::Network net_of(const pbkd_net_desc* d) {
    if (!d || d->n_blocks < 0 || !d->layer_counts) throw pbkd::SpecError("null network description");
    pbkd::Network net;
    net.name = "network";
    net.in_c = d->in_c, net.in_h = d->in_h, net.in_w = d->in_w;
    const pbkd_layer_desc* L = d->layers;
    for (int i = 0; i <= d->n_blocks; ++i) {
        pbkd::Block b = block_of(L, d->layer_counts[i], d->spec_kinds ? d->spec_kinds[i] : "");
        L += d->layer_counts[i];
        if (i < d->n_blocks) {
            b.name = "block" + std::to_string(i + 1);
            net.blocks.push_back(std::move(b));
        } else {
            b.name = "classifier";
            net.classifier = std::move(b);
        }
    }
    return net;
}

size_t net_floats(pbkd::Network& net) {
    size_t k = 0;
    pbkd::for_each_array(net, [&](const std::string&, pbkd::Tensor& t) { k += t.data.size(); });
    return k;
}

Engine& engine(pbkd_ctx* ctx) {
    if (!ctx || !ctx->eng) throw std::invalid_argument("null context");
    return *ctx->eng;
}

}  // namespace

// error state lives in cabi.cpp (pbkd_last_error)
extern "C" void pbkd_internal_set_error(const char* msg, int kind);

namespace {
int fail(const std::exception& e, int kind) {
    pbkd_internal_set_error(e.what(), kind);
    return 1;
}
}  // namespace

extern "C" {

int pbkd_block_forward(pbkd_ctx* ctx, const pbkd_layer_desc* layers, int n_layers, float* arrays, size_t n_arrays,
                       const float* x, int n, int c, int h, int w, int train, float* y, size_t y_cap, int* y_shape,
                       pbkd_block_cache** cache) {
    return guard([&] {
        pbkd::Block b = block_of(layers, n_layers);
        if (floats_of(b) != n_arrays) throw pbkd::ShapeError("block arrays: size does not match the layer list");
        if (n_layers > 0 && c != layers[0].in_channels)
            throw pbkd::ShapeError("block input has " + std::to_string(c) + " channels, the block expects " +
                                   std::to_string(layers[0].in_channels));
        NetExec& X = engine(ctx).exec();
        DevBlock d = X.make_block(b, arrays, false);
        std::unique_ptr<pbkd_block_cache> pc;
        if (cache) pc = std::make_unique<pbkd_block_cache>();
        DTensor out = X.forward(d, X.upload_nchw(x, n, c, h, w), train != 0, pc ? &pc->c : nullptr);
        if (static_cast<size_t>(out.size()) > y_cap) throw pbkd::ShapeError("block output buffer too small");
        X.download_nchw(out, y);
        if (y_shape) y_shape[0] = out.n, y_shape[1] = out.c, y_shape[2] = out.h, y_shape[3] = out.w;
        if (train) X.arrays_to_host(d, arrays);  // moving statistics (ops.hpp:297-298)
        if (pc) {
            pc->n = n, pc->ch = c, pc->h = h, pc->w = w;
            pc->n_layers = static_cast<size_t>(n_layers);
            *cache = pc.release();
        }
    });
}

int pbkd_block_backward(pbkd_ctx* ctx, const pbkd_layer_desc* layers, int n_layers, const float* arrays,
                        size_t n_arrays, const pbkd_block_cache* cache, const float* gy, int n, int c, int h, int w,
                        int need_input_grad, int param_grads, float* grads, float* gx, size_t gx_cap) {
    return guard([&] {
        if (!cache) throw std::logic_error("block_backward: no cache");
        if (cache->n_layers != static_cast<size_t>(n_layers))
            throw std::logic_error("block_backward: cache does not match block");
        pbkd::Block b = block_of(layers, n_layers);
        if (floats_of(b) != n_arrays) throw pbkd::ShapeError("block arrays: size does not match the layer list");
        NetExec& X = engine(ctx).exec();
        DevBlock d = X.make_block(b, arrays, false);
        DTensor g = X.backward(d, cache->c, X.upload_nchw(gy, n, c, h, w), need_input_grad != 0, param_grads != 0);
        if (param_grads && grads && n_arrays) {
            std::vector<float> acc(n_arrays);
            X.grads_to_host(d, acc.data());
            for (size_t i = 0; i < n_arrays; ++i) grads[i] += acc[i];
        }
        if (need_input_grad && gx) {
            if (static_cast<size_t>(g.size()) > gx_cap) throw pbkd::ShapeError("input-gradient buffer too small");
            X.download_nchw(g, gx);
        }
    });
}

void pbkd_block_cache_free(pbkd_block_cache* cache) { delete cache; }

int pbkd_mse_local_loss(pbkd_ctx* ctx, const float* s, const float* t, size_t count, float* loss) {
    return guard([&] {
        NetExec& X = engine(ctx).exec();
        const int k = static_cast<int>(count);
        *loss = X.mse(X.upload_nchw(s, 1, 1, 1, k), X.upload_nchw(t, 1, 1, 1, k));
    });
}

int pbkd_mse_local_loss_bwd(pbkd_ctx* ctx, const float* s, const float* t, size_t count, float scale, float* g) {
    return guard([&] {
        NetExec& X = engine(ctx).exec();
        const int k = static_cast<int>(count);
        DTensor gd = X.upload_nchw(g, 1, 1, 1, k);
        X.mse_bwd(X.upload_nchw(s, 1, 1, 1, k), X.upload_nchw(t, 1, 1, 1, k), scale, gd);
        X.download_nchw(gd, g);
    });
}

int pbkd_softmax_ce(pbkd_ctx* ctx, const float* logits, int n, int k, const int* labels, float* loss,
                    float* probs) {
    return guard([&] {
        for (int i = 0; i < n; ++i)
            if (labels[i] < 0 || labels[i] >= k)
                throw std::invalid_argument("softmax_cross_entropy: label " + std::to_string(labels[i]) +
                                            " out of range [0," + std::to_string(k) + ")");
        NetExec& X = engine(ctx).exec();
        DTensor lab = X.upload_ints(std::vector<int>(labels, labels + n));
        DTensor p;
        *loss = static_cast<float>(X.softmax_ce(X.upload_nchw(logits, n, k, 1, 1), reinterpret_cast<const int*>(lab.p),
                                                probs ? &p : nullptr));
        if (probs) X.download_nchw(p, probs);
    });
}

int pbkd_softmax_ce_bwd(pbkd_ctx* ctx, const float* probs, int n, int k, const int* labels, float scale, float* g) {
    return guard([&] {
        NetExec& X = engine(ctx).exec();
        DTensor lab = X.upload_ints(std::vector<int>(labels, labels + n));
        DTensor gd = X.upload_nchw(g, n, k, 1, 1);
        X.softmax_ce_bwd(X.upload_nchw(probs, n, k, 1, 1), reinterpret_cast<const int*>(lab.p), scale, gd);
        X.download_nchw(gd, g);
    });
}

int pbkd_evaluate_network(pbkd_ctx* ctx, const pbkd_net_desc* nd, const float* arrays, size_t n_arrays,
                          const int* idx, int n_idx, int batch_size, double* acc) {
    return guard([&] {
        pbkd::Network net = net_of(nd);
        if (net_floats(net) != n_arrays) throw pbkd::ShapeError("network arrays: size does not match the layers");
        Engine& e = engine(ctx);
        NetTrainer tr = e.trainer();
        DevNet dn = make_devnet(e.exec(), net, arrays, false);
        *acc = tr.evaluate(dn, std::vector<int>(idx, idx + std::max(0, n_idx)), batch_size);
    });
}

int pbkd_fit_network(pbkd_ctx* ctx, const pbkd_net_desc* nd, float* arrays, size_t n_arrays, const int* train_idx,
                     int n_train, const int* eval_idx, int n_eval_idx, int epochs, int freeze_non_replaced, float lr,
                     float momentum, int batch_size, uint64_t seed, int teacher_mode, double* initial_eval,
                     double* final_eval, double* loss_hist, int* eval_epochs, double* eval_acc, int* n_eval) {
    return guard([&] {
        pbkd::Network net = net_of(nd);
        if (net_floats(net) != n_arrays) throw pbkd::ShapeError("network arrays: size does not match the layers");
        Engine& e = engine(ctx);
        NetTrainer tr = e.trainer();
        DevNet dn = make_devnet(e.exec(), net, arrays, false);
        FitResult r = tr.fit(dn, std::vector<int>(train_idx, train_idx + std::max(0, n_train)),
                             std::vector<int>(eval_idx, eval_idx + std::max(0, n_eval_idx)), epochs,
                             !teacher_mode && freeze_non_replaced, lr, momentum, batch_size, seed, teacher_mode != 0);
        devnet_to_host(e.exec(), dn, arrays);
        if (initial_eval) *initial_eval = r.initial_eval;
        if (final_eval) *final_eval = r.final_eval;
        for (size_t i = 0; loss_hist && i < r.loss_history.size(); ++i) loss_hist[i] = r.loss_history[i];
        for (size_t i = 0; i < r.eval_history.size(); ++i) {
            if (eval_epochs) eval_epochs[i] = r.eval_history[i].epoch;
            if (eval_acc) eval_acc[i] = r.eval_history[i].accuracy;
        }
        if (n_eval) *n_eval = static_cast<int>(r.eval_history.size());
    });
}

int pbkd_fit_assembled(pbkd_ctx* ctx, const char* spec, const float* tw, size_t n_teacher, const int* blocks,
                       const int* kinds, const float* cand_w, int n_rep, const int* train_idx, int n_train,
                       const int* eval_idx, int n_eval_idx, int epochs, int freeze, float lr, float momentum,
                       int batch_size, uint64_t seed, int teacher_mode, double* initial_eval, double* final_eval,
                       double* loss_hist, int* eval_epochs, double* eval_acc, int* n_eval, float* net_out, size_t cap,
                       size_t* n_out) {
    return guard([&] {
        if (!spec) throw std::invalid_argument("null model spec");
        pbkd::Network net = pbkd::parse_model_spec(spec, "spec");
        if (net_floats(net) != n_teacher) throw pbkd::ShapeError("teacher weights: size does not match the spec");
        const float* w = tw;
        pbkd::for_each_array(net, [&](const std::string&, pbkd::Tensor& t) {
            std::copy(w, w + t.data.size(), t.data.begin());
            w += t.data.size();
        });
        const float* cw = cand_w;
        for (int i = 0; i < n_rep; ++i) {  // reassemble (distill.cpp:313-318)
            if (blocks[i] < 1 || blocks[i] > static_cast<int>(net.blocks.size()))
                throw pbkd::SpecError("result references block " + std::to_string(blocks[i]));
            pbkd::Block& tb = net.blocks[static_cast<size_t>(blocks[i]) - 1];
            pbkd::Block nb = pbkd::build_candidate(static_cast<pbkd::CandidateKind>(kinds[i]), tb.in_channels,
                                                   tb.out_channels, tb.stride, 0)
                                 .block;
            pbkd::for_each_block_array(nb, [&](const std::string&, pbkd::Tensor& t) {
                std::copy(cw, cw + t.data.size(), t.data.begin());
                cw += t.data.size();
            });
            nb.name = tb.name;
            nb.replaceable = false;
            tb = std::move(nb);
        }
        const size_t total = net_floats(net);
        if (total > cap) throw pbkd::ShapeError("network output buffer too small");
        std::vector<float> flat;
        pbkd::for_each_array(net, [&](const std::string&, pbkd::Tensor& t) {
            flat.insert(flat.end(), t.data.begin(), t.data.end());
        });
        Engine& e = engine(ctx);
        NetTrainer tr = e.trainer();
        DevNet dn = make_devnet(e.exec(), net, flat.data(), false);
        FitResult r = tr.fit(dn, std::vector<int>(train_idx, train_idx + std::max(0, n_train)),
                             std::vector<int>(eval_idx, eval_idx + std::max(0, n_eval_idx)), epochs,
                             !teacher_mode && freeze, lr, momentum, batch_size, seed, teacher_mode != 0);
        devnet_to_host(e.exec(), dn, net_out);
        *n_out = total;
        if (initial_eval) *initial_eval = r.initial_eval;
        if (final_eval) *final_eval = r.final_eval;
        for (size_t i = 0; loss_hist && i < r.loss_history.size(); ++i) loss_hist[i] = r.loss_history[i];
        for (size_t i = 0; i < r.eval_history.size(); ++i) {
            if (eval_epochs) eval_epochs[i] = r.eval_history[i].epoch;
            if (eval_acc) eval_acc[i] = r.eval_history[i].accuracy;
        }
        if (n_eval) *n_eval = static_cast<int>(r.eval_history.size());
    });
}

}  // extern "C"
