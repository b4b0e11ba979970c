// pbkd_oracle.cpp -- TEST INFRASTRUCTURE ONLY (the CPU oracle / checker).
//
// A from-scratch CPU restatement of the reference "pbkd" distillation path
// (/root/reference/proj).  It is the checker the GPU product is compared
// against; it is never linked into, loaded by, or called from the product.
// Parity of this restatement is PINNED two ways (tests/test_oracle.py):
//   * bitwise against the reference library itself, compiled from its own
//     sources into oracle/_ref/libpbkd_ref.so (oracle/Makefile), and
//   * against the golden vectors committed in tests/golden/ (generated from
//     the reference build by tests/golden/make_golden.py) and the reference
//     tests' known-answer values.
//
// Arithmetic discipline: every loop below runs in the same order as the
// reference (cited file:line) with float accumulators and no contraction
// (-ffp-contract=off, matching the reference's FMA-free -O3 build), so results
// agree bit for bit.  Randomness uses the same libstdc++ engines/distributions.
#include "oracle_api.h"

#include <algorithm>
#include <array>
#include <atomic>
#include <thread>
#include <cmath>
#include <cstring>
#include <functional>
#include <numbers>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include <json.hpp>

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

// ---------------------------------------------------------------------------
// Tensor (tensor.hpp:18-62): NCHW float, zero-filled on construction.
// ---------------------------------------------------------------------------
struct T4 {
    int n = 0, c = 0, h = 0, w = 0;
    std::vector<float> d;
    T4() = default;
    T4(int n_, int c_, int h_, int w_) : n(n_), c(c_), h(h_), w(w_) {
        if (n <= 0 || c <= 0 || h <= 0 || w <= 0) throw std::invalid_argument("T4: bad dims");
        d.assign(static_cast<size_t>(n) * c * h * w, 0.0f);
    }
    size_t at(int i, int j, int y, int x) const {
        return ((static_cast<size_t>(i) * c + j) * h + y) * w + x;
    }
    size_t plane() const { return static_cast<size_t>(h) * w; }
};

uint64_t splitmix(uint64_t a, uint64_t b) {  // tensor.hpp:94-99
    uint64_t z = a + 0x9e3779b97f4a7c15ull * (b + 1);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
}

int out_dim(int in, int k, int s, int p) {  // ops.hpp:23-31
    const int span = in + 2 * p - k;
    if (span < 0) throw std::invalid_argument("conv: kernel larger than padded input");
    const int o = span / s + 1;
    if (o < 1) throw std::invalid_argument("conv: output dim < 1");
    return o;
}

// ---------------------------------------------------------------------------
// Kernels (ops.hpp).  Backward functions accumulate into caller buffers.
// ---------------------------------------------------------------------------

// ops.hpp:37-75 -- acc over (j, ky, kx), out-of-bounds taps skipped.
T4 conv_fwd(const T4& x, const T4& k, int s, int p) {
    const int ho = out_dim(x.h, k.h, s, p), wo = out_dim(x.w, k.w, s, p);
    T4 y(x.n, k.n, ho, wo);
    for (int n = 0; n < x.n; ++n)
        for (int o = 0; o < k.n; ++o)
            for (int oy = 0; oy < ho; ++oy)
                for (int ox = 0; ox < wo; ++ox) {
                    float acc = 0.0f;
                    for (int j = 0; j < x.c; ++j)
                        for (int ky = 0; ky < k.h; ++ky) {
                            const int iy = oy * s - p + ky;
                            if (iy < 0 || iy >= x.h) continue;
                            for (int kx = 0; kx < k.w; ++kx) {
                                const int ix = ox * s - p + kx;
                                if (ix < 0 || ix >= x.w) continue;
                                acc += x.d[x.at(n, j, iy, ix)] * k.d[k.at(o, j, ky, kx)];
                            }
                        }
                    y.d[y.at(n, o, oy, ox)] = acc;
                }
    return y;
}

// ops.hpp:77-108
void conv_bwd(const T4& x, const T4& k, const T4& gy, int s, int p, float* gx, float* gk) {
    for (int n = 0; n < x.n; ++n)
        for (int o = 0; o < k.n; ++o)
            for (int oy = 0; oy < gy.h; ++oy)
                for (int ox = 0; ox < gy.w; ++ox) {
                    const float g = gy.d[gy.at(n, o, oy, ox)];
                    if (g == 0.0f) continue;
                    for (int j = 0; j < x.c; ++j)
                        for (int ky = 0; ky < k.h; ++ky) {
                            const int iy = oy * s - p + ky;
                            if (iy < 0 || iy >= x.h) continue;
                            for (int kx = 0; kx < k.w; ++kx) {
                                const int ix = ox * s - p + kx;
                                if (ix < 0 || ix >= x.w) continue;
                                if (gk) gk[k.at(o, j, ky, kx)] += g * x.d[x.at(n, j, iy, ix)];
                                if (gx) gx[x.at(n, j, iy, ix)] += g * k.d[k.at(o, j, ky, kx)];
                            }
                        }
                }
}

// ops.hpp:114-147 -- per output a serial 9-term sum in (ky, kx) order.
T4 dw_fwd(const T4& x, const T4& k, int s, int p) {
    const int ho = out_dim(x.h, k.h, s, p), wo = out_dim(x.w, k.w, s, p);
    T4 y(x.n, x.c, ho, wo);
    for (int n = 0; n < x.n; ++n)
        for (int j = 0; j < x.c; ++j)
            for (int oy = 0; oy < ho; ++oy)
                for (int ox = 0; ox < wo; ++ox) {
                    float acc = 0.0f;
                    for (int ky = 0; ky < k.h; ++ky) {
                        const int iy = oy * s - p + ky;
                        if (iy < 0 || iy >= x.h) continue;
                        for (int kx = 0; kx < k.w; ++kx) {
                            const int ix = ox * s - p + kx;
                            if (ix < 0 || ix >= x.w) continue;
                            acc += x.d[x.at(n, j, iy, ix)] * k.d[k.at(j, 0, ky, kx)];
                        }
                    }
                    y.d[y.at(n, j, oy, ox)] = acc;
                }
    return y;
}

// ops.hpp:149-178
void dw_bwd(const T4& x, const T4& k, const T4& gy, int s, int p, float* gx, float* gk) {
    for (int n = 0; n < x.n; ++n)
        for (int j = 0; j < x.c; ++j)
            for (int oy = 0; oy < gy.h; ++oy)
                for (int ox = 0; ox < gy.w; ++ox) {
                    const float g = gy.d[gy.at(n, j, oy, ox)];
                    if (g == 0.0f) continue;
                    for (int ky = 0; ky < k.h; ++ky) {
                        const int iy = oy * s - p + ky;
                        if (iy < 0 || iy >= x.h) continue;
                        for (int kx = 0; kx < k.w; ++kx) {
                            const int ix = ox * s - p + kx;
                            if (ix < 0 || ix >= x.w) continue;
                            if (gk) gk[k.at(j, 0, ky, kx)] += g * x.d[x.at(n, j, iy, ix)];
                            if (gx) gx[x.at(n, j, iy, ix)] += g * k.d[k.at(j, 0, ky, kx)];
                        }
                    }
                }
}

// ops.hpp:184-209 -- y[n,o,:] accumulates w[o,j]*x[n,j,:] for ascending j.
T4 pw_fwd(const T4& x, const T4& k, int s) {
    const int ho = out_dim(x.h, 1, s, 0), wo = out_dim(x.w, 1, s, 0);
    T4 y(x.n, k.n, ho, wo);
    for (int n = 0; n < x.n; ++n)
        for (int o = 0; o < k.n; ++o) {
            float* yr = &y.d[y.at(n, o, 0, 0)];
            for (int j = 0; j < x.c; ++j) {
                const float wt = k.d[k.at(o, j, 0, 0)];
                const float* xr = &x.d[x.at(n, j, 0, 0)];
                size_t q = 0;
                for (int oy = 0; oy < ho; ++oy)
                    for (int ox = 0; ox < wo; ++ox)
                        yr[q++] += wt * xr[static_cast<size_t>(oy * s) * x.w + ox * s];
            }
        }
    return y;
}

// ops.hpp:211-239
void pw_bwd(const T4& x, const T4& k, const T4& gy, int s, float* gx, float* gk) {
    for (int n = 0; n < x.n; ++n)
        for (int o = 0; o < k.n; ++o) {
            const float* gr = &gy.d[gy.at(n, o, 0, 0)];
            for (int j = 0; j < x.c; ++j) {
                const float wt = k.d[k.at(o, j, 0, 0)];
                const float* xr = &x.d[x.at(n, j, 0, 0)];
                float* gxr = gx ? gx + x.at(n, j, 0, 0) : nullptr;
                float kacc = 0.0f;
                size_t q = 0;
                for (int oy = 0; oy < gy.h; ++oy)
                    for (int ox = 0; ox < gy.w; ++ox) {
                        const float g = gr[q++];
                        const size_t in = static_cast<size_t>(oy * s) * x.w + ox * s;
                        kacc += g * xr[in];
                        if (gxr) gxr[in] += g * wt;
                    }
                if (gk) gk[k.at(o, j, 0, 0)] += kacc;
            }
        }
}

constexpr double kEps = 1e-5;        // ops.hpp:245
constexpr float kBnMomentum = 0.9f;  // model.cpp:15

struct BnCache {
    T4 xhat;
    std::vector<float> inv_std;
};

// ops.hpp:261-301 -- float sum / sum-of-squares per channel, (n, pixel) order.
T4 bn_train_fwd(const T4& x, const float* gamma, const float* beta, float* mm, float* mv,
                float mom, BnCache* cache) {
    const size_t m = static_cast<size_t>(x.n) * x.h * x.w;
    T4 y(x.n, x.c, x.h, x.w);
    if (cache) {
        cache->xhat = T4(x.n, x.c, x.h, x.w);
        cache->inv_std.assign(x.c, 0.0f);
    }
    const size_t pl = x.plane();
    for (int j = 0; j < x.c; ++j) {
        float sum = 0.0f, sq = 0.0f;
        for (int n = 0; n < x.n; ++n) {
            const float* p = &x.d[x.at(n, j, 0, 0)];
            for (size_t i = 0; i < pl; ++i) {
                sum += p[i];
                sq += p[i] * p[i];
            }
        }
        const float mean = sum / static_cast<float>(m);
        float var = sq / static_cast<float>(m) - mean * mean;
        if (var < 0.0f) var = 0.0f;
        const float inv = 1.0f / std::sqrt(var + static_cast<float>(kEps));
        for (int n = 0; n < x.n; ++n) {
            const float* p = &x.d[x.at(n, j, 0, 0)];
            float* q = &y.d[y.at(n, j, 0, 0)];
            float* xh = cache ? &cache->xhat.d[cache->xhat.at(n, j, 0, 0)] : nullptr;
            for (size_t i = 0; i < pl; ++i) {
                const float nv = (p[i] - mean) * inv;
                if (xh) xh[i] = nv;
                q[i] = gamma[j] * nv + beta[j];
            }
        }
        if (cache) cache->inv_std[j] = inv;
        mm[j] = mom * mm[j] + (1.0f - mom) * mean;
        mv[j] = mom * mv[j] + (1.0f - mom) * var;
    }
    return y;
}

// ops.hpp:304-321
T4 bn_infer(const T4& x, const float* gamma, const float* beta, const float* mm, const float* mv) {
    T4 y(x.n, x.c, x.h, x.w);
    const size_t pl = x.plane();
    for (int j = 0; j < x.c; ++j) {
        const float inv = 1.0f / std::sqrt(mv[j] + static_cast<float>(kEps));
        const float scale = gamma[j] * inv;
        const float shift = beta[j] - mm[j] * scale;
        for (int n = 0; n < x.n; ++n) {
            const float* p = &x.d[x.at(n, j, 0, 0)];
            float* q = &y.d[y.at(n, j, 0, 0)];
            for (size_t i = 0; i < pl; ++i) q[i] = scale * p[i] + shift;
        }
    }
    return y;
}

// ops.hpp:325-357
void bn_train_bwd(const BnCache& cache, const float* gamma, const T4& gy, float* gx, float* ggamma,
                  float* gbeta) {
    const T4& xh = cache.xhat;
    const size_t m = static_cast<size_t>(xh.n) * xh.h * xh.w;
    const size_t pl = xh.plane();
    for (int j = 0; j < xh.c; ++j) {
        float sg = 0.0f, sgx = 0.0f;
        for (int n = 0; n < xh.n; ++n) {
            const float* g = &gy.d[gy.at(n, j, 0, 0)];
            const float* x = &xh.d[xh.at(n, j, 0, 0)];
            for (size_t i = 0; i < pl; ++i) {
                sg += g[i];
                sgx += g[i] * x[i];
            }
        }
        if (ggamma) ggamma[j] += sgx;
        if (gbeta) gbeta[j] += sg;
        if (gx) {
            const float inv_m = 1.0f / static_cast<float>(m);
            const float kk = gamma[j] * cache.inv_std[j];
            for (int n = 0; n < xh.n; ++n) {
                const float* g = &gy.d[gy.at(n, j, 0, 0)];
                const float* x = &xh.d[xh.at(n, j, 0, 0)];
                float* q = gx + xh.at(n, j, 0, 0);
                for (size_t i = 0; i < pl; ++i) q[i] += kk * (g[i] - inv_m * sg - x[i] * inv_m * sgx);
            }
        }
    }
}

T4 relu_fwd(const T4& x) {  // ops.hpp:380-385
    T4 y(x.n, x.c, x.h, x.w);
    for (size_t i = 0; i < x.d.size(); ++i) y.d[i] = x.d[i] > 0.0f ? x.d[i] : 0.0f;
    return y;
}

void relu_bwd(const T4& x, const T4& gy, float* gx) {  // ops.hpp:387-393
    if (!gx) return;
    for (size_t i = 0; i < x.d.size(); ++i)
        if (x.d[i] > 0.0f) gx[i] += gy.d[i];
}

T4 gap_fwd(const T4& x) {  // ops.hpp:395-407
    T4 y(x.n, x.c, 1, 1);
    const size_t pl = x.plane();
    for (int n = 0; n < x.n; ++n)
        for (int j = 0; j < x.c; ++j) {
            const float* p = &x.d[x.at(n, j, 0, 0)];
            float sum = 0.0f;
            for (size_t i = 0; i < pl; ++i) sum += p[i];
            y.d[y.at(n, j, 0, 0)] = sum / static_cast<float>(pl);
        }
    return y;
}

T4 dense_fwd(const T4& x, const T4& k, const T4& b) {  // ops.hpp:425-442
    T4 y(x.n, k.n, 1, 1);
    for (int n = 0; n < x.n; ++n)
        for (int o = 0; o < k.n; ++o) {
            float acc = b.d.empty() ? 0.0f : b.d[o];
            for (int j = 0; j < x.c; ++j) acc += k.d[k.at(o, j, 0, 0)] * x.d[x.at(n, j, 0, 0)];
            y.d[y.at(n, o, 0, 0)] = acc;
        }
    return y;
}

T4 add_fwd(const T4& a, const T4& b) {  // ops.hpp:460-466
    T4 y(a.n, a.c, a.h, a.w);
    for (size_t i = 0; i < a.d.size(); ++i) y.d[i] = a.d[i] + b.d[i];
    return y;
}

float mse(const float* s, const float* t, size_t count) {  // ops.hpp:518-527
    float total = 0.0f;
    for (size_t i = 0; i < count; ++i) {
        const float d = s[i] - t[i];
        total += d * d;
    }
    return total / static_cast<float>(count);
}

void mse_bwd(const float* s, const float* t, size_t count, float scale, float* g) {  // :531-539
    const float k = scale * 2.0f / static_cast<float>(count);
    for (size_t i = 0; i < count; ++i) g[i] += k * (s[i] - t[i]);
}

void sgd(float* w, const float* g, float* v, size_t n, float lr, float mom) {  // ops.hpp:545-558
    if (!(lr > 0.0f)) throw std::invalid_argument("sgd_step: lr must be > 0");
    if (mom < 0.0f || mom >= 1.0f) throw std::invalid_argument("sgd_step: momentum must be in [0,1)");
    for (size_t i = 0; i < n; ++i) {
        v[i] = mom * v[i] + g[i];
        w[i] -= lr * v[i];
    }
}

// ---------------------------------------------------------------------------
// Model graph (model.hpp:40-72, model.cpp)
// ---------------------------------------------------------------------------
enum Kind { Conv3, Conv1, DW, PW, BN, RELU, GAP, DENSE, ADD };

struct Layer {
    Kind kind;
    int cin = 0, cout = 0, k = 0, stride = 1, pad = 0;
    T4 weight, bias, gamma, beta, mm, mv;
    T4 wgrad, bgrad, ggrad, btgrad;  // gradient buffers of trainable tensors
};

struct Block {
    std::string name, spec_kind;
    bool replaceable = false;
    int cin = 0, cout = 0, stride = 1, pad = 1;
    std::vector<Layer> layers;
};

struct Net {
    int in_c = 0, in_h = 0, in_w = 0;
    std::vector<Block> blocks;
    Block cls;
};

Layer conv_layer(Kind kind, int cin, int cout, int k, int s, int p) {  // model.cpp:157-171
    Layer l;
    l.kind = kind;
    l.cin = cin;
    l.cout = kind == DW ? cin : cout;
    l.k = k;
    l.stride = s;
    l.pad = p;
    l.weight = kind == DW ? T4(cin, 1, k, k) : T4(l.cout, cin, k, k);
    return l;
}

Layer bn_layer(int c) {  // model.cpp:173-184
    Layer l;
    l.kind = BN;
    l.cin = l.cout = c;
    l.gamma = T4(1, c, 1, 1);
    l.beta = T4(1, c, 1, 1);
    l.mm = T4(1, c, 1, 1);
    l.mv = T4(1, c, 1, 1);
    std::fill(l.gamma.d.begin(), l.gamma.d.end(), 1.0f);
    std::fill(l.mv.d.begin(), l.mv.d.end(), 1.0f);
    return l;
}

Layer plain_layer(Kind kind, int c) {
    Layer l;
    l.kind = kind;
    l.cin = l.cout = c;
    return l;
}

Layer add_layer(int cin, int cout, int s) {  // model.cpp:211-219
    Layer l;
    l.kind = ADD;
    l.cin = cin;
    l.cout = cout;
    l.stride = s;
    if (cin != cout || s != 1) l.weight = T4(cout, cin, 1, 1);
    return l;
}

// (c, h, w) after the layer (model.cpp:30-73)
void layer_shape(const Layer& l, int& c, int& h, int& w) {
    switch (l.kind) {
        case Conv3:
        case Conv1:
        case DW:
            h = out_dim(h, l.k, l.stride, l.pad);
            w = out_dim(w, l.k, l.stride, l.pad);
            c = l.cout;
            break;
        case PW:
            h = out_dim(h, 1, l.stride, 0);
            w = out_dim(w, 1, l.stride, 0);
            c = l.cout;
            break;
        case GAP:
            h = w = 1;
            break;
        case DENSE:
            c = l.cout;
            break;
        default:
            break;
    }
}

Net parse_spec(const char* text) {  // model.cpp:225-344 (well-formed specs)
    using nlohmann::json;
    const json doc = json::parse(text);
    Net net;
    net.in_c = doc.at("input_shape")[0].get<int>();
    net.in_h = doc.at("input_shape")[1].get<int>();
    net.in_w = doc.at("input_shape")[2].get<int>();
    int c = net.in_c, h = net.in_h, w = net.in_w;
    const json& blocks = doc.at("blocks");
    for (size_t i = 0; i < blocks.size(); ++i) {
        const json& e = blocks[i];
        const std::string kind = e.at("kind").get<std::string>();
        const int out_c = e.at("out_channels").get<int>();
        const int s = e.value("stride", 1);
        const int p = e.value("padding", kind == "conv1x1" ? 0 : 1);
        Block b;
        b.name = e.value("name", "block" + std::to_string(i + 1));
        b.spec_kind = kind;
        b.cin = c;
        b.cout = out_c;
        b.stride = s;
        b.pad = p;
        if (kind == "conv3x3" || kind == "conv1x1") {  // model.cpp:83-98
            const bool k3 = kind == "conv3x3";
            b.replaceable = k3;
            b.layers.push_back(conv_layer(k3 ? Conv3 : Conv1, c, out_c, k3 ? 3 : 1, s, p));
            b.layers.push_back(bn_layer(out_c));
            b.layers.push_back(plain_layer(RELU, out_c));
        } else if (kind == "residual3x3") {  // model.cpp:102-119
            b.replaceable = true;
            b.layers.push_back(conv_layer(Conv3, c, out_c, 3, s, p));
            b.layers.push_back(bn_layer(out_c));
            b.layers.push_back(plain_layer(RELU, out_c));
            b.layers.push_back(conv_layer(Conv3, out_c, out_c, 3, 1, 1));
            b.layers.push_back(bn_layer(out_c));
            b.layers.push_back(add_layer(c, out_c, s));
            b.layers.push_back(plain_layer(RELU, out_c));
        } else {
            throw std::invalid_argument("unknown block kind '" + kind + "'");
        }
        for (const Layer& l : b.layers) layer_shape(l, c, h, w);
        net.blocks.push_back(std::move(b));
    }
    net.cls.name = "classifier";
    net.cls.cin = c;
    for (const json& e : doc.at("classifier")) {
        const std::string kind = e.at("kind").get<std::string>();
        if (kind == "global_avg_pool") {
            net.cls.layers.push_back(plain_layer(GAP, c));
        } else if (kind == "relu") {
            net.cls.layers.push_back(plain_layer(RELU, c));
        } else if (kind == "dense") {  // model.cpp:200-209
            Layer l;
            l.kind = DENSE;
            l.cin = c;
            l.cout = e.at("out_features").get<int>();
            l.k = 1;
            l.weight = T4(l.cout, c, 1, 1);
            l.bias = T4(1, l.cout, 1, 1);
            net.cls.layers.push_back(std::move(l));
        } else {
            throw std::invalid_argument("unknown classifier layer '" + kind + "'");
        }
        layer_shape(net.cls.layers.back(), c, h, w);
    }
    return net;
}

// model.cpp:384-419 -- a fresh normal_distribution per tensor, layer order.
void init_block(Block& b, std::mt19937_64& rng) {
    auto fill = [&rng](T4& t, double fan_in) {
        std::normal_distribution<float> dist(0.0f, static_cast<float>(std::sqrt(2.0 / fan_in)));
        for (float& v : t.d) v = dist(rng);
    };
    for (Layer& l : b.layers) {
        switch (l.kind) {
            case Conv3:
            case Conv1:
                fill(l.weight, static_cast<double>(l.cin) * l.k * l.k);
                break;
            case DW:
                fill(l.weight, static_cast<double>(l.k) * l.k);
                break;
            case PW:
                fill(l.weight, l.cin);
                break;
            case DENSE:
                fill(l.weight, l.cin);
                std::fill(l.bias.d.begin(), l.bias.d.end(), 0.0f);
                break;
            case BN:
                std::fill(l.gamma.d.begin(), l.gamma.d.end(), 1.0f);
                std::fill(l.beta.d.begin(), l.beta.d.end(), 0.0f);
                std::fill(l.mm.d.begin(), l.mm.d.end(), 0.0f);
                std::fill(l.mv.d.begin(), l.mv.d.end(), 1.0f);
                break;
            case ADD:
                if (!l.weight.d.empty()) fill(l.weight, l.cin);
                break;
            default:
                break;
        }
    }
}

// model.cpp:448-478 -- serialization order of a block's arrays.
void each_array(Block& b, const std::function<void(T4&)>& fn) {
    for (Layer& l : b.layers) {
        switch (l.kind) {
            case Conv3:
            case Conv1:
            case DW:
            case PW:
                fn(l.weight);
                break;
            case DENSE:
                fn(l.weight);
                fn(l.bias);
                break;
            case BN:
                fn(l.gamma);
                fn(l.beta);
                fn(l.mm);
                fn(l.mv);
                break;
            case ADD:
                if (!l.weight.d.empty()) fn(l.weight);
                break;
            default:
                break;
        }
    }
}

void each_net_array(Net& net, const std::function<void(T4&)>& fn) {
    for (Block& b : net.blocks) each_array(b, fn);
    if (!net.cls.layers.empty()) each_array(net.cls, fn);
}

size_t block_store(Block& b, float* out, size_t cap) {
    size_t at = 0;
    each_array(b, [&](T4& t) {
        if (out) {
            if (at + t.d.size() > cap) throw std::length_error("buffer too small");
            std::copy(t.d.begin(), t.d.end(), out + at);
        }
        at += t.d.size();
    });
    return at;
}

void block_load(Block& b, const float* in) {
    size_t at = 0;
    each_array(b, [&](T4& t) {
        std::copy(in + at, in + at + t.d.size(), t.d.begin());
        at += t.d.size();
    });
}

Net load_net(const char* spec, const float* tw) {
    Net net = parse_spec(spec);
    if (tw) {
        size_t at = 0;
        each_net_array(net, [&](T4& t) {
            std::copy(tw + at, tw + at + t.d.size(), t.d.begin());
            at += t.d.size();
        });
    }
    return net;
}

// replacement.cpp:11-16, 36-72
Block candidate(int kind, int cin, int cout, int s, uint64_t seed) {
    if (cin < 1 || cout < 1) throw std::invalid_argument("build_candidate: channel counts");
    if (s != 1 && s != 2) throw std::invalid_argument("build_candidate: stride must be 1 or 2");
    static const char* names[] = {"two_layer", "three_layer", "two_layer_skip", "three_layer_skip"};
    Block b;
    b.name = "replacement";
    b.spec_kind = names[kind];
    b.cin = cin;
    b.cout = cout;
    b.stride = s;
    const bool skip = kind == 2 || kind == 3;
    const int units = (kind == 1 || kind == 3) ? 3 : 2;
    auto unit = [&b](int ci, int co, int st, bool relu) {
        b.layers.push_back(conv_layer(DW, ci, ci, 3, st, 1));
        b.layers.push_back(conv_layer(PW, ci, co, 1, 1, 0));
        b.layers.push_back(bn_layer(co));
        if (relu) b.layers.push_back(plain_layer(RELU, co));
    };
    unit(cin, cout, s, true);
    for (int u = 1; u < units; ++u) unit(cout, cout, 1, !(skip && u == units - 1));
    if (skip) {
        b.layers.push_back(add_layer(cin, cout, s));
        b.layers.push_back(plain_layer(RELU, cout));
    }
    std::mt19937_64 rng(seed);
    init_block(b, rng);
    return b;
}

// ---------------------------------------------------------------------------
// Execution (model.cpp:498-656)
// ---------------------------------------------------------------------------
struct LayerCache {
    T4 input;
    BnCache bn;
};
struct BlockCache {
    bool train = false;
    std::vector<LayerCache> layers;
};

T4 block_forward(Block& b, const T4& x, bool train, BlockCache* cache) {
    if (cache) {
        cache->train = train;
        cache->layers.assign(b.layers.size(), LayerCache{});
    }
    T4 cur = x;
    for (size_t i = 0; i < b.layers.size(); ++i) {
        Layer& l = b.layers[i];
        if (cache) cache->layers[i].input = cur;
        T4 next;
        switch (l.kind) {
            case Conv3:
            case Conv1:
                next = conv_fwd(cur, l.weight, l.stride, l.pad);
                break;
            case DW:
                next = dw_fwd(cur, l.weight, l.stride, l.pad);
                break;
            case PW:
                next = pw_fwd(cur, l.weight, l.stride);
                break;
            case BN:
                next = train ? bn_train_fwd(cur, l.gamma.d.data(), l.beta.d.data(), l.mm.d.data(),
                                            l.mv.d.data(), kBnMomentum,
                                            cache ? &cache->layers[i].bn : nullptr)
                             : bn_infer(cur, l.gamma.d.data(), l.beta.d.data(), l.mm.d.data(),
                                        l.mv.d.data());
                break;
            case RELU:
                next = relu_fwd(cur);
                break;
            case GAP:
                next = gap_fwd(cur);
                break;
            case DENSE:
                next = dense_fwd(cur, l.weight, l.bias);
                break;
            case ADD:
                next = add_fwd(cur, l.weight.d.empty() ? x : pw_fwd(x, l.weight, l.stride));
                break;
        }
        cur = std::move(next);
    }
    return cur;
}

T4 block_infer(const Block& b, const T4& x) {
    return block_forward(const_cast<Block&>(b), x, false, nullptr);
}

void ensure(T4& g, const T4& like) {
    if (g.d.size() != like.d.size()) g = T4(like.n, like.c, like.h, like.w);
}

// Parameter-gradient backward of a train-mode block (need_input_grad=false,
// the only mode train_block uses for LocalOnly: distill.cpp:247).
void block_backward(Block& b, const BlockCache& cache, const T4& gy) {
    T4 g = gy;
    for (int i = static_cast<int>(b.layers.size()) - 1; i >= 0; --i) {
        Layer& l = b.layers[i];
        const T4& x = cache.layers[i].input;
        const bool want_gx = i > 0;
        float* gw = nullptr;
        if (!l.weight.d.empty() && l.kind != ADD) {
            ensure(l.wgrad, l.weight);
            gw = l.wgrad.d.data();
        }
        T4 gx;
        if (want_gx && l.kind != ADD) gx = T4(x.n, x.c, x.h, x.w);
        float* gxp = gx.d.empty() ? nullptr : gx.d.data();
        switch (l.kind) {
            case Conv3:
            case Conv1:
                conv_bwd(x, l.weight, g, l.stride, l.pad, gxp, gw);
                break;
            case DW:
                dw_bwd(x, l.weight, g, l.stride, l.pad, gxp, gw);
                break;
            case PW:
                pw_bwd(x, l.weight, g, l.stride, gxp, gw);
                break;
            case BN:
                ensure(l.ggrad, l.gamma);
                ensure(l.btgrad, l.beta);
                bn_train_bwd(cache.layers[i].bn, l.gamma.d.data(), g, gxp, l.ggrad.d.data(),
                             l.btgrad.d.data());
                break;
            case RELU:
                relu_bwd(x, g, gxp);
                break;
            case ADD:
                if (!l.weight.d.empty()) {
                    ensure(l.wgrad, l.weight);
                    pw_bwd(cache.layers[0].input, l.weight, g, l.stride, nullptr, l.wgrad.d.data());
                }
                gx = std::move(g);
                break;
            default:
                throw std::logic_error("oracle: layer kind has no student backward");
        }
        g = want_gx ? std::move(gx) : T4();
    }
}

// SgdState (distill.cpp:114-133) over collect_block_trainable order
// (model.cpp:427-438): weight, bias, gamma, beta per layer.
struct Sgd {
    std::vector<std::pair<T4*, T4*>> params;  // (tensor, grad)
    std::vector<std::vector<float>> vel;
    explicit Sgd(Block& b) {
        for (Layer& l : b.layers) {
            if (!l.weight.d.empty()) {
                ensure(l.wgrad, l.weight);
                params.push_back({&l.weight, &l.wgrad});
            }
            if (!l.bias.d.empty()) {
                ensure(l.bgrad, l.bias);
                params.push_back({&l.bias, &l.bgrad});
            }
            if (l.kind == BN) {
                ensure(l.ggrad, l.gamma);
                ensure(l.btgrad, l.beta);
                params.push_back({&l.gamma, &l.ggrad});
                params.push_back({&l.beta, &l.btgrad});
            }
        }
        for (auto& p : params) vel.emplace_back(p.first->d.size(), 0.0f);
    }
    void zero() {
        for (auto& p : params) std::fill(p.second->d.begin(), p.second->d.end(), 0.0f);
    }
    void step(float lr, float mom) {
        for (size_t i = 0; i < params.size(); ++i)
            sgd(params[i].first->d.data(), params[i].second->d.data(), vel[i].data(),
                params[i].first->d.size(), lr, mom);
    }
};

T4 prefix(const Net& net, const T4& x, int k, bool inclusive) {  // model.cpp:695-704
    if (k < 1 || k > static_cast<int>(net.blocks.size())) throw std::out_of_range("prefix_infer: k");
    const int take = inclusive ? k : k - 1;
    T4 cur = x;
    for (int i = 0; i < take; ++i) cur = block_infer(net.blocks[i], cur);
    return cur;
}

// ---------------------------------------------------------------------------
// Data (dataset.cpp)
// ---------------------------------------------------------------------------
struct Data {
    int c, h, w, classes, count;
    const float* images;
    const int* labels;
    size_t isz() const { return static_cast<size_t>(c) * h * w; }
};

T4 gather(const Data& d, const std::vector<int>& idx) {  // dataset.cpp:166-179
    T4 b(static_cast<int>(idx.size()), d.c, d.h, d.w);
    for (size_t i = 0; i < idx.size(); ++i) {
        if (idx[i] < 0 || idx[i] >= d.count) throw std::out_of_range("gather_batch: index");
        std::copy_n(d.images + static_cast<size_t>(idx[i]) * d.isz(), d.isz(), &b.d[i * d.isz()]);
    }
    return b;
}

std::vector<std::vector<int>> batches_of(const std::vector<int>& idx, int bs) {  // distill.cpp:22-30
    std::vector<std::vector<int>> out;
    for (size_t at = 0; at < idx.size(); at += static_cast<size_t>(bs))
        out.emplace_back(idx.begin() + at, idx.begin() + std::min(idx.size(), at + bs));
    return out;
}

long correct_of(const T4& logits, const Data& d, const std::vector<int>& idx) {  // distill.cpp:38-55
    long correct = 0;
    for (int i = 0; i < logits.n; ++i) {
        int best = 0;
        float bv = logits.d[logits.at(i, 0, 0, 0)];
        for (int c = 1; c < logits.c; ++c) {
            const float v = logits.d[logits.at(i, c, 0, 0)];
            if (v > bv) {
                bv = v;
                best = c;
            }
        }
        if (best == d.labels[idx[i]]) ++correct;
    }
    return correct;
}

double eval_student(const Net& net, int k, const Block& student, const Data& d,
                    const std::vector<int>& eval_idx, int bs) {  // distill.cpp:264-283
    if (eval_idx.empty()) throw std::invalid_argument("evaluation split is empty");
    long correct = 0;
    for (const auto& batch : batches_of(eval_idx, bs)) {
        T4 cur = prefix(net, gather(d, batch), k, false);
        cur = block_infer(student, cur);
        for (size_t bi = static_cast<size_t>(k); bi < net.blocks.size(); ++bi)
            cur = block_infer(net.blocks[bi], cur);
        if (!net.cls.layers.empty()) cur = block_infer(net.cls, cur);
        correct += correct_of(cur, d, batch);
    }
    return static_cast<double>(correct) / static_cast<double>(eval_idx.size());
}

Data to_data(const orc_dataset* d) {
    return Data{d->c, d->h, d->w, d->classes, d->count, d->images, d->labels};
}

void validate(const orc_task* t, const Net& net) {  // distill.cpp:86-100
    if (t->epochs < 1) throw std::invalid_argument("epochs must be at least 1");
    if (t->eval_every < 1) throw std::invalid_argument("eval_every must be at least 1");
    if (t->batch_size < 1) throw std::invalid_argument("batch_size must be at least 1");
    if (t->lambda_local < 0) throw std::invalid_argument("lambda_local must be non-negative");
    if (t->threshold < 0.0 || t->threshold > 1.0) throw std::invalid_argument("threshold");
    if (t->max_steps < 0) throw std::invalid_argument("max_steps must be non-negative");
    if (t->block_index < 1 || t->block_index > static_cast<int>(net.blocks.size()) ||
        !net.blocks[t->block_index - 1].replaceable)
        throw std::invalid_argument("block " + std::to_string(t->block_index) + " is not replaceable");
    if (t->loss_mode != 0) throw std::invalid_argument("oracle restates LocalOnly mode only");
}

// Runs f(i) for i in [0, n) on up to `threads` host threads (dynamic
// assignment; results must not depend on which thread runs which i).
void parallel_for(int n, int threads, const std::function<void(int)>& f) {
    std::atomic<int> next{0};
    std::string err;
    std::atomic<bool> bad{false};
    auto body = [&] {
        for (int i; (i = next.fetch_add(1)) < n && !bad;) {
            try {
                f(i);
            } catch (const std::exception& e) {
                if (!bad.exchange(true)) err = e.what();
            }
        }
    };
    const int nt = std::max(1, std::min(threads, n));
    std::vector<std::thread> pool;
    for (int t = 1; t < nt; ++t) pool.emplace_back(body);
    body();
    for (std::thread& t : pool) t.join();
    if (bad) throw std::runtime_error(err);
}

T4 wrap(const float* p, int n, int c, int h, int w) {
    T4 t(n, c, h, w);
    std::copy(p, p + t.d.size(), t.d.begin());
    return t;
}

}  // namespace

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }

uint64_t orc_mix_seed(uint64_t a, uint64_t b) { return splitmix(a, b); }

void orc_shuffle(int* idx, int n, uint64_t seed) {
    std::mt19937_64 rng(seed);
    std::shuffle(idx, idx + n, rng);
}

int orc_stratified_split(const int* labels, int n, double frac, uint64_t seed, int* train_out,
                         int* n_train, int* eval_out, int* n_eval) {
    return guard([&] {  // dataset.cpp:136-164
        if (n == 0) throw std::invalid_argument("stratified_split: dataset is empty");
        if (frac <= 0.0 || frac >= 1.0) throw std::invalid_argument("stratified_split: fraction");
        std::vector<std::vector<int>> by;
        for (int i = 0; i < n; ++i) {
            if (labels[i] >= static_cast<int>(by.size())) by.resize(labels[i] + 1);
            by[labels[i]].push_back(i);
        }
        std::vector<int> tr, ev;
        for (size_t cls = 0; cls < by.size(); ++cls) {
            auto& m = by[cls];
            if (m.empty()) continue;
            std::mt19937_64 rng(splitmix(seed, cls));
            std::shuffle(m.begin(), m.end(), rng);
            if (m.size() < 2) throw std::invalid_argument("stratified_split: class too small");
            auto take = static_cast<size_t>(std::lround(frac * m.size()));
            take = std::clamp<size_t>(take, 1, m.size() - 1);
            ev.insert(ev.end(), m.begin(), m.begin() + take);
            tr.insert(tr.end(), m.begin() + take, m.end());
        }
        std::sort(ev.begin(), ev.end());
        std::sort(tr.begin(), tr.end());
        std::copy(tr.begin(), tr.end(), train_out);
        std::copy(ev.begin(), ev.end(), eval_out);
        *n_train = static_cast<int>(tr.size());
        *n_eval = static_cast<int>(ev.size());
    });
}

int orc_synthetic_dataset(int count, uint64_t seed, int threads, float* images, int* labels) {
    return guard([&] {  // dataset.cpp:21-48, 52-84 (threads do not change the bytes)
        (void)threads;
        constexpr int side = 16;
        constexpr float pi = std::numbers::pi_v<float>;
        static constexpr float scale[3] = {1.0f, 0.75f, 0.5f};
        for (int i = 0; i < count; ++i) {
            const int label = i % 10;
            labels[i] = label;
            std::mt19937_64 rng(splitmix(seed, static_cast<uint64_t>(i)));
            std::uniform_real_distribution<float> phase_d(0.0f, 2.0f * pi);
            std::uniform_real_distribution<float> amp_d(0.7f, 1.0f);
            std::normal_distribution<float> noise(0.0f, 0.05f);
            const float theta = pi * static_cast<float>(label % 5) / 5.0f;
            const float freq = label < 5 ? 2.0f : 4.0f;
            const float phase = phase_d(rng);
            const float amp = amp_d(rng);
            const float ct = std::cos(theta), st = std::sin(theta);
            float* out = images + static_cast<size_t>(i) * 3 * side * side;
            size_t q = 0;
            for (int ch = 0; ch < 3; ++ch)
                for (int y = 0; y < side; ++y) {
                    const float v = static_cast<float>(y) / (side - 1) - 0.5f;
                    for (int x = 0; x < side; ++x) {
                        const float u = static_cast<float>(x) / (side - 1) - 0.5f;
                        const float t = ct * u + st * v;
                        const float s = std::sin(2.0f * pi * freq * t + phase);
                        const float val = 0.5f + 0.5f * amp * s * scale[ch] + noise(rng);
                        out[q++] = std::clamp(val, 0.0f, 1.0f);
                    }
                }
        }
    });
}

int orc_round_robin(const int* ids, int n, int workers, int* out_ids, int* out_counts) {
    return guard([&] {  // scheduler.cpp:43-55
        if (workers < 1) throw std::invalid_argument("worker_count must be at least 1");
        std::vector<std::vector<int>> a(workers);
        for (int i = 0; i < n; ++i) a[i % workers].push_back(ids[i]);
        int at = 0;
        for (int w = 0; w < workers; ++w) {
            out_counts[w] = static_cast<int>(a[w].size());
            for (int id : a[w]) out_ids[at++] = id;
        }
    });
}

int orc_wfd(const int* ids, const double* weights, int n, int workers, int* out_ids,
            int* out_counts, double* mk) {
    return guard([&] {  // scheduler.cpp:57-81
        if (workers < 1) throw std::invalid_argument("worker_count must be at least 1");
        std::vector<std::pair<int, double>> order;
        for (int i = 0; i < n; ++i) {
            if (!(weights[i] > 0)) throw std::invalid_argument("non-positive weight");
            order.push_back({ids[i], weights[i]});
        }
        std::stable_sort(order.begin(), order.end(), [](const auto& a, const auto& b) {
            if (a.second != b.second) return a.second > b.second;
            return a.first < b.first;
        });
        std::vector<std::vector<int>> a(workers);
        std::vector<double> load(workers, 0.0);
        for (const auto& t : order) {
            int bin = 0;
            for (int w = 1; w < workers; ++w)
                if (load[w] < load[bin]) bin = w;
            a[bin].push_back(t.first);
            load[bin] += t.second;
        }
        int at = 0;
        for (int w = 0; w < workers; ++w) {
            out_counts[w] = static_cast<int>(a[w].size());
            for (int id : a[w]) out_ids[at++] = id;
        }
        *mk = *std::max_element(load.begin(), load.end());
    });
}

int orc_teacher_num_floats(const char* spec, size_t* n) {
    return guard([&] {
        Net net = parse_spec(spec);
        size_t at = 0;
        each_net_array(net, [&](T4& t) { at += t.d.size(); });
        *n = at;
    });
}

int orc_teacher_num_blocks(const char* spec, int* n) {
    return guard([&] { *n = static_cast<int>(parse_spec(spec).blocks.size()); });
}

int orc_teacher_init(const char* spec, uint64_t seed, float* out, size_t cap) {
    return guard([&] {  // model.cpp:421-425
        Net net = parse_spec(spec);
        std::mt19937_64 rng(seed);
        for (Block& b : net.blocks) init_block(b, rng);
        init_block(net.cls, rng);
        size_t at = 0;
        each_net_array(net, [&](T4& t) {
            if (at + t.d.size() > cap) throw std::length_error("teacher buffer too small");
            std::copy(t.d.begin(), t.d.end(), out + at);
            at += t.d.size();
        });
    });
}

int orc_block_macs(const char* spec, int k, long long* macs) {
    return guard([&] {  // model.cpp:724-777, summed over one block's rows
        Net net = parse_spec(spec);
        int c = net.in_c, h = net.in_h, w = net.in_w;
        for (int bi = 0; bi < k - 1; ++bi)
            for (const Layer& l : net.blocks.at(bi).layers) layer_shape(l, c, h, w);
        long long s = 0;
        for (const Layer& l : net.blocks.at(k - 1).layers) {
            layer_shape(l, c, h, w);
            const long long sp = static_cast<long long>(h) * w;
            if (l.kind == Conv3 || l.kind == Conv1) s += sp * l.k * l.k * l.cin * l.cout;
            if (l.kind == ADD && !l.weight.d.empty()) s += sp * l.cin * l.cout;
        }
        *macs = s;
    });
}

int orc_candidate_num_floats(int kind, int cin, int cout, int stride, size_t* n) {
    return guard([&] {
        Block b = candidate(kind, cin, cout, stride, 0);
        *n = block_store(b, nullptr, 0);
    });
}

int orc_build_candidate(int kind, int cin, int cout, int stride, uint64_t seed, float* out,
                        size_t cap) {
    return guard([&] {
        Block b = candidate(kind, cin, cout, stride, seed);
        block_store(b, out, cap);
    });
}

void orc_dw_fwd(const float* x, int n, int c, int h, int w, const float* k, int kk, int s, int p,
                float* y) {
    T4 t = dw_fwd(wrap(x, n, c, h, w), wrap(k, c, 1, kk, kk), s, p);
    std::copy(t.d.begin(), t.d.end(), y);
}

void orc_dw_bwd(const float* x, int n, int c, int h, int w, const float* k, int kk, int s, int p,
                const float* gy, float* gx, float* gk) {
    const int ho = out_dim(h, kk, s, p), wo = out_dim(w, kk, s, p);
    dw_bwd(wrap(x, n, c, h, w), wrap(k, c, 1, kk, kk), wrap(gy, n, c, ho, wo), s, p, gx, gk);
}

void orc_pw_fwd(const float* x, int n, int c, int h, int w, const float* k, int co, int s,
                float* y) {
    T4 t = pw_fwd(wrap(x, n, c, h, w), wrap(k, co, c, 1, 1), s);
    std::copy(t.d.begin(), t.d.end(), y);
}

void orc_pw_bwd(const float* x, int n, int c, int h, int w, const float* k, int co, int s,
                const float* gy, float* gx, float* gk) {
    const int ho = out_dim(h, 1, s, 0), wo = out_dim(w, 1, s, 0);
    pw_bwd(wrap(x, n, c, h, w), wrap(k, co, c, 1, 1), wrap(gy, n, co, ho, wo), s, gx, gk);
}

void orc_conv_fwd(const float* x, int n, int c, int h, int w, const float* k, int co, int kk,
                  int s, int p, float* y) {
    T4 t = conv_fwd(wrap(x, n, c, h, w), wrap(k, co, c, kk, kk), s, p);
    std::copy(t.d.begin(), t.d.end(), y);
}

void orc_bn_train_fwd(const float* x, int n, int c, int h, int w, const float* gamma,
                      const float* beta, float* mm, float* mv, float mom, float* y, float* xhat,
                      float* inv_std) {
    BnCache cache;
    T4 t = bn_train_fwd(wrap(x, n, c, h, w), gamma, beta, mm, mv, mom, &cache);
    std::copy(t.d.begin(), t.d.end(), y);
    if (xhat) std::copy(cache.xhat.d.begin(), cache.xhat.d.end(), xhat);
    if (inv_std) std::copy(cache.inv_std.begin(), cache.inv_std.end(), inv_std);
}

void orc_bn_train_bwd(const float* xhat, const float* inv_std, const float* gamma,
                      const float* gy, int n, int c, int h, int w, float* gx, float* ggamma,
                      float* gbeta) {
    BnCache cache;
    cache.xhat = wrap(xhat, n, c, h, w);
    cache.inv_std.assign(inv_std, inv_std + c);
    bn_train_bwd(cache, gamma, wrap(gy, n, c, h, w), gx, ggamma, gbeta);
}

void orc_bn_infer_fwd(const float* x, int n, int c, int h, int w, const float* gamma,
                      const float* beta, const float* mm, const float* mv, float* y) {
    T4 t = bn_infer(wrap(x, n, c, h, w), gamma, beta, mm, mv);
    std::copy(t.d.begin(), t.d.end(), y);
}

float orc_mse(const float* s, const float* t, size_t count) { return mse(s, t, count); }

void orc_mse_bwd(const float* s, const float* t, size_t count, float scale, float* g) {
    mse_bwd(s, t, count, scale, g);
}

void orc_sgd(float* w, const float* g, float* v, size_t n, float lr, float mom) {
    sgd(w, g, v, n, lr, mom);
}

int orc_prefix_infer(const char* spec, const float* tw, const float* x, int n, int k,
                     int inclusive, float* out, size_t cap, int* shape) {
    return guard([&] {
        Net net = load_net(spec, tw);
        T4 y = prefix(net, wrap(x, n, net.in_c, net.in_h, net.in_w), k, inclusive != 0);
        if (y.d.size() > cap) throw std::length_error("prefix buffer too small");
        std::copy(y.d.begin(), y.d.end(), out);
        shape[0] = y.n, shape[1] = y.c, shape[2] = y.h, shape[3] = y.w;
    });
}

int orc_candidate_infer(int kind, int cin, int cout, int stride, const float* bw, const float* x,
                        int n, int h, int w, float* out, size_t cap) {
    return guard([&] {
        Block b = candidate(kind, cin, cout, stride, 0);
        block_load(b, bw);
        T4 y = block_infer(b, wrap(x, n, cin, h, w));
        if (y.d.size() > cap) throw std::length_error("output buffer too small");
        std::copy(y.d.begin(), y.d.end(), out);
    });
}

int orc_eval_with_student(const char* spec, const float* tw, const orc_dataset* d,
                          const int* eval_idx, int n_eval, int k, int kind, const float* sw,
                          int bs, double* acc) {
    return guard([&] {
        Net net = load_net(spec, tw);
        const Block& tb = net.blocks.at(k - 1);
        Block st = candidate(kind, tb.cin, tb.cout, tb.stride, 0);
        block_load(st, sw);
        *acc = eval_student(net, k, st, to_data(d), std::vector<int>(eval_idx, eval_idx + n_eval), bs);
    });
}

int orc_train_block(const char* spec, const float* tw, const orc_dataset* dd, const orc_split* s,
                    const orc_task* t, orc_result* r, float* block_w, size_t cap) {
    return orc_train_block_f64(spec, tw, dd, s, t, r, block_w, cap, nullptr);
}

int orc_train_block_f64(const char* spec, const float* tw, const orc_dataset* dd, const orc_split* s,
                        const orc_task* t, orc_result* r, float* block_w, size_t cap, double* hist64) {
    auto mse64 = [](const T4& a, const T4& b) {
        double acc = 0.0;
        for (size_t q = 0; q < a.d.size(); ++q) {
            const double df = static_cast<double>(a.d[q]) - static_cast<double>(b.d[q]);
            acc += df * df;
        }
        return acc / static_cast<double>(a.d.size());
    };
    return guard([&] {  // distill.cpp:135-262 (LocalOnly)
        Net net = load_net(spec, tw);
        validate(t, net);
        if (s->n_train == 0) throw std::invalid_argument("training split is empty");
        if (s->n_eval == 0) throw std::invalid_argument("evaluation split is empty");
        const Data d = to_data(dd);
        const std::vector<int> train(s->train_idx, s->train_idx + s->n_train);
        const std::vector<int> evalv(s->eval_idx, s->eval_idx + s->n_eval);
        const int k = t->block_index;
        const Block& tb = net.blocks[k - 1];
        Block student = candidate(t->kind, tb.cin, tb.cout, tb.stride, splitmix(t->seed, 0));
        Sgd opt(student);
        std::memset(r, 0, sizeof(*r));
        r->best_eval = -1.0;
        Block best;
        auto record = [&](int epoch) {
            const double acc = eval_student(net, k, student, d, evalv, t->batch_size);
            r->eval_epoch[r->n_eval] = epoch;
            r->eval_acc[r->n_eval++] = acc;
            if (acc > r->best_eval) {
                r->best_eval = acc;
                best = student;
            }
        };
        {  // epoch-0 baseline, inference mode, unshuffled (distill.cpp:166-192)
            double sum = 0.0, sum64 = 0.0;
            const auto bs = batches_of(train, t->batch_size);
            for (const auto& b : bs) {
                const T4 a = prefix(net, gather(d, b), k, false);
                const T4 tt = block_infer(tb, a);
                const T4 so = block_infer(student, a);
                sum += static_cast<double>(mse(so.d.data(), tt.d.data(), so.d.size()));
                if (hist64) sum64 += mse64(so, tt);
            }
            if (hist64) hist64[r->n_loss] = sum64 / static_cast<double>(bs.size());
            r->loss_history[r->n_loss++] = sum / static_cast<double>(bs.size());
            r->final_local_loss = sum / static_cast<double>(bs.size());
        }
        record(0);
        long steps = 0;
        bool cap_hit = false;
        for (int epoch = 1; epoch <= t->epochs && !cap_hit; ++epoch) {
            std::vector<int> order = train;
            std::mt19937_64 rng(splitmix(t->seed, static_cast<uint64_t>(epoch)));
            std::shuffle(order.begin(), order.end(), rng);
            double sum = 0.0, sum64 = 0.0;
            int done = 0;
            for (const auto& b : batches_of(order, t->batch_size)) {
                if (t->max_steps > 0 && steps >= t->max_steps) {
                    cap_hit = true;
                    break;
                }
                const T4 a = prefix(net, gather(d, b), k, false);
                const T4 tt = block_infer(tb, a);
                BlockCache cache;
                const T4 so = block_forward(student, a, true, &cache);
                const double local = mse(so.d.data(), tt.d.data(), so.d.size());
                if (hist64) sum64 += mse64(so, tt);
                if (!std::isfinite(local)) {
                    r->failed = 1;
                    std::snprintf(r->failure, sizeof(r->failure),
                                  "block %d diverged at epoch %d batch %d (loss %g)", k, epoch, done,
                                  local);
                    break;
                }
                T4 gs(so.n, so.c, so.h, so.w);
                mse_bwd(so.d.data(), tt.d.data(), so.d.size(), 1.0f, gs.d.data());
                opt.zero();
                block_backward(student, cache, gs);
                opt.step(t->lr, t->momentum);
                sum += local;
                ++done;
                ++steps;
            }
            if (r->failed) break;
            if (done == 0) break;
            if (hist64) hist64[r->n_loss] = sum64 / done;
            r->loss_history[r->n_loss++] = sum / done;
            r->final_local_loss = sum / done;
            if (epoch % t->eval_every == 0) record(epoch);
        }
        if (block_w && !best.layers.empty()) block_store(best, block_w, cap);
    });
}

int orc_train_replay(const char* spec, const float* tw, const orc_dataset* dd, const orc_split* s,
                     const orc_task* t, int n_steps, float* step_loss, float* final_w,
                     size_t cap) {
    return orc_train_replay_f64(spec, tw, dd, s, t, n_steps, step_loss, nullptr, final_w, cap);
}

int orc_train_replay_f64(const char* spec, const float* tw, const orc_dataset* dd, const orc_split* s,
                         const orc_task* t, int n_steps, float* step_loss, double* loss64,
                         float* final_w, size_t cap) {
    return guard([&] {
        Net net = load_net(spec, tw);
        const Data d = to_data(dd);
        const std::vector<int> train(s->train_idx, s->train_idx + s->n_train);
        const int k = t->block_index;
        const Block& tb = net.blocks.at(k - 1);
        Block student = candidate(t->kind, tb.cin, tb.cout, tb.stride, splitmix(t->seed, 0));
        Sgd opt(student);
        int done = 0;
        for (int epoch = 1; done < n_steps; ++epoch) {
            std::vector<int> order = train;
            std::mt19937_64 rng(splitmix(t->seed, static_cast<uint64_t>(epoch)));
            std::shuffle(order.begin(), order.end(), rng);
            for (const auto& b : batches_of(order, t->batch_size)) {
                if (done >= n_steps) break;
                const T4 a = prefix(net, gather(d, b), k, false);
                const T4 tt = block_infer(tb, a);
                BlockCache cache;
                const T4 so = block_forward(student, a, true, &cache);
                step_loss[done] = mse(so.d.data(), tt.d.data(), so.d.size());
                if (loss64) {
                    double acc = 0.0;
                    for (size_t q = 0; q < so.d.size(); ++q) {
                        const double df = static_cast<double>(so.d[q]) - static_cast<double>(tt.d[q]);
                        acc += df * df;
                    }
                    loss64[done] = acc / static_cast<double>(so.d.size());
                }
                T4 gs(so.n, so.c, so.h, so.w);
                mse_bwd(so.d.data(), tt.d.data(), so.d.size(), 1.0f, gs.d.data());
                opt.zero();
                block_backward(student, cache, gs);
                opt.step(t->lr, t->momentum);
                ++done;
            }
        }
        block_store(student, final_w, cap);
    });
}


int orc_train_replay_multi(const char* spec, const float* tw, const orc_dataset* dd,
                           const orc_split* s, const orc_task* tasks, int n_tasks, int n_steps,
                           const int* ck_steps, int n_ck, int threads, float* step_loss,
                           double* loss64, float* ck_w, const size_t* w_off) {
    return guard([&] {
        const Net net = load_net(spec, tw);
        const Data d = to_data(dd);
        const std::vector<int> train(s->train_idx, s->train_idx + s->n_train);
        const int nt = static_cast<int>(train.size());
        int maxk = 0;
        for (int i = 0; i < n_tasks; ++i) maxk = std::max(maxk, tasks[i].block_index);
        if (maxk < 1 || maxk > static_cast<int>(net.blocks.size())) throw std::out_of_range("block index");
        // boundary j (0 = the input images) of every training sample, train order
        std::vector<std::vector<float>> bnd(static_cast<size_t>(maxk) + 1);
        std::vector<std::array<int, 3>> dims(static_cast<size_t>(maxk) + 1);
        {
            T4 cur = gather(d, {train.at(0)});
            for (int j = 0; j <= maxk; ++j) {
                if (j > 0) cur = block_infer(net.blocks[j - 1], cur);
                dims[j] = {cur.c, cur.h, cur.w};
                bnd[j].resize(static_cast<size_t>(nt) * cur.d.size());
            }
        }
        parallel_for(nt, threads, [&](int i) {
            T4 cur = gather(d, {train[i]});
            for (int j = 0; j <= maxk; ++j) {
                if (j > 0) cur = block_infer(net.blocks[j - 1], cur);
                std::copy(cur.d.begin(), cur.d.end(), bnd[j].begin() + static_cast<size_t>(i) * cur.d.size());
            }
        });
        auto rows = [&](int j, const std::vector<int>& pos) {
            const auto& dm = dims[j];
            T4 out(static_cast<int>(pos.size()), dm[0], dm[1], dm[2]);
            const size_t row = static_cast<size_t>(dm[0]) * dm[1] * dm[2];
            for (size_t q = 0; q < pos.size(); ++q)
                std::copy_n(bnd[j].begin() + static_cast<size_t>(pos[q]) * row, row, out.d.begin() + q * row);
            return out;
        };
        parallel_for(n_tasks, threads, [&](int ti) {
            const orc_task* t = &tasks[ti];
            const int k = t->block_index;
            const Block& tb = net.blocks.at(k - 1);
            Block student = candidate(t->kind, tb.cin, tb.cout, tb.stride, splitmix(t->seed, 0));
            Sgd opt(student);
            const size_t nf = n_ck > 0 ? (w_off[ti + 1] - w_off[ti]) / static_cast<size_t>(n_ck) : 0;
            int done = 0, ck = 0;
            for (int epoch = 1; done < n_steps; ++epoch) {
                // std::shuffle's permutation depends only on the length and the
                // engine, so shuffling positions equals shuffling train_idx
                std::vector<int> pos(nt);
                for (int q = 0; q < nt; ++q) pos[q] = q;
                std::mt19937_64 rng(splitmix(t->seed, static_cast<uint64_t>(epoch)));
                std::shuffle(pos.begin(), pos.end(), rng);
                for (const auto& b : batches_of(pos, t->batch_size)) {
                    if (done >= n_steps) break;
                    const T4 a = rows(k - 1, b);
                    const T4 tt = rows(k, b);
                    BlockCache cache;
                    const T4 so = block_forward(student, a, true, &cache);
                    float* sl = step_loss + static_cast<size_t>(ti) * n_steps;
                    sl[done] = mse(so.d.data(), tt.d.data(), so.d.size());
                    if (loss64) {
                        double acc = 0.0;
                        for (size_t q = 0; q < so.d.size(); ++q) {
                            const double df = static_cast<double>(so.d[q]) - static_cast<double>(tt.d[q]);
                            acc += df * df;
                        }
                        loss64[static_cast<size_t>(ti) * n_steps + done] = acc / static_cast<double>(so.d.size());
                    }
                    T4 gs(so.n, so.c, so.h, so.w);
                    mse_bwd(so.d.data(), tt.d.data(), so.d.size(), 1.0f, gs.d.data());
                    opt.zero();
                    block_backward(student, cache, gs);
                    opt.step(t->lr, t->momentum);
                    ++done;
                    while (ck < n_ck && ck_steps[ck] == done) {
                        block_store(student, ck_w + w_off[ti] + static_cast<size_t>(ck) * nf, nf);
                        ++ck;
                    }
                }
            }
        });
    });
}

int orc_run_parallel(const char* spec, const float* tw, const orc_dataset* dd, const orc_split* s,
                     const orc_task* tasks, int n_tasks, const int* plan_ids, const int* plan_counts,
                     int workers, int policy, orc_result* results, float* block_w, const size_t* w_off) {
    (void)policy;  // results are schedule-invariant (test_runtime.cpp:206-253)
    return guard([&] {  // runtime.cpp:124-243, workers as threads over the plan's queues
        std::vector<int> order(n_tasks);
        for (int i = 0; i < n_tasks; ++i) order[i] = i;
        std::sort(order.begin(), order.end(),
                  [&](int a, int b) { return tasks[a].block_index < tasks[b].block_index; });
        std::vector<std::vector<int>> queues(workers);
        for (int w = 0, at = 0; w < workers; ++w)
            for (int q = 0; q < plan_counts[w]; ++q, ++at) {
                int ti = -1;
                for (int i = 0; i < n_tasks; ++i)
                    if (tasks[i].block_index == plan_ids[at]) ti = i;
                if (ti < 0) throw std::invalid_argument("plan references unknown task id");
                queues[w].push_back(ti);
            }
        parallel_for(workers, workers, [&](int w) {
            for (int ti : queues[w]) {
                const int slot = static_cast<int>(std::find(order.begin(), order.end(), ti) - order.begin());
                const size_t cap = w_off[slot + 1] - w_off[slot];
                if (orc_train_block(spec, tw, dd, s, &tasks[ti], &results[slot], block_w + w_off[slot], cap)) {
                    std::memset(&results[slot], 0, sizeof(orc_result));
                    results[slot].failed = 1;
                    std::snprintf(results[slot].failure, sizeof(results[slot].failure), "%s", g_err.c_str());
                }
            }
        });
    });
}

}  // extern "C"
