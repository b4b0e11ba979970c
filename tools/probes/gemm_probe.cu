// Diagnosis probe (not part of the product): times grouped launches of the
// TMA GEMM kernel on pre-split operands for the pointwise shapes of the
// VGG-16 bench epoch, CUDA events around each launch, inputs L2-resident.
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++20 -I paper_2012_03096_b200/csrc \
//        -I paper_2012_03096_b200/include -I include tools/probes/gemm_probe.cu \
//        -L paper_2012_03096_b200 -lpbkd_b200 -lcuda -o tools/probes/_build/gemm_probe
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "ops.cuh"

using namespace pbkd_gpu;


#define CK(x)                                                                      \
    do {                                                                           \
        cudaError_t e_ = (x);                                                      \
        if (e_ != cudaSuccess) {                                                   \
            std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); \
            std::exit(1);                                                          \
        }                                                                          \
    } while (0)

struct Shape {
    int M, K, N;
};

static float* dalloc(size_t n) {
    float* p = nullptr;
    CK(cudaMalloc(&p, n * 4));
    std::vector<float> h(n);
    for (size_t i = 0; i < n; ++i) h[i] = static_cast<float>((i * 2654435761u) % 1000) / 1000.0f - 0.5f;
    CK(cudaMemcpy(p, h.data(), n * 4, cudaMemcpyHostToDevice));
    return p;
}

// epi: 0 store, 1 store + BN partials (fwd: A = X [M][K], B = W [N][K], both
// K-major); dgrad (epi 0, bmn): B = W [K][N] MN-major; wgrad: C[cout][cin] =
// sum_rows gp[row][cout] d[row][cin], both MN-major, split-K over rows as the engine
static void run(const char* name, std::vector<Shape> shapes, int epi, bool wgrad, int iters, bool bmn = false) {
    std::vector<GemmOp> ops;
    double flops = 0, bytes = 0;
    for (const Shape& s : shapes) {
        GemmOp g{};
        if (!wgrad) {
            g.M = s.M, g.N = s.N, g.K = s.K;
            const float* a = dalloc(static_cast<size_t>(s.M) * s.K);
            const float* b = dalloc(static_cast<size_t>(s.N) * s.K);
            g.A = a, g.lda = s.K, g.a_kmajor = 1;
            if (bmn) g.B = b, g.ldb = s.N, g.b_kmajor = 0;
            else g.B = b, g.ldb = s.K, g.b_kmajor = 1;
            g.a_hi = dalloc(static_cast<size_t>(s.M) * s.K), g.a_lo = dalloc(static_cast<size_t>(s.M) * s.K);
            g.b_hi = dalloc(static_cast<size_t>(s.N) * s.K), g.b_lo = dalloc(static_cast<size_t>(s.N) * s.K);
            g.a_ts_req = std::getenv("PROBE_TS") ? 1 : 0;
            g.C = dalloc(static_cast<size_t>(s.M) * s.N), g.ldc = s.N;
            g.ksplit = 1;
        } else {  // dW[N=cin? ] : C[cout][cin] = sum_rows dY[row][cout] X[row][cin]
            g.M = s.N, g.N = s.K, g.K = s.M;  // M = cout, N = cin, K = rows
            const float* dy = dalloc(static_cast<size_t>(s.M) * s.N);
            const float* x = dalloc(static_cast<size_t>(s.M) * s.K);
            g.A = dy, g.lda = s.N, g.a_kmajor = 0;
            g.B = x, g.ldb = s.K, g.b_kmajor = 0;
            g.a_hi = dalloc(static_cast<size_t>(s.M) * s.N), g.a_lo = dalloc(static_cast<size_t>(s.M) * s.N);
            g.b_hi = dalloc(static_cast<size_t>(s.M) * s.K), g.b_lo = dalloc(static_cast<size_t>(s.M) * s.K);
            g.a_ts_req = std::getenv("PROBE_TS") ? 1 : 0;
            g.ksplit = std::max(1, std::min(64, (s.M + 511) / 512));
            g.epi = 2;
        }
        flops += 2.0 * s.M * s.K * s.N;
        bytes += 4.0 * (static_cast<double>(s.M) * s.K + static_cast<double>(s.K) * s.N + static_cast<double>(s.M) * s.N);
        gemm_finalize(g);
        if (wgrad) {
            g.C = dalloc(static_cast<size_t>(g.ksplit) * g.M * g.N), g.ldc = g.N;
            gemm_finalize(g);
        }
        if (epi == 1 && !wgrad) {
            g.epi = 1;
            g.part0 = dalloc(static_cast<size_t>(g.tiles_m) * g.N), g.part1 = dalloc(static_cast<size_t>(g.tiles_m) * g.N);
        }
        ops.push_back(g);
    }
    const int cls = gemm_bn_class(ops[0]);
    for (const GemmOp& o : ops)
        if (gemm_bn_class(o) != cls) {
            std::printf("%s: mixed classes (%d vs %d), skipped\n", name, gemm_bn_class(o), cls);
            return;
        }
    int total = 0;
    long long chunks = 0;
    for (GemmOp& o : ops) {
        o.cta_begin = total;
        total += std::max(1, ctas_gemm(o));
        chunks += static_cast<long long>(ctas_gemm(o)) * ((std::min(o.K, o.kchunk) + 31) / 32);
    }
    GemmOp* d = nullptr;
    CK(cudaMalloc(&d, ops.size() * sizeof(GemmOp)));
    CK(cudaMemcpy(d, ops.data(), ops.size() * sizeof(GemmOp), cudaMemcpyHostToDevice));
    cudaStream_t st;
    CK(cudaStreamCreate(&st));
    for (int i = 0; i < 5; ++i) launch_gemm_bn(d, static_cast<int>(ops.size()), total, cls, st);
    CK(cudaStreamSynchronize(st));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    std::vector<float> ms(iters);
    for (int i = 0; i < iters; ++i) {
        CK(cudaEventRecord(e0, st));
        launch_gemm_bn(d, static_cast<int>(ops.size()), total, cls, st);
        CK(cudaEventRecord(e1, st));
        CK(cudaEventSynchronize(e1));
        CK(cudaEventElapsedTime(&ms[i], e0, e1));
    }
    std::sort(ms.begin(), ms.end());
    const double us = ms[iters / 2] * 1e3;
    {  // back-to-back launches (launch latency hidden) and a captured graph of them
        constexpr int kB = 20;
        float t = 0.0f;
        CK(cudaEventRecord(e0, st));
        for (int i = 0; i < kB; ++i) launch_gemm_bn(d, static_cast<int>(ops.size()), total, cls, st);
        CK(cudaEventRecord(e1, st));
        CK(cudaEventSynchronize(e1));
        CK(cudaEventElapsedTime(&t, e0, e1));
        cudaGraph_t gr;
        cudaGraphExec_t ge;
        CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
        for (int i = 0; i < kB; ++i) launch_gemm_bn(d, static_cast<int>(ops.size()), total, cls, st);
        CK(cudaStreamEndCapture(st, &gr));
        CK(cudaGraphInstantiate(&ge, gr, 0));
        CK(cudaGraphLaunch(ge, st));
        CK(cudaStreamSynchronize(st));
        float tg = 0.0f;
        CK(cudaEventRecord(e0, st));
        CK(cudaGraphLaunch(ge, st));
        CK(cudaEventRecord(e1, st));
        CK(cudaEventSynchronize(e1));
        CK(cudaEventElapsedTime(&tg, e0, e1));
        std::printf("    back-to-back %.2f us/launch, graph %.2f us/launch\n", t * 1e3 / kB, tg * 1e3 / kB);
        CK(cudaGraphExecDestroy(ge));
        CK(cudaGraphDestroy(gr));
    }
    const int grid = std::min(total, 148);
    std::printf("%-28s cls=%6d tiles=%5d chunks=%6lld  %8.2f us  %7.1f GB/s  %6.1f TF/s  chunks/CTA %.1f -> %.3f us/chunk\n",
                name, cls, total, chunks, us, bytes / us * 1e-3, flops / us * 1e-6, double(chunks) / grid,
                us / (double(chunks) / grid));
    CK(cudaFree(d));
}

__global__ void empty_kernel() {}

int main(int argc, char** argv) {
    {
        cudaStream_t st;
        CK(cudaStreamCreate(&st));
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        for (int i = 0; i < 10; ++i) empty_kernel<<<148, 448, 0, st>>>();
        float t1 = 0, t20 = 0;
        CK(cudaEventRecord(e0, st));
        empty_kernel<<<148, 448, 0, st>>>();
        CK(cudaEventRecord(e1, st));
        CK(cudaEventSynchronize(e1));
        CK(cudaEventElapsedTime(&t1, e0, e1));
        CK(cudaEventRecord(e0, st));
        for (int i = 0; i < 20; ++i) empty_kernel<<<148, 448, 0, st>>>();
        CK(cudaEventRecord(e1, st));
        CK(cudaEventSynchronize(e1));
        CK(cudaEventElapsedTime(&t20, e0, e1));
        std::printf("empty kernel: single %.2f us, back-to-back %.2f us/launch\n", t1 * 1e3, t20 * 1e3 / 20);
    }
    const int iters = argc > 1 ? std::atoi(argv[1]) : 50;
    if (argc > 6 && std::string(argv[2]) == "one") {  // one M K N epi
        run("one", {{std::atoi(argv[3]), std::atoi(argv[4]), std::atoi(argv[5])}}, std::atoi(argv[6]), false, iters);
        return 0;
    }
    if (argc > 2 && std::string(argv[2]) == "ksweep") {  // fixed cost vs per-chunk cost
        for (int k : {32, 64, 128, 256, 512, 1024, 2048}) {
            run(("1 tile K" + std::to_string(k)).c_str(), {{128, k, 128}}, 0, false, iters);
            run(("16 tiles K" + std::to_string(k)).c_str(), {{512, k, 512}}, 0, false, iters);
            run(("16 tiles epi1 K" + std::to_string(k)).c_str(), {{512, k, 512}}, 1, false, iters);
            run(("148 tiles K" + std::to_string(k)).c_str(), {{148 * 128, k, 128}}, 0, false, iters);
            run(("1 tile N64 K" + std::to_string(k)).c_str(), {{128, k, 64}}, 0, false, iters);
            run(("148 tiles N64 K" + std::to_string(k)).c_str(), {{148 * 128, k, 64}}, 0, false, iters);
        }
        return 0;
    }
    // steady state: 148 x 4 tiles of 128x128, K = 512 (16 chunks each)
    run("steady K512 N128", {{148 * 128 * 4, 512, 128}}, 0, false, iters);
    run("steady K512 N256 (2 tn)", {{148 * 128 * 2, 512, 256}}, 0, false, iters);
    run("steady K64 N64", {{148 * 128 * 8, 64, 64}}, 0, false, iters);
    run("b9 fwd 512^3", {{512, 512, 512}}, 1, false, iters);
    run("fwd u2 BN128 class",
        {{8192, 128, 128}, {8192, 128, 128}, {2048, 256, 256}, {2048, 256, 256}, {2048, 256, 256},
         {512, 512, 512}, {512, 512, 512}, {512, 512, 512}, {128, 512, 512}, {128, 512, 512}, {128, 512, 512}},
        1, false, iters);
    run("fwd u2 BN64 class", {{32768, 64, 64}, {32768, 64, 64}}, 1, false, iters);
    run("dgrad u2 BN128 class",
        {{8192, 128, 128}, {8192, 128, 128}, {2048, 256, 256}, {2048, 256, 256}, {2048, 256, 256},
         {512, 512, 512}, {512, 512, 512}, {512, 512, 512}, {128, 512, 512}, {128, 512, 512}, {128, 512, 512}},
        0, false, iters, true);
    run("wgrad u2 512 blocks",
        {{512, 512, 512}, {512, 512, 512}, {512, 512, 512}, {128, 512, 512}, {128, 512, 512}, {128, 512, 512}}, 2,
        true, iters);
    run("wgrad u2 b1-2", {{32768, 64, 64}, {32768, 64, 64}}, 2, true, iters);
    return 0;
}
