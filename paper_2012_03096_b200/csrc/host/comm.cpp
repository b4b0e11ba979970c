// comm.cpp -- NCCL all-to-all-v of teacher boundary activations (multi-GPU).
//
// The paper's only communication is the dispatch/gather pair;
// the B200 path adds one exchange per RUN: every GPU runs the teacher forward
// once on its shard of the training samples and ships the boundary rows the
// other GPUs' blocks read straight between the boundary buffers (grouped
// ncclSend/ncclRecv over NVLink; inference-mode teacher rows are per-sample
// and epoch-invariant, so one exchange serves every epoch).
//
// NCCL is resolved at run time with dlopen("libnccl.so.2") so the process
// shares whichever NCCL torch.distributed already loaded (one NCCL per process).
#include <dlfcn.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <stdexcept>
#include <string>

#include "../comm.hpp"
#include "nccl.h"

namespace pbkd_gpu {

namespace {
struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*comm_init_all)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*group_start)() = nullptr;
    ncclResult_t (*group_end)() = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;

    NcclApi() {
        h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("/usr/lib/x86_64-linux-gnu/libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return;
        auto sym = [this](const char* n) { return dlsym(h, n); };
        get_unique_id = reinterpret_cast<decltype(get_unique_id)>(sym("ncclGetUniqueId"));
        comm_init_rank = reinterpret_cast<decltype(comm_init_rank)>(sym("ncclCommInitRank"));
        comm_destroy = reinterpret_cast<decltype(comm_destroy)>(sym("ncclCommDestroy"));
        comm_init_all = reinterpret_cast<decltype(comm_init_all)>(sym("ncclCommInitAll"));
        send = reinterpret_cast<decltype(send)>(sym("ncclSend"));
        recv = reinterpret_cast<decltype(recv)>(sym("ncclRecv"));
        group_start = reinterpret_cast<decltype(group_start)>(sym("ncclGroupStart"));
        group_end = reinterpret_cast<decltype(group_end)>(sym("ncclGroupEnd"));
        error_string = reinterpret_cast<decltype(error_string)>(sym("ncclGetErrorString"));
    }
    bool ok() const { return h && get_unique_id && comm_init_rank && send && recv && group_start && group_end; }
};

NcclApi& api() {
    static NcclApi a;
    if (!a.ok()) throw std::runtime_error("NCCL (libnccl.so.2) could not be loaded");
    return a;
}

void check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        throw std::runtime_error(std::string(what) + ": " + (api().error_string ? api().error_string(r) : "nccl error"));
}
}  // namespace

void nccl_unique_id(char* out128) {
    ncclUniqueId id;
    check(api().get_unique_id(&id), "ncclGetUniqueId");
    std::memcpy(out128, id.internal, NCCL_UNIQUE_ID_BYTES);
}

NcclComm::NcclComm(const char* id128, int rank, int world) : rank_(rank), world_(world) {
    ncclUniqueId id;
    std::memcpy(id.internal, id128, NCCL_UNIQUE_ID_BYTES);
    ncclComm_t c = nullptr;
    check(api().comm_init_rank(&c, world, id, rank), "ncclCommInitRank");
    comm_ = c;
}

std::vector<std::unique_ptr<NcclComm>> NcclComm::clique(const std::vector<int>& devices) {
    auto& a = api();
    if (!a.comm_init_all) throw std::runtime_error("NCCL: ncclCommInitAll not available");
    std::vector<ncclComm_t> c(devices.size(), nullptr);
    check(a.comm_init_all(c.data(), static_cast<int>(devices.size()), devices.data()), "ncclCommInitAll");
    std::vector<std::unique_ptr<NcclComm>> out;
    for (size_t i = 0; i < c.size(); ++i)
        out.emplace_back(new NcclComm(c[i], static_cast<int>(i), static_cast<int>(c.size())));
    return out;
}

NcclComm::~NcclComm() {
    if (comm_) api().comm_destroy(static_cast<ncclComm_t>(comm_));
}

void NcclComm::exchange(const BoundaryPlan& plan, const std::vector<float*>& bnd, cudaStream_t st) {
    auto& a = api();
    auto c = static_cast<ncclComm_t>(comm_);
    check(a.group_start(), "ncclGroupStart");
    for (int p = 0; p < world_; ++p) {
        if (p == rank_) continue;
        // per peer pair, NCCL matches sends and receives in issue order: both
        // sides walk transfers(src, dst) in the same (j ascending) order
        for (const BoundaryPlan::Xfer& x : plan.transfers(rank_, p)) {
            const long long r = plan.row[static_cast<size_t>(x.j)];
            check(a.send(bnd[static_cast<size_t>(x.j)] + static_cast<size_t>(x.row0) * r,
                         static_cast<size_t>(x.rows) * r, ncclFloat, p, c, st), "ncclSend");
        }
        for (const BoundaryPlan::Xfer& x : plan.transfers(p, rank_)) {
            const long long r = plan.row[static_cast<size_t>(x.j)];
            check(a.recv(bnd[static_cast<size_t>(x.j)] + static_cast<size_t>(x.row0) * r,
                         static_cast<size_t>(x.rows) * r, ncclFloat, p, c, st), "ncclRecv");
        }
    }
    check(a.group_end(), "ncclGroupEnd");
}

}  // namespace pbkd_gpu

namespace pbkd_gpu {

std::vector<BoundaryPlan::Xfer> BoundaryPlan::transfers(int src, int dst) const {
    std::vector<Xfer> v;
    if (src == dst || shard_rows(src) == 0) return v;
    for (int j = 1; j <= kmax(); ++j)
        if (need[static_cast<size_t>(dst)][static_cast<size_t>(j)])
            v.push_back({j, shard_begin[static_cast<size_t>(src)], shard_rows(src)});
    return v;
}

size_t BoundaryPlan::count(int src, int dst) const {
    size_t n = 0;
    for (const Xfer& x : transfers(src, dst)) n += static_cast<size_t>(x.rows) * static_cast<size_t>(row[static_cast<size_t>(x.j)]);
    return n;
}

BoundaryPlan make_boundary_plan(const std::vector<int>& blocks, const std::vector<int>& owners,
                                const std::vector<long long>& row, int world, int n_train,
                                const std::vector<double>& share) {
    if (blocks.size() != owners.size()) throw std::invalid_argument("boundary plan: blocks / owners differ in length");
    if (world < 1) throw std::invalid_argument("boundary plan: world must be at least 1");
    BoundaryPlan p;
    p.world = world;
    p.row = row;
    int kmax = 0;
    for (int k : blocks) kmax = std::max(kmax, k);
    if (static_cast<int>(row.size()) < kmax + 1) throw std::invalid_argument("boundary plan: row sizes missing");
    p.row.resize(static_cast<size_t>(kmax) + 1);
    p.need.assign(static_cast<size_t>(world), std::vector<char>(static_cast<size_t>(kmax) + 1, 0));
    for (size_t i = 0; i < blocks.size(); ++i) {
        const int k = blocks[i], o = owners[i];
        if (k < 1 || o < 0 || o >= world) throw std::invalid_argument("boundary plan: bad block or owner");
        p.need[static_cast<size_t>(o)][static_cast<size_t>(k) - 1] = 1;
        p.need[static_cast<size_t>(o)][static_cast<size_t>(k)] = 1;
    }
    std::vector<double> sh = share;
    if (static_cast<int>(sh.size()) != world) sh.assign(static_cast<size_t>(world), 1.0);
    p.shard_begin = shard_bounds(n_train, sh);
    return p;
}

std::vector<int> shard_bounds(int n, const std::vector<double>& share) {
    const size_t w = share.size();
    double total = 0.0;
    for (double s : share) total += s;
    std::vector<int> b(w + 1, 0);
    double acc = 0.0;
    for (size_t i = 0; i < w; ++i) {
        acc += share[i];
        b[i + 1] = (i + 1 == w) ? n : static_cast<int>(std::lround(acc / total * n));
        if (b[i + 1] < b[i]) b[i + 1] = b[i];
    }
    return b;
}

}  // namespace pbkd_gpu
