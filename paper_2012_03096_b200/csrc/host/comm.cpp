// comm.cpp -- NCCL all-to-all-v of teacher boundary activations (multi-GPU).
//
// The paper's only communication is the dispatch/gather pair;
// the B200 path adds one exchange per epoch: every GPU runs the teacher forward
// on its shard of the training samples and ships each block's boundary rows to
// the GPU that owns that block (grouped ncclSend/ncclRecv over NVLink).
//
// NCCL is resolved at run time with dlopen("libnccl.so.2") so the process
// shares whichever NCCL torch.distributed already loaded (one NCCL per process).
#include <dlfcn.h>

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

NcclComm::~NcclComm() {
    if (comm_) api().comm_destroy(static_cast<ncclComm_t>(comm_));
}

void NcclComm::all_to_all_v(const float* send, const std::vector<size_t>& send_off, const std::vector<size_t>& send_cnt,
                            float* recv, const std::vector<size_t>& recv_off, const std::vector<size_t>& recv_cnt,
                            cudaStream_t st) {
    auto& a = api();
    auto c = static_cast<ncclComm_t>(comm_);
    check(a.group_start(), "ncclGroupStart");
    for (int p = 0; p < world_; ++p) {
        if (send_cnt[static_cast<size_t>(p)])
            check(a.send(send + send_off[static_cast<size_t>(p)], send_cnt[static_cast<size_t>(p)], ncclFloat, p, c, st),
                  "ncclSend");
        if (recv_cnt[static_cast<size_t>(p)])
            check(a.recv(recv + recv_off[static_cast<size_t>(p)], recv_cnt[static_cast<size_t>(p)], ncclFloat, p, c, st),
                  "ncclRecv");
    }
    check(a.group_end(), "ncclGroupEnd");
}

}  // namespace pbkd_gpu

namespace pbkd_gpu {

size_t ExchangePlan::count(int src, int dst) const {
    size_t n = 0;
    const size_t rows = static_cast<size_t>(shard_rows(src));
    for (size_t b = 0; b < blocks.size(); ++b)
        if (owner[b] == dst) n += rows * static_cast<size_t>(in_row[b] + out_row[b]);
    return n;
}

size_t ExchangePlan::offset_in(int src, int dst, size_t bp) const {
    size_t off = 0;
    const size_t rows = static_cast<size_t>(shard_rows(src));
    for (size_t b = 0; b < bp; ++b)
        if (owner[b] == dst) off += rows * static_cast<size_t>(in_row[b] + out_row[b]);
    return off;
}

size_t ExchangePlan::offset_tgt(int src, int dst, size_t bp) const {
    return offset_in(src, dst, bp) + static_cast<size_t>(shard_rows(src)) * static_cast<size_t>(in_row[bp]);
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
