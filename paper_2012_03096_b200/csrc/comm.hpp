// comm.hpp -- exchange of teacher boundary activations between GPUs.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <vector>

namespace pbkd_gpu {

// 128-byte ncclUniqueId (rank 0 creates it, the launcher broadcasts it)
void nccl_unique_id(char* out128);

class NcclComm {
public:
    NcclComm(const char* id128, int rank, int world);
    ~NcclComm();
    NcclComm(const NcclComm&) = delete;
    NcclComm& operator=(const NcclComm&) = delete;
    int rank() const { return rank_; }
    int world() const { return world_; }
    // grouped ncclSend/ncclRecv, counts and offsets in floats, per peer
    void all_to_all_v(const float* send, const std::vector<size_t>& send_off, const std::vector<size_t>& send_cnt,
                      float* recv, const std::vector<size_t>& recv_off, const std::vector<size_t>& recv_cnt,
                      cudaStream_t st);

private:
    void* comm_ = nullptr;
    int rank_ = 0, world_ = 1;
};

// Who produces and who consumes which rows.  Pure host arithmetic, identical
// on every rank (checked across ranks by tests/test_multigpu_plan.py).
struct ExchangePlan {
    int world = 1;
    std::vector<int> shard_begin;           // world+1 train positions
    std::vector<int> blocks;                // all distilled blocks, ascending
    std::vector<int> owner;                 // owner rank per entry of blocks
    std::vector<long long> in_row, out_row; // floats per sample at boundary k-1 / k
    // layout of the buffer rank `src` sends to rank `dst`:
    // for each block b owned by dst (ascending): [in rows][tgt rows] for src's shard
    size_t count(int src, int dst) const;
    size_t offset_in(int src, int dst, size_t block_pos) const;   // within that buffer
    size_t offset_tgt(int src, int dst, size_t block_pos) const;
    int shard_rows(int s) const { return shard_begin[static_cast<size_t>(s) + 1] - shard_begin[static_cast<size_t>(s)]; }
};

// shards proportional to `share` (rounded, contiguous, covering [0, n))
std::vector<int> shard_bounds(int n, const std::vector<double>& share);

}  // namespace pbkd_gpu
