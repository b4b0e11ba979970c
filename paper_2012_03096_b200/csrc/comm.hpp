// comm.hpp -- exchange of teacher boundary activations between GPUs.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <memory>
#include <vector>

namespace pbkd_gpu {

// 128-byte ncclUniqueId (rank 0 creates it, the launcher broadcasts it)
void nccl_unique_id(char* out128);

struct BoundaryPlan;

class NcclComm {
public:
    NcclComm(const char* id128, int rank, int world);
    // one process driving several GPUs: a clique over `devices`
    // (ncclCommInitAll), rank i on devices[i]
    static std::vector<std::unique_ptr<NcclComm>> clique(const std::vector<int>& devices);
    ~NcclComm();
    NcclComm(const NcclComm&) = delete;
    NcclComm& operator=(const NcclComm&) = delete;
    int rank() const { return rank_; }
    int world() const { return world_; }
    // one grouped ncclSend / ncclRecv round: this rank's shard rows of every
    // boundary a peer needs go out, the peers' rows of the boundaries this
    // rank needs come in, straight between the boundary buffers bnd[j]
    void exchange(const BoundaryPlan& plan, const std::vector<float*>& bnd, cudaStream_t st);

private:
    NcclComm(void* comm, int rank, int world) : comm_(comm), rank_(rank), world_(world) {}
    void* comm_ = nullptr;
    int rank_ = 0, world_ = 1;
};

// Who computes and who reads which teacher boundary rows.  Every rank holds
// boundaries 0..kmax for ALL training rows in train order; it computes the
// rows of its own shard (boundary 0, the images, it gathers itself for every
// row) and receives, once per run, the other shards' rows of each boundary
// j >= 1 that one of its blocks reads (block k reads k-1 and k).  A boundary
// shared by two blocks of one owner travels once.  Pure host arithmetic,
// identical on every rank (tests/test_multigpu.py checks it across ranks).
struct BoundaryPlan {
    int world = 1;
    std::vector<int> shard_begin;             // world+1 train rows
    std::vector<long long> row;               // floats per sample of boundary j = 0..kmax
    std::vector<std::vector<char>> need;      // need[rank][j]
    struct Xfer {
        int j, row0, rows;                    // boundary, first train row, rows
    };
    int kmax() const { return static_cast<int>(row.size()) - 1; }
    int shard_rows(int s) const { return shard_begin[static_cast<size_t>(s) + 1] - shard_begin[static_cast<size_t>(s)]; }
    // what src sends dst, in issue order (j ascending); empty for src == dst
    std::vector<Xfer> transfers(int src, int dst) const;
    size_t count(int src, int dst) const;     // floats
};

// blocks / owners: every distilled block with its owner rank; row: floats per
// sample of boundaries 0..max(blocks); shares as in shard_bounds
BoundaryPlan make_boundary_plan(const std::vector<int>& blocks, const std::vector<int>& owners,
                                const std::vector<long long>& row, int world, int n_train,
                                const std::vector<double>& share);

// shards proportional to `share` (rounded, contiguous, covering [0, n))
std::vector<int> shard_bounds(int n, const std::vector<double>& share);

}  // namespace pbkd_gpu
