// Multi-GPU plumbing of libamgb200 (one process per GPU): the NCCL
// communicator and per-matrix halo plans.  Single-GPU builds never touch
// NCCL; nranks > 1 is wired in a later pass.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

namespace amg {

struct Comm {
    void *nccl = nullptr;  // ncclComm_t
    int rank = 0, nranks = 1;
};

struct HaloPlan {
    int64_t n_halo = 0;
    bool empty() const { return n_halo == 0; }
};

inline std::string &halo_err_ref()
{
    static thread_local std::string e;
    return e;
}
inline const std::string &halo_error() { return halo_err_ref(); }

inline int comm_init(Comm &c, const void *, int rank, int nranks)
{
    c.rank = rank;
    c.nranks = nranks;
    halo_err_ref() = "multi-GPU (nranks > 1) is not available in this build";
    return nranks > 1 ? 1 : 0;
}
inline void comm_destroy(Comm &) {}
inline void halo_free(HaloPlan &) {}
inline int halo_exchange(Comm &, const HaloPlan &, double *, cudaStream_t) { return 0; }

}  // namespace amg
