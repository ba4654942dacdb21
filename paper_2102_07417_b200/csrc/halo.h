// Multi-GPU plumbing of libamgb200 (one process per GPU): NCCL loaded with
// dlopen (the process may already hold torch's bundled libnccl; single-GPU
// use never touches NCCL), per-matrix halo plans produced by the host planner
// (paper_2102_07417_b200/partition.py), and the exchange: a pack kernel
// gathers the owned entries each peer needs, then one grouped
// ncclSend / ncclRecv per peer receives straight into the halo segment of
// the input vector.  Everything is enqueued on the handle's stream, so it is
// captured into the PCG iteration graph with the kernels.
#pragma once
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>
#include <stdint.h>
#include <stdlib.h>

#include <string>
#include <vector>

namespace amg {

struct NcclApi {
    bool loaded = false;
    void *lib = nullptr;
    decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
    decltype(&ncclCommInitRank) CommInitRank = nullptr;
    decltype(&ncclCommDestroy) CommDestroy = nullptr;
    decltype(&ncclGetErrorString) GetErrorString = nullptr;
    decltype(&ncclGroupStart) GroupStart = nullptr;
    decltype(&ncclGroupEnd) GroupEnd = nullptr;
    decltype(&ncclSend) Send = nullptr;
    decltype(&ncclRecv) Recv = nullptr;
    decltype(&ncclAllGather) AllGather = nullptr;
    decltype(&ncclBroadcast) Broadcast = nullptr;
};

inline std::string &halo_err_ref()
{
    static thread_local std::string e;
    return e;
}
inline const std::string &halo_error() { return halo_err_ref(); }

inline NcclApi &nccl()
{
    static NcclApi api;
    if (api.loaded) return api;
    // AMGB200_NCCL: an explicit library (the Python shim points it at the NCCL
    // that torch ships, so both share one NCCL build); else the loader's choice
    const char *env = getenv("AMGB200_NCCL");
    if (env && *env) api.lib = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
    const char *names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char *n : names) {
        if (api.lib) break;
        api.lib = dlopen(n, RTLD_NOW | RTLD_GLOBAL);
    }
    if (!api.lib) return api;
#define AMG_SYM(F) api.F = reinterpret_cast<decltype(api.F)>(dlsym(api.lib, "nccl" #F))
    AMG_SYM(GetUniqueId);
    AMG_SYM(CommInitRank);
    AMG_SYM(CommDestroy);
    AMG_SYM(GetErrorString);
    AMG_SYM(GroupStart);
    AMG_SYM(GroupEnd);
    AMG_SYM(Send);
    AMG_SYM(Recv);
    AMG_SYM(AllGather);
    AMG_SYM(Broadcast);
#undef AMG_SYM
    api.loaded = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.GroupStart && api.GroupEnd &&
                 api.Send && api.Recv && api.AllGather && api.Broadcast && api.GetErrorString;
    return api;
}

struct Comm {
    ncclComm_t comm = nullptr;
    int rank = 0, nranks = 1;
};

struct HaloPlan {
    int64_t n_own = 0, n_halo = 0;
    std::vector<int> recv_peers, send_peers;
    std::vector<int64_t> recv_counts, send_counts, send_displ;
    int32_t *send_idx = nullptr;  // device, concatenated per send peer
    double *send_buf = nullptr;   // device
    int64_t n_send = 0;
    bool empty() const { return recv_peers.empty() && send_peers.empty(); }
};

#define AMG_NCCL_OK(call, what)                                                                     \
    do {                                                                                            \
        ncclResult_t r_ = (call);                                                                   \
        if (r_ != ncclSuccess) {                                                                    \
            halo_err_ref() = std::string(what) + ": " + nccl().GetErrorString(r_);                  \
            return 1;                                                                               \
        }                                                                                           \
    } while (0)

inline int comm_init(Comm &c, const void *uid, int rank, int nranks)
{
    c.rank = rank;
    c.nranks = nranks;
    if (nranks == 1) return 0;
    NcclApi &api = nccl();
    if (!api.loaded) {
        halo_err_ref() = "libnccl.so.2 could not be loaded (multi-GPU needs NCCL)";
        return 1;
    }
    ncclUniqueId id;
    memcpy(&id, uid, sizeof(id));
    AMG_NCCL_OK(api.CommInitRank(&c.comm, nranks, id, rank), "ncclCommInitRank");
    return 0;
}

inline void comm_destroy(Comm &c)
{
    if (c.comm) nccl().CommDestroy(c.comm);
    c.comm = nullptr;
}

inline void halo_free(HaloPlan &p)
{
    if (p.send_idx) cudaFree(p.send_idx);
    if (p.send_buf) cudaFree(p.send_buf);
    p.send_idx = nullptr;
    p.send_buf = nullptr;
}

}  // namespace amg
