// comm.cu -- NCCL inside the engine handle: the
// multi-GPU exchanges of a sharded batch run as NCCL collectives on the
// engine's stream, on device buffers, with no Python in the loop.
//
//   phase bookkeeping   a few hundred bytes per phase (max rounds, summed
//                       updates / edges / warnings / frontier flags / eligible
//                       counts, max |delta|): ncclAllReduce, grouped
//   label migration     components that changed owner: ncclAllReduce(max) of
//                       the migrated rows, non-owners contributing -inf
//                       (bit-exact: max picks the owner's value)
//   row partition       per global round: ncclAllGather of the round's packed
//                       evaluated rows (vertex, masks, C label words) straight
//                       from and into device buffers, then k_rows_apply
//
// libnccl is opened at run time (dlopen "libnccl.so.2": the copy torch
// already mapped, else the system one), so a single-GPU user never needs it.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <vector>

#include "engine.cuh"

namespace dlp {

namespace {

struct NcclApi {
    void* h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi& api() {
    static NcclApi a;
    return a;
}

bool load_nccl(std::string* err) {
    NcclApi& a = api();
    if (a.h) return true;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
        *err = std::string("cannot open libnccl.so.2: ") + dlerror();
        return false;
    }
#define DLP_SYM(name, field)                                        \
    a.field = reinterpret_cast<decltype(a.field)>(dlsym(h, name));  \
    if (!a.field) {                                                 \
        *err = std::string("libnccl.so.2 lacks ") + name;           \
        return false;                                               \
    }
    DLP_SYM("ncclGetUniqueId", GetUniqueId)
    DLP_SYM("ncclCommInitRank", CommInitRank)
    DLP_SYM("ncclCommDestroy", CommDestroy)
    DLP_SYM("ncclAllReduce", AllReduce)
    DLP_SYM("ncclAllGather", AllGather)
    DLP_SYM("ncclGroupStart", GroupStart)
    DLP_SYM("ncclGroupEnd", GroupEnd)
    DLP_SYM("ncclGetErrorString", GetErrorString)
#undef DLP_SYM
    a.h = h;
    return true;
}

struct NcclFailure {};

void nccl_try(ncclResult_t r, Engine& E, const char* what) {
    if (r != ncclSuccess) {
        E.err = std::string(what) + ": " + api().GetErrorString(r);
        throw NcclFailure{};
    }
}

}  // namespace

int nccl_unique_id(void* out, std::string* err) {
    if (!load_nccl(err)) return DLP_EINTERNAL;
    ncclUniqueId id;
    ncclResult_t r = api().GetUniqueId(&id);
    if (r != ncclSuccess) {
        *err = std::string("ncclGetUniqueId: ") + api().GetErrorString(r);
        return DLP_EINTERNAL;
    }
    memcpy(out, &id, sizeof(id));
    return DLP_OK;
}

int nccl_attach(Engine& E, const void* id, int world, int rank) {
    std::string err;
    if (!load_nccl(&err)) {
        E.err = err;
        return DLP_EINTERNAL;
    }
    ncclUniqueId uid;
    memcpy(&uid, id, sizeof(uid));
    ncclComm_t comm = nullptr;
    ncclResult_t r = api().CommInitRank(&comm, world, uid, rank);
    if (r != ncclSuccess) {
        E.err = std::string("ncclCommInitRank: ") + api().GetErrorString(r);
        return DLP_EINTERNAL;
    }
    E.nccl = comm;
    E.shard_rank = rank;
    E.shard_world = world;
    return DLP_OK;
}

void nccl_detach(Engine& E) {
    if (E.nccl && api().h) api().CommDestroy((ncclComm_t)E.nccl);
    E.nccl = nullptr;
}

// The engine's reduction (dlp_allreduce_fn shape) over NCCL: the three host
// arrays travel in one device buffer, three grouped all-reduces, one copy
// back.  ctx = the Engine.
int nccl_reduce(void* ctx, int64_t* imax, int32_t nimax, int64_t* isum, int32_t nisum, double* dmax,
                int32_t ndmax) {
    Engine& E = *static_cast<Engine*>(ctx);
    try {
        const size_t n = (size_t)nimax + nisum + ndmax;
        E.comm_buf.reserve(n + 1, 0, E.st);
        unsigned long long* d = E.comm_buf.p;
        std::vector<unsigned long long> h(n);
        memcpy(h.data(), imax, nimax * 8);
        memcpy(h.data() + nimax, isum, nisum * 8);
        memcpy(h.data() + nimax + nisum, dmax, ndmax * 8);
        DLP_CUDA_TRY(cudaMemcpyAsync(d, h.data(), n * 8, cudaMemcpyHostToDevice, E.st));
        ncclComm_t c = (ncclComm_t)E.nccl;
        nccl_try(api().GroupStart(), E, "ncclGroupStart");
        if (nimax) nccl_try(api().AllReduce(d, d, nimax, ncclInt64, ncclMax, c, E.st), E, "ncclAllReduce");
        if (nisum)
            nccl_try(api().AllReduce(d + nimax, d + nimax, nisum, ncclInt64, ncclSum, c, E.st), E, "ncclAllReduce");
        if (ndmax)
            nccl_try(api().AllReduce(d + nimax + nisum, d + nimax + nisum, ndmax, ncclFloat64, ncclMax, c, E.st), E,
                     "ncclAllReduce");
        nccl_try(api().GroupEnd(), E, "ncclGroupEnd");
        DLP_CUDA_TRY(cudaMemcpyAsync(h.data(), d, n * 8, cudaMemcpyDeviceToHost, E.st));
        DLP_CUDA_TRY(cudaStreamSynchronize(E.st));
        memcpy(imax, h.data(), nimax * 8);
        memcpy(isum, h.data() + nimax, nisum * 8);
        memcpy(dmax, h.data() + nimax + nisum, ndmax * 8);
    } catch (const NcclFailure&) {
        return 1;
    } catch (const CudaFailure& f) {
        E.err = std::string("CUDA error in the NCCL reduction: ") + cudaGetErrorString(f.err) + " (" + f.expr + ")";
        return 1;
    }
    return 0;
}

// Device-resident max-reduction of a device array (label migration).
int nccl_max_f64(Engine& E, double* d, size_t n) {
    try {
        nccl_try(api().AllReduce(d, d, n, ncclFloat64, ncclMax, (ncclComm_t)E.nccl, E.st), E, "ncclAllReduce");
    } catch (const NcclFailure&) {
        return 1;
    }
    return 0;
}

// All-gather of `count` 8-byte words per rank, device to device.
int nccl_allgather_u64(Engine& E, const unsigned long long* send, unsigned long long* recv, size_t count) {
    try {
        nccl_try(api().AllGather(send, recv, count, ncclUint64, (ncclComm_t)E.nccl, E.st), E, "ncclAllGather");
    } catch (const NcclFailure&) {
        return 1;
    }
    return 0;
}

}  // namespace dlp
