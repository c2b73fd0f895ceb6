// NCCL mode of the multi-GPU x-slab layer behind the C ABI, for hosts that
// do not go through torch.distributed.  The same exchange
// DistributedSimulation performs with torch.distributed / NCCL
// (parallel.py SlabExchange), as plain entry points over an NCCL
// communicator:
//
//   * vpfv_halo_exchange_x -- the reference cluster's ghost exchange
//     (Exchanger, /root/reference/pkg/src/vpfv/partition.py:679-724) for an
//     x-slab layout: x is the slowest dim, so each side is one contiguous run
//     of 3 padded planes; the ranks form a periodic ring in x;
//   * vpfv_density_allgather -- every slab's density rows to every rank
//     (runner.py:336-392: one global field solve, replicated);
//   * vpfv_flag_allreduce -- the step's divergence verdict (max over ranks,
//     runner.py:453-464).
//
// All calls are stream-ordered and graph-capturable (NCCL >= 2.9); the
// communicator is an opaque pointer.  libnccl.so.2 is opened by soname on
// the first call (dlopen), not linked: inside a PyTorch process that is the
// NCCL torch already loaded, and loading libvpfv.so never pins a different
// NCCL under torch's feet.
#include <dlfcn.h>
#include <nccl.h>
#include <stdio.h>
#include <string.h>

#include "common.cuh"

using vpfv::NG;

namespace {

struct Nccl {
    decltype(&ncclGetUniqueId) GetUniqueId;
    decltype(&ncclCommInitRank) CommInitRank;
    decltype(&ncclCommDestroy) CommDestroy;
    decltype(&ncclCommCount) CommCount;
    decltype(&ncclCommUserRank) CommUserRank;
    decltype(&ncclGroupStart) GroupStart;
    decltype(&ncclGroupEnd) GroupEnd;
    decltype(&ncclSend) Send;
    decltype(&ncclRecv) Recv;
    decltype(&ncclAllGather) AllGather;
    decltype(&ncclAllReduce) AllReduce;
    decltype(&ncclGetErrorString) GetErrorString;
    bool ok = false;
};

const Nccl *nccl() {
    static Nccl n;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL | RTLD_NOLOAD);  // torch's, if loaded
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return nullptr;
#define VPFV_SYM(f) n.f = (decltype(n.f))dlsym(h, "nccl" #f)
        VPFV_SYM(GetUniqueId);
        VPFV_SYM(CommInitRank);
        VPFV_SYM(CommDestroy);
        VPFV_SYM(CommCount);
        VPFV_SYM(CommUserRank);
        VPFV_SYM(GroupStart);
        VPFV_SYM(GroupEnd);
        VPFV_SYM(Send);
        VPFV_SYM(Recv);
        VPFV_SYM(AllGather);
        VPFV_SYM(AllReduce);
        VPFV_SYM(GetErrorString);
#undef VPFV_SYM
        n.ok = n.GetUniqueId && n.CommInitRank && n.CommDestroy && n.CommCount && n.CommUserRank && n.GroupStart &&
               n.GroupEnd && n.Send && n.Recv && n.AllGather && n.AllReduce && n.GetErrorString;
    }
    return n.ok ? &n : nullptr;
}

int nccl_err(ncclResult_t r, const char *what) {
    char buf[200];
    snprintf(buf, sizeof buf, "%s: %s", what, nccl()->GetErrorString(r));
    return vpfv::set_error(VPFV_ENCCL, buf);
}

#define NCCL_OR_FAIL(what)                                                          \
    const Nccl *N_ = nccl();                                                        \
    if (!N_) return vpfv::set_error(VPFV_ENCCL, what ": libnccl.so.2 not available")

}  // namespace

extern "C" int vpfv_comm_id_size(void) { return (int)sizeof(ncclUniqueId); }

extern "C" int vpfv_comm_unique_id(unsigned char *id_out) {
    NCCL_OR_FAIL("comm_unique_id");
    ncclUniqueId id;
    ncclResult_t r = N_->GetUniqueId(&id);
    if (r != ncclSuccess) return nccl_err(r, "comm_unique_id");
    memcpy(id_out, &id, sizeof id);
    return VPFV_OK;
}

extern "C" int vpfv_comm_init(void **comm_out, int world, int rank, const unsigned char *id, int device) {
    if (!comm_out || world < 1 || rank < 0 || rank >= world || !id)
        return vpfv::set_error(VPFV_EARG, "comm_init: bad arguments");
    NCCL_OR_FAIL("comm_init");
    if (cudaSetDevice(device) != cudaSuccess) return vpfv::set_error(VPFV_ECUDA, "comm_init: cudaSetDevice");
    ncclUniqueId uid;
    memcpy(&uid, id, sizeof uid);
    ncclComm_t c;
    ncclResult_t r = N_->CommInitRank(&c, world, uid, rank);
    if (r != ncclSuccess) return nccl_err(r, "comm_init");
    *comm_out = c;
    return VPFV_OK;
}

extern "C" int vpfv_comm_destroy(void *comm) {
    if (!comm) return VPFV_OK;
    NCCL_OR_FAIL("comm_destroy");
    ncclResult_t r = N_->CommDestroy((ncclComm_t)comm);
    return r == ncclSuccess ? VPFV_OK : nccl_err(r, "comm_destroy");
}

extern "C" int vpfv_halo_exchange_x(void *comm, double *f, int ndim, const int *N, void *stream) {
    if (!comm || !f || ndim < 2 || ndim > 4 || N[0] < NG) return vpfv::set_error(VPFV_EARG, "halo_exchange_x: bad arguments");
    NCCL_OR_FAIL("halo_exchange_x");
    ncclComm_t c = (ncclComm_t)comm;
    int world = 0, rank = 0;
    N_->CommCount(c, &world);
    N_->CommUserRank(c, &rank);
    size_t plane = 1;
    for (int k = 1; k < ndim; ++k) plane *= (size_t)(N[k] + 2 * NG);
    const size_t n = NG * plane;
    const int lo = (rank + world - 1) % world, hi = (rank + 1) % world;
    cudaStream_t s = (cudaStream_t)stream;
    ncclResult_t r = N_->GroupStart();
    // my first 3 interior planes -> the low neighbour's high ghosts; my last 3 -> the high neighbour's low ghosts
    if (r == ncclSuccess) r = N_->Send(f + NG * plane, n, ncclDouble, lo, c, s);
    if (r == ncclSuccess) r = N_->Send(f + (size_t)N[0] * plane, n, ncclDouble, hi, c, s);
    if (r == ncclSuccess) r = N_->Recv(f + (size_t)(N[0] + NG) * plane, n, ncclDouble, hi, c, s);
    if (r == ncclSuccess) r = N_->Recv(f, n, ncclDouble, lo, c, s);
    ncclResult_t e = N_->GroupEnd();
    if (r != ncclSuccess) return nccl_err(r, "halo_exchange_x");
    return e == ncclSuccess ? VPFV_OK : nccl_err(e, "halo_exchange_x");
}

extern "C" int vpfv_density_allgather(void *comm, const double *n_local, double *n, long long count, void *stream) {
    if (!comm || !n_local || !n || count < 0) return vpfv::set_error(VPFV_EARG, "density_allgather: bad arguments");
    NCCL_OR_FAIL("density_allgather");
    ncclResult_t r = N_->AllGather(n_local, n, (size_t)count, ncclDouble, (ncclComm_t)comm, (cudaStream_t)stream);
    return r == ncclSuccess ? VPFV_OK : nccl_err(r, "density_allgather");
}

extern "C" int vpfv_flag_allreduce(void *comm, long long *flag, void *stream) {
    if (!comm || !flag) return vpfv::set_error(VPFV_EARG, "flag_allreduce: bad arguments");
    NCCL_OR_FAIL("flag_allreduce");
    ncclResult_t r = N_->AllReduce(flag, flag, 1, ncclInt64, ncclMax, (ncclComm_t)comm, (cudaStream_t)stream);
    return r == ncclSuccess ? VPFV_OK : nccl_err(r, "flag_allreduce");
}
