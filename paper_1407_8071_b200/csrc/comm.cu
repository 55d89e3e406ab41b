// Multi-GPU estimate exchange: one NCCL communicator per bank process group,
// driven from the native bank loop (bank.cu) so a sharded run is still ONE
// host call per record.
//
// The reference's only parallelism is a fork pool over filters whose
// estimates are pickled back and averaged (ensemble.py:96-108).  Here each
// rank owns a contiguous block of global filter ids; after an observation's
// estimate kernels, the (M_total, width) fp64 row block of that observation -
// this rank's rows filled, every other row zero - is all-reduced (sum) on a
// side stream that waits on an event of the compute stream.  x + 0 is exact,
// so every rank receives the exact per-filter estimates and the left-to-right
// average is bit-identical for any GPU count (dist.py).  Nothing downstream
// of the estimate waits for the all-reduce, so it overlaps the next interval.
//
// NCCL is bound at run time (dlopen): the copy torch already loaded
// (libnccl.so.2, RTLD_NOLOAD) is preferred, so one NCCL lives in the process.
#include "common.cuh"

#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>

namespace pf {

namespace {

struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId *) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_reduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t,
                             ncclComm_t, cudaStream_t) = nullptr;
  const char *(*error_string)(ncclResult_t) = nullptr;
  ncclResult_t (*get_version)(int *) = nullptr;
  bool ok = false;
  std::string why;
};

NcclApi &nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_LOCAL);
    if (!h) {
      api.why = std::string("libnccl.so.2 not loadable: ") + dlerror();
      return;
    }
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    api.comm_init_rank =
        reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(dlsym(h, "ncclAllReduce"));
    api.error_string =
        reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
    api.get_version = reinterpret_cast<decltype(api.get_version)>(dlsym(h, "ncclGetVersion"));
    api.ok = api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.all_reduce &&
             api.error_string && api.get_version;
    if (!api.ok) api.why = "libnccl.so.2 lacks a required symbol";
  });
  return api;
}

}  // namespace

}  // namespace pf

struct pf_comm {
  ncclComm_t nccl = nullptr;
  cudaStream_t side = nullptr;  // the exchange stream
  cudaEvent_t ready = nullptr;  // compute stream -> side stream
  cudaEvent_t done = nullptr;   // side stream -> joining stream
  int nranks = 0, rank = 0, device = 0;
};

using namespace pf;

#define PF_NCCL(call, what)                                                          \
  do {                                                                               \
    ncclResult_t r_ = (call);                                                        \
    if (r_ != ncclSuccess) {                                                         \
      set_error("%s: NCCL error %d (%s)", what, static_cast<int>(r_),                \
                nccl().error_string ? nccl().error_string(r_) : "?");                \
      return PF_ECUDA;                                                               \
    }                                                                                \
  } while (0)

namespace pf {

// Issue the all-reduce (sum, in place) of `count` doubles at `buf` on the
// communicator's side stream, after everything enqueued so far on `s`.
int comm_allreduce_after(pf_comm *c, double *buf, int64_t count, cudaStream_t s) {
  if (count <= 0) return PF_OK;
  if (cudaEventRecord(c->ready, s) != cudaSuccess ||
      cudaStreamWaitEvent(c->side, c->ready, 0) != cudaSuccess)
    return check_launch("pf_comm: event");
  PF_NCCL(nccl().all_reduce(buf, buf, static_cast<size_t>(count), ncclFloat64, ncclSum, c->nccl,
                            c->side),
          "ncclAllReduce");
  return PF_OK;
}

}  // namespace pf

extern "C" {

int pf_comm_available(void) { return nccl().ok ? 1 : 0; }

int pf_comm_nccl_version(void) {
  int v = 0;
  if (nccl().ok) nccl().get_version(&v);
  return v;
}

int pf_comm_unique_id(uint8_t *id_out) {
  PF_REQUIRE(id_out, "pf_comm_unique_id: null");
  PF_REQUIRE(nccl().ok, "pf_comm_unique_id: %s", nccl().why.c_str());
  static_assert(sizeof(ncclUniqueId) == PF_COMM_ID_BYTES, "ncclUniqueId size");
  ncclUniqueId id;
  PF_NCCL(nccl().get_unique_id(&id), "ncclGetUniqueId");
  std::memcpy(id_out, &id, sizeof(id));
  return PF_OK;
}

int pf_comm_init(const uint8_t *id, int32_t nranks, int32_t rank, pf_comm **out) {
  PF_REQUIRE(id && out && nranks >= 1 && rank >= 0 && rank < nranks, "pf_comm_init: bad arguments");
  PF_REQUIRE(nccl().ok, "pf_comm_init: %s", nccl().why.c_str());
  *out = nullptr;
  auto *c = new pf_comm();
  c->nranks = nranks;
  c->rank = rank;
  cudaGetDevice(&c->device);
  ncclUniqueId uid;
  std::memcpy(&uid, id, sizeof(uid));
  ncclResult_t r = nccl().comm_init_rank(&c->nccl, nranks, uid, rank);
  if (r != ncclSuccess) {
    set_error("ncclCommInitRank(%d ranks, rank %d): %s", nranks, rank, nccl().error_string(r));
    delete c;
    return PF_ECUDA;
  }
  if (cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ready, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->done, cudaEventDisableTiming) != cudaSuccess) {
    nccl().comm_destroy(c->nccl);
    delete c;
    return check_launch("pf_comm_init: stream/event");
  }
  *out = c;
  return PF_OK;
}

int pf_comm_destroy(pf_comm *c) {
  if (!c) return PF_OK;
  cudaStreamSynchronize(c->side);
  if (c->nccl) nccl().comm_destroy(c->nccl);
  if (c->ready) cudaEventDestroy(c->ready);
  if (c->done) cudaEventDestroy(c->done);
  if (c->side) cudaStreamDestroy(c->side);
  delete c;
  return PF_OK;
}

int pf_comm_allreduce_f64(pf_comm *c, double *buf, int64_t count, void *stream) {
  PF_REQUIRE(c && (buf || count == 0) && count >= 0, "pf_comm_allreduce_f64: bad arguments");
  const int rc = comm_allreduce_after(c, buf, count, as_stream(stream));
  if (rc != PF_OK) return rc;
  return pf_comm_join(c, stream);
}

int pf_comm_exchange_steps(pf_comm *c, double *est, int64_t step_stride, int64_t count,
                           int32_t k0, int32_t n_steps, void *stream) {
  PF_REQUIRE(c && est && count >= 0 && k0 >= 0 && n_steps >= 0 && step_stride >= count,
             "pf_comm_exchange_steps: bad arguments");
  for (int32_t i = 0; i < n_steps; ++i) {
    const int rc = comm_allreduce_after(c, est + static_cast<int64_t>(k0 + i) * step_stride,
                                        count, as_stream(stream));
    if (rc != PF_OK) return rc;
  }
  return PF_OK;
}

int pf_comm_join(pf_comm *c, void *stream) {
  PF_REQUIRE(c, "pf_comm_join: null");
  if (cudaEventRecord(c->done, c->side) != cudaSuccess ||
      cudaStreamWaitEvent(as_stream(stream), c->done, 0) != cudaSuccess)
    return check_launch("pf_comm_join");
  return PF_OK;
}

}  // extern "C"
