// NCCL-aware entry points of the C ABI (SURVEY.md 8(b) `alto_mttkrp_sharded`,
// 8(e) sharding): communicator setup and the collectives of the sharded
// MTTKRP / Phi / CP-ALS update, plus the sharded MTTKRP itself (this rank's
// ALTO-ordered shard -> factor-sized partial -> summed over the ranks).
//
// The reference is single-process (pkg/src/alto/kernels.py:130-142 fans out
// over threads and sums nothing across processes), so there is no reference
// interface to mirror beyond the summed result: rank r's shard is
// [bounds[r], bounds[r+1]) of balanced_bounds(M, W) (partition.py:69-75) and
// the sum of the shards' partials equals the single-process MTTKRP up to the
// order of the fp64 additions.
//
// NCCL is resolved at run time (dlopen of libnccl.so.2, reusing the copy
// torch.distributed already loaded in the process when there is one), so the
// library loads on hosts without NCCL and the symbols below then report
// ALTO_ERR_UNSUPPORTED. Every collective is enqueued on the caller's stream
// (capturable in CUDA graphs); failures and asynchronous communicator errors
// map to ALTO_ERR_CUDA (RuntimeError in the Python shim).
#include <dlfcn.h>
#include <nccl.h>
#include <string.h>

#include <mutex>

#include "alto_common.cuh"

namespace alto {
namespace {

struct NcclApi {
  bool tried = false, ok = false;
  ncclResult_t (*get_unique_id)(ncclUniqueId *) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*comm_abort)(ncclComm_t) = nullptr;
  ncclResult_t (*comm_async_error)(ncclComm_t, ncclResult_t *) = nullptr;
  ncclResult_t (*all_reduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*reduce_scatter)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                 cudaStream_t) = nullptr;
  ncclResult_t (*all_gather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*comm_count)(const ncclComm_t, int *) = nullptr;
  ncclResult_t (*comm_user_rank)(const ncclComm_t, int *) = nullptr;
  const char *(*error_string)(ncclResult_t) = nullptr;
  ncclResult_t (*get_version)(int *) = nullptr;
};

NcclApi g_nccl;
std::mutex g_nccl_mu;

template <class F>
bool bind(void *h, const char *name, F &fn) {
  fn = reinterpret_cast<F>(dlsym(h, name));
  return fn != nullptr;
}

const NcclApi *nccl() {
  std::lock_guard<std::mutex> lk(g_nccl_mu);
  if (g_nccl.tried) return g_nccl.ok ? &g_nccl : nullptr;
  g_nccl.tried = true;
  // the process's NCCL first (torch.distributed's), then the loader's path
  void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
  if (h == nullptr) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
  if (h == nullptr) h = dlopen("libnccl.so", RTLD_NOW | RTLD_LOCAL);
  if (h == nullptr) return nullptr;
  NcclApi &a = g_nccl;
  a.ok = bind(h, "ncclGetUniqueId", a.get_unique_id) && bind(h, "ncclCommInitRank", a.comm_init_rank) &&
         bind(h, "ncclCommDestroy", a.comm_destroy) && bind(h, "ncclCommAbort", a.comm_abort) &&
         bind(h, "ncclCommGetAsyncError", a.comm_async_error) && bind(h, "ncclAllReduce", a.all_reduce) &&
         bind(h, "ncclReduceScatter", a.reduce_scatter) && bind(h, "ncclAllGather", a.all_gather) &&
         bind(h, "ncclCommCount", a.comm_count) && bind(h, "ncclCommUserRank", a.comm_user_rank) &&
         bind(h, "ncclGetErrorString", a.error_string) && bind(h, "ncclGetVersion", a.get_version);
  return a.ok ? &g_nccl : nullptr;
}

int nccl_status(const NcclApi *a, ncclResult_t r, const char *what) {
  if (r == ncclSuccess) return ALTO_OK;
  set_error("%s: NCCL error %d (%s)", what, (int)r, a->error_string(r));
  return r == ncclInvalidArgument ? ALTO_ERR_VALUE : ALTO_ERR_CUDA;
}

#define ALTO_NCCL_API(a)                                                                         \
  const NcclApi *a = nccl();                                                                     \
  ALTO_REQUIRE(a != nullptr, ALTO_ERR_UNSUPPORTED, "NCCL (libnccl.so.2) is not available here")

#define ALTO_NCCL(a, call, what)                     \
  do {                                               \
    int _rc = nccl_status(a, (call), what);          \
    if (_rc) return _rc;                             \
  } while (0)

}  // namespace
}  // namespace alto

using namespace alto;

extern "C" {

int alto_nccl_version(int32_t *host_version) {
  ALTO_REQUIRE(host_version != nullptr, ALTO_ERR_VALUE, "null output");
  *host_version = 0;
  ALTO_NCCL_API(a);
  int v = 0;
  ALTO_NCCL(a, a->get_version(&v), "ncclGetVersion");
  *host_version = v;
  return ALTO_OK;
}

int alto_nccl_unique_id(uint8_t *host_id, int64_t host_len) {
  ALTO_REQUIRE(host_id != nullptr && host_len >= (int64_t)sizeof(ncclUniqueId), ALTO_ERR_VALUE,
               "the unique id needs %d bytes", (int)sizeof(ncclUniqueId));
  ALTO_NCCL_API(a);
  ncclUniqueId id;
  ALTO_NCCL(a, a->get_unique_id(&id), "ncclGetUniqueId");
  memcpy(host_id, &id, sizeof(id));
  return ALTO_OK;
}

int alto_nccl_comm_init(const uint8_t *host_id, int64_t host_len, int32_t world, int32_t rank, void **host_comm) {
  ALTO_REQUIRE(host_id != nullptr && host_len >= (int64_t)sizeof(ncclUniqueId), ALTO_ERR_VALUE,
               "the unique id needs %d bytes", (int)sizeof(ncclUniqueId));
  ALTO_REQUIRE(host_comm != nullptr, ALTO_ERR_VALUE, "null communicator output");
  ALTO_REQUIRE(world >= 1 && rank >= 0 && rank < world, ALTO_ERR_VALUE, "rank %d outside a world of %d", rank,
               world);
  ALTO_NCCL_API(a);
  ncclUniqueId id;
  memcpy(&id, host_id, sizeof(id));
  ncclComm_t c = nullptr;
  ALTO_NCCL(a, a->comm_init_rank(&c, world, id, rank), "ncclCommInitRank");
  *host_comm = c;
  return ALTO_OK;
}

int alto_nccl_comm_destroy(void *comm, int32_t abort) {
  if (comm == nullptr) return ALTO_OK;
  ALTO_NCCL_API(a);
  ncclComm_t c = static_cast<ncclComm_t>(comm);
  ALTO_NCCL(a, abort ? a->comm_abort(c) : a->comm_destroy(c), abort ? "ncclCommAbort" : "ncclCommDestroy");
  return ALTO_OK;
}

int alto_nccl_comm_info(void *comm, int32_t *host_world, int32_t *host_rank) {
  ALTO_REQUIRE(comm != nullptr && host_world != nullptr && host_rank != nullptr, ALTO_ERR_VALUE, "null argument");
  ALTO_NCCL_API(a);
  int w = 0, r = 0;
  ncclComm_t c = static_cast<ncclComm_t>(comm);
  ALTO_NCCL(a, a->comm_count(c, &w), "ncclCommCount");
  ALTO_NCCL(a, a->comm_user_rank(c, &r), "ncclCommUserRank");
  *host_world = w;
  *host_rank = r;
  return ALTO_OK;
}

int alto_nccl_check(void *comm) {
  ALTO_REQUIRE(comm != nullptr, ALTO_ERR_VALUE, "null communicator");
  ALTO_NCCL_API(a);
  ncclResult_t e = ncclSuccess;
  ALTO_NCCL(a, a->comm_async_error(static_cast<ncclComm_t>(comm), &e), "ncclCommGetAsyncError");
  ALTO_NCCL(a, e, "asynchronous communicator error");
  return ALTO_OK;
}

int alto_nccl_allreduce_f64(double *buf, int64_t count, void *comm, void *stream) {
  ALTO_REQUIRE(comm != nullptr && count >= 0, ALTO_ERR_VALUE, "bad all-reduce arguments");
  ALTO_NCCL_API(a);
  if (count == 0) return ALTO_OK;
  ALTO_NCCL(a,
            a->all_reduce(buf, buf, (size_t)count, ncclFloat64, ncclSum, static_cast<ncclComm_t>(comm),
                          static_cast<cudaStream_t>(stream)),
            "ncclAllReduce");
  return ALTO_OK;
}

int alto_nccl_reduce_scatter_f64(const double *send, double *recv, int64_t recvcount, void *comm, void *stream) {
  ALTO_REQUIRE(comm != nullptr && recvcount >= 0, ALTO_ERR_VALUE, "bad reduce-scatter arguments");
  ALTO_NCCL_API(a);
  if (recvcount == 0) return ALTO_OK;
  ALTO_NCCL(a,
            a->reduce_scatter(send, recv, (size_t)recvcount, ncclFloat64, ncclSum, static_cast<ncclComm_t>(comm),
                              static_cast<cudaStream_t>(stream)),
            "ncclReduceScatter");
  return ALTO_OK;
}

int alto_nccl_allgather_f64(const double *send, double *recv, int64_t sendcount, void *comm, void *stream) {
  ALTO_REQUIRE(comm != nullptr && sendcount >= 0, ALTO_ERR_VALUE, "bad all-gather arguments");
  ALTO_NCCL_API(a);
  if (sendcount == 0) return ALTO_OK;
  ALTO_NCCL(a,
            a->all_gather(send, recv, (size_t)sendcount, ncclFloat64, static_cast<ncclComm_t>(comm),
                          static_cast<cudaStream_t>(stream)),
            "ncclAllGather");
  return ALTO_OK;
}

int alto_mttkrp_sharded(const alto_layout_t *host_layout, const void *keys, const double *vals, int64_t M,
                        const alto_factors_t *host_factors, int32_t mode, double *out, int64_t ldo, int64_t rows,
                        const int64_t *bounds, const int64_t *lo, int32_t L, int64_t acc_rows, int32_t privatize,
                        int32_t owner_rows, void *comm, void *stream) {
  ALTO_REQUIRE(host_layout != nullptr && host_factors != nullptr, ALTO_ERR_VALUE, "null layout or factors");
  ALTO_REQUIRE(mode >= 0 && mode < host_layout->nmodes, ALTO_ERR_INDEX, "mode %d out of range", mode);
  ALTO_REQUIRE(rows == host_layout->dims[mode], ALTO_ERR_VALUE, "rows must equal the mode's dimension");
  ALTO_REQUIRE(ldo >= host_factors->rank, ALTO_ERR_VALUE, "ldo < rank");
  ALTO_REQUIRE(comm != nullptr, ALTO_ERR_VALUE, "null communicator");
  ALTO_NCCL_API(a);
  int world = 0, me = 0;
  ALTO_NCCL(a, a->comm_count(static_cast<ncclComm_t>(comm), &world), "ncclCommCount");
  ALTO_NCCL(a, a->comm_user_rank(static_cast<ncclComm_t>(comm), &me), "ncclCommUserRank");
  const int64_t chunk = (rows + world - 1) / world;
  const int64_t prow = owner_rows ? chunk * world : rows;  // rows of `out` (padded for the row owners)
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  ALTO_CUDA(cudaMemsetAsync(out, 0, (size_t)prow * ldo * sizeof(double), st));
  int rc;
  if (bounds != nullptr)
    rc = alto_mttkrp_segment(host_layout, keys, vals, M, host_factors, mode, out, ldo, bounds, lo, L, acc_rows,
                             privatize, stream);
  else
    rc = alto_mttkrp_stream(host_layout, keys, vals, M, host_factors, mode, out, ldo, ALTO_ALGO_ATOMIC, nullptr,
                            nullptr, 0, stream);
  if (rc) return rc;
  if (owner_rows) {
    // in place: rank r's block is out + r * chunk * ldo (NCCL's in-place rule)
    double *blk = out + (int64_t)me * chunk * ldo;
    return alto_nccl_reduce_scatter_f64(out, blk, chunk * ldo, comm, stream);
  }
  return alto_nccl_allreduce_f64(out, rows * ldo, comm, stream);
}

}  // extern "C"
