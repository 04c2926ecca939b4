// rowpart.cu — row-partitioned multi-GPU SpMV / SpMM through the C-ABI
// (the `sfg_rowpart_spmm(..., ncclComm_t, ..., gather)` entry
// of §8b).
//
// One process per GPU. Rank r holds the nnz-balanced row block
// [bounds[r], bounds[r+1]) of A (sfg_row_partition + sfg_coo_slice_rows,
// then its own conversion) and a replica of x / B. The product lands
// directly in rank r's chunk of a padded output buffer of P equal chunks,
// and one in-place NCCL all-gather over NVLink / NVSwitch completes the
// output on every rank — the path's only exchange. Rows past the block in
// a rank's chunk are padding.
//
// NCCL is resolved at run time (dlopen / dlsym): the copy the process has
// already loaded (PyTorch's) is preferred, so a communicator created here
// and torch.distributed's live in the same NCCL; otherwise libnccl.so.2
// from the library path. nccl.h supplies only the (stable) types.
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>

#include "internal.cuh"

namespace sfg {

namespace {

struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  std::string load_error;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char* e = dlerror();
      api.load_error = std::string("cannot load libnccl.so.2: ") + (e ? e : "?");
      return;
    }
    auto sym = [&](const char* name) {
      void* p = dlsym(h, name);
      if (!p) api.load_error = std::string("libnccl.so.2 lacks ") + name;
      return p;
    };
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(sym("ncclGetUniqueId"));
    api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(sym("ncclCommInitRank"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(sym("ncclCommDestroy"));
    api.all_gather = reinterpret_cast<decltype(api.all_gather)>(sym("ncclAllGather"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(sym("ncclGetErrorString"));
  });
  if (!api.load_error.empty()) raise(SFG_ERR_NCCL, api.load_error);
  return api;
}

void check(ncclResult_t r, const char* what) {
  if (r != ncclSuccess) raise(SFG_ERR_NCCL, std::string(what) + ": " + nccl().error_string(r));
}

}  // namespace

}  // namespace sfg

struct sfg_comm {
  ncclComm_t comm = nullptr;
  int32_t nranks = 0;
  int32_t rank = 0;
};

namespace sfg {

void comm_unique_id(uint8_t* out) {
  static_assert(sizeof(ncclUniqueId) == SFG_COMM_ID_BYTES, "ncclUniqueId size");
  ncclUniqueId id;
  check(nccl().get_unique_id(&id), "ncclGetUniqueId");
  std::memcpy(out, &id, sizeof id);
}

sfg_comm* comm_create(sfg_context* ctx, int32_t nranks, int32_t rank, const uint8_t* id_bytes) {
  ncclUniqueId id;
  std::memcpy(&id, id_bytes, sizeof id);
  SFG_CUDA(cudaSetDevice(ctx->device));
  auto* c = new sfg_comm;
  c->nranks = nranks;
  c->rank = rank;
  ncclResult_t r = nccl().comm_init_rank(&c->comm, nranks, id, rank);
  if (r != ncclSuccess) {
    delete c;
    check(r, "ncclCommInitRank");
  }
  return c;
}

void comm_destroy(sfg_comm* c) {
  if (c->comm) nccl().comm_destroy(c->comm);
  delete c;
}

// In place: rank r's chunk is buf[r * chunk_elems, (r + 1) * chunk_elems).
void allgather_chunks(sfg_context* ctx, sfg_comm* c, float* buf, int64_t chunk_elems) {
  if (chunk_elems == 0) return;  // one rank too: the same NCCL call (a no-op copy)
  check(nccl().all_gather(buf + (int64_t)c->rank * chunk_elems, buf, (size_t)chunk_elems, ncclFloat32, c->comm,
                          ctx->stream),
        "ncclAllGather");
}

void rowpart_spmv(sfg_context* ctx, sfg_comm* c, const sfg_tensor* a, const float* x, float* y,
                  int64_t chunk_rows, bool gather) {
  if (a->m > chunk_rows) raise(SFG_ERR_INVALID_OPERATION, "row block larger than the chunk");
  spmv(ctx, a, x, y + (int64_t)c->rank * chunk_rows, false);
  if (gather) allgather_chunks(ctx, c, y, chunk_rows);
}

void rowpart_spmm(sfg_context* ctx, sfg_comm* c, const sfg_tensor* a, const void* b, int b_dtype, int64_t nd,
                  int64_t ldb, float* cbuf, int64_t chunk_rows, bool gather) {
  if (a->m > chunk_rows) raise(SFG_ERR_INVALID_OPERATION, "row block larger than the chunk");
  spmm(ctx, a, b, b_dtype, nd, ldb, cbuf + (int64_t)c->rank * chunk_rows * nd, nd, false);
  if (gather) allgather_chunks(ctx, c, cbuf, chunk_rows * nd);
}

}  // namespace sfg
