// NCCL transport: one communicator for the world (ncclCommInitRank on the caller-shared
// unique id), one per grid line via ncclCommSplit ("only incur communication on a
// sub-group"). On an NVSwitch B200 node every pair of GPUs has full NVLink 5 bandwidth, so
// the row/column/depth communicators need no placement (contrast P:L155-157).
#include <nccl.h>

#include <cstring>

#include "tp_internal.h"

namespace tp {

struct NcclWorld {
  ncclComm_t world = nullptr;
  int size = 0, rank = 0;
};

namespace {

tp_status nccl_fail(ncclResult_t r, const char* what) {
  return fail(TP_ERR_NCCL, std::string(what) + ": " + ncclGetErrorString(r));
}

#define TP_NCCL(call)                                \
  do {                                               \
    ncclResult_t r_ = (call);                        \
    if (r_ != ncclSuccess) return nccl_fail(r_, #call); \
  } while (0)

ncclDataType_t nt(tp_dtype d) { return d == TP_BF16 ? ncclBfloat16 : ncclFloat32; }

class NcclComm final : public Comm {
 public:
  NcclComm(ncclComm_t c, int size, int pos, bool owns = true)
      : c_(c), size_(size), pos_(pos), owns_(owns) {}
  ~NcclComm() override {
    if (scratch_) cudaFree(scratch_);
    if (c_ && owns_) ncclCommDestroy(c_);
  }
  int size() const override { return size_; }
  int pos() const override { return pos_; }
  tp_status bcast(void* buf, size_t count, tp_dtype dt, int root, cudaStream_t s) override {
    if (!count) return TP_OK;
    TP_NCCL(ncclBroadcast(buf, buf, count, nt(dt), root, c_, s));
    return TP_OK;
  }
  tp_status reduce(const void* send, void* recv, size_t count, tp_dtype dt, int root,
                   cudaStream_t s) override {
    if (!count) return TP_OK;
    TP_NCCL(ncclReduce(send, recv, count, nt(dt), ncclSum, root, c_, s));
    return TP_OK;
  }
  tp_status allreduce(const void* send, void* recv, size_t count, tp_dtype dt,
                      cudaStream_t s) override {
    if (!count) return TP_OK;
    TP_NCCL(ncclAllReduce(send, recv, count, nt(dt), ncclSum, c_, s));
    return TP_OK;
  }
  tp_status allgather(const void* send, void* recv, size_t count, tp_dtype dt,
                      cudaStream_t s) override {
    if (!count) return TP_OK;
    TP_NCCL(ncclAllGather(send, recv, count, nt(dt), c_, s));
    return TP_OK;
  }
  tp_status reducescatter(const void* send, void* recv, size_t count, tp_dtype dt,
                          cudaStream_t s) override {
    if (!count) return TP_OK;
    TP_NCCL(ncclReduceScatter(send, recv, count, nt(dt), ncclSum, c_, s));
    return TP_OK;
  }
  tp_status shift(const void* send, void* recv, size_t count, tp_dtype dt, int offset,
                  cudaStream_t s) override {
    if (!count) return TP_OK;
    const int n = size_;
    const int off = ((offset % n) + n) % n;
    if (off == 0) {
      if (send != recv)
        TP_CUDA(cudaMemcpyAsync(recv, send, count * dtype_size(dt), cudaMemcpyDeviceToDevice, s));
      return TP_OK;
    }
    TP_NCCL(ncclGroupStart());
    TP_NCCL(ncclSend(send, count, nt(dt), (pos_ - off + n) % n, c_, s));
    TP_NCCL(ncclRecv(recv, count, nt(dt), (pos_ + off) % n, c_, s));
    TP_NCCL(ncclGroupEnd());
    return TP_OK;
  }
  tp_status group_start() override {
    TP_NCCL(ncclGroupStart());
    return TP_OK;
  }
  tp_status async_error() override {
    ncclResult_t e = ncclSuccess;
    TP_NCCL(ncclCommGetAsyncError(c_, &e));
    if (e != ncclSuccess && e != ncclInProgress) return nccl_fail(e, "communicator async error");
    return TP_OK;
  }
  void abort() override {
    if (c_ && owns_) {
      ncclCommAbort(c_);
      c_ = nullptr;
    }
  }
  tp_status group_end() override {
    TP_NCCL(ncclGroupEnd());
    return TP_OK;
  }
  // a 4-byte all-reduce: stream-ordered, completes on each member only after every member's
  // prior work on its stream
  tp_status barrier(cudaStream_t s) override {
    if (!scratch_) TP_CUDA(cudaMalloc(&scratch_, 256));
    TP_NCCL(ncclAllReduce(scratch_, scratch_, 1, ncclInt32, ncclSum, c_, s));
    return TP_OK;
  }
  tp_status host_allgather(const void* in, size_t bytes, void* out) override {
    char* d = nullptr;
    cudaStream_t st = nullptr;
    TP_CUDA(cudaMalloc(&d, bytes * (size_ + 1)));
    TP_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    tp_status rc = TP_OK;
    if (cudaMemcpyAsync(d, in, bytes, cudaMemcpyHostToDevice, st) != cudaSuccess) rc = TP_ERR_CUDA;
    if (rc == TP_OK) {
      ncclResult_t r = ncclAllGather(d, d + bytes, bytes, ncclChar, c_, st);
      if (r != ncclSuccess) rc = nccl_fail(r, "ncclAllGather (registration)");
    }
    if (rc == TP_OK && cudaMemcpyAsync(out, d + bytes, bytes * size_, cudaMemcpyDeviceToHost, st) !=
                           cudaSuccess)
      rc = TP_ERR_CUDA;
    if (cudaStreamSynchronize(st) != cudaSuccess && rc == TP_OK) rc = TP_ERR_CUDA;
    cudaStreamDestroy(st);
    cudaFree(d);
    if (rc == TP_ERR_CUDA) return fail(TP_ERR_CUDA, "host_allgather: CUDA copy failed");
    return rc;
  }

 private:
  ncclComm_t c_;
  int size_, pos_;
  bool owns_;
  int* scratch_ = nullptr;
};

}  // namespace

tp_status nccl_unique_id(void* id128) {
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  ncclUniqueId id;
  TP_NCCL(ncclGetUniqueId(&id));
  std::memcpy(id128, &id, sizeof(id));
  return TP_OK;
}

NcclWorld* nccl_world_create(int world, int rank, const void* id128, tp_status* st) {
  ncclUniqueId id;
  std::memcpy(&id, id128, sizeof(id));
  auto* w = new NcclWorld();
  w->size = world;
  w->rank = rank;
  ncclResult_t r = ncclCommInitRank(&w->world, world, id, rank);
  if (r != ncclSuccess) {
    *st = nccl_fail(r, "ncclCommInitRank");
    delete w;
    return nullptr;
  }
  *st = TP_OK;
  return w;
}

tp_status nccl_world_async_error(NcclWorld* w) {
  if (!w || !w->world) return TP_OK;
  ncclResult_t e = ncclSuccess;
  TP_NCCL(ncclCommGetAsyncError(w->world, &e));
  if (e != ncclSuccess && e != ncclInProgress) return nccl_fail(e, "world communicator async error");
  return TP_OK;
}

void nccl_world_abort(NcclWorld* w) {
  if (w && w->world) {
    ncclCommAbort(w->world);
    w->world = nullptr;
  }
}

void nccl_world_destroy(NcclWorld* w) {
  if (!w) return;
  if (w->world) ncclCommDestroy(w->world);
  delete w;
}

// Collective over the world communicator: every rank calls it once per axis.
std::unique_ptr<Comm> make_nccl_comm(NcclWorld* w, int color, int key, int size, int pos,
                                     tp_status* st) {
  ncclComm_t c = nullptr;
  ncclResult_t r = ncclCommSplit(w->world, color, key, &c, nullptr);
  if (r != ncclSuccess) {
    *st = nccl_fail(r, "ncclCommSplit");
    return nullptr;
  }
  *st = TP_OK;
  return std::make_unique<NcclComm>(c, size, pos);
}

std::unique_ptr<Comm> make_nccl_self_comm(tp_status* st) {
  ncclUniqueId id;
  ncclComm_t c = nullptr;
  ncclResult_t r = ncclGetUniqueId(&id);
  if (r == ncclSuccess) r = ncclCommInitRank(&c, 1, id, 0);
  if (r != ncclSuccess) {
    *st = nccl_fail(r, "ncclCommInitRank (1-rank line)");
    return nullptr;
  }
  *st = TP_OK;
  return std::make_unique<NcclComm>(c, 1, 0);
}

// Non-owning view of the world communicator (destroyed with the NcclWorld).
std::unique_ptr<Comm> make_nccl_world_comm(NcclWorld* w) {
  return std::make_unique<NcclComm>(w->world, w->size, w->rank, /*owns=*/false);
}

}  // namespace tp
