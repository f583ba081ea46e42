// Test infrastructure (not product code): an NCCL stand-in for multi-PROCESS worlds whose ranks
// share ONE GPU. Real NCCL rejects two ranks of a communicator on one device ("Duplicate GPU
// detected"), and the test boxes have one GPU, so the library's multi-process NCCL control
// path (ncclCommInitRank on a shared id, ncclCommSplit per grid line, grouped broadcasts /
// reduces / all-gathers / reduce-scatters / all-reduces, send+recv shifts, and the order in
// which every rank issues them) is exercised by LD_PRELOADing this library into each rank.
//
// Semantics follow nccl.h: stream-ordered collectives over the communicator's members, in-place
// variants allowed, NCCL_SPLIT_NOCOLOR, ncclGroupStart/End deferral. Implementation: a
// file-backed shared mapping per communicator (header + one staging slot per rank); each
// operation synchronises its stream, copies the rank's send buffer into its slot, meets the
// other members at a sense-reversing barrier, computes its result from the slots on the host
// (sums in fp32 in member order, bf16 rounded to nearest even) and copies it back on the same
// stream. Grouped operations run at the outermost ncclGroupEnd in issue order (a group of
// send/recv pairs as one exchange). Barrier waits time out (TPSHIM_TIMEOUT_S, default 300 s)
// with a message naming the operation instead of hanging the test.
#include <cuda_runtime.h>
#include <fcntl.h>
#include <nccl.h>
#include <sys/mman.h>
#include <unistd.h>

#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

namespace {

constexpr int kMaxRanks = 64;
constexpr size_t kHdr = 1 << 16;

struct Shared {
  std::atomic<int> arrive;
  std::atomic<int> sense;
  int split_color[kMaxRanks];
  int split_key[kMaxRanks];
};

size_t slot_bytes() {
  const char* e = getenv("TPSHIM_SLOT_MB");
  return size_t(e ? atoll(e) : 512) << 20;
}

}  // namespace

struct ncclComm {
  std::string name;
  int n = 0, rank = 0;
  Shared* sh = nullptr;
  char* base = nullptr;
  size_t map_bytes = 0, slot = 0;
  int gen = 0;
  int splits = 0;
  char* slot_of(int r) const { return base + kHdr + size_t(r) * slot; }
};

namespace {

double timeout_s() {
  const char* e = getenv("TPSHIM_TIMEOUT_S");
  return e ? atof(e) : 300.0;
}

void barrier(ncclComm* c, const char* what) {
  if (c->n == 1) return;
  const int g = c->gen ^ 1;
  c->gen = g;
  if (c->sh->arrive.fetch_add(1) == c->n - 1) {
    c->sh->arrive.store(0);
    c->sh->sense.store(g);
    return;
  }
  const auto t0 = std::chrono::steady_clock::now();
  int spins = 0;
  while (c->sh->sense.load() != g) {
    if (++spins > 1000) std::this_thread::sleep_for(std::chrono::microseconds(20));
    if ((spins & 1023) == 0 &&
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > timeout_s()) {
      fprintf(stderr, "[ncclshim] rank %d of %s (n=%d): barrier timeout in %s\n", c->rank,
              c->name.c_str(), c->n, what);
      fflush(stderr);
      abort();
    }
  }
}

ncclResult_t open_comm(ncclComm** out, const std::string& name, int n, int rank) {
  if (n < 1 || n > kMaxRanks || rank < 0 || rank >= n) return ncclInvalidArgument;
  auto* c = new ncclComm();
  c->name = name;
  c->n = n;
  c->rank = rank;
  c->slot = slot_bytes();
  c->map_bytes = kHdr + size_t(n) * c->slot;
  const std::string path = "/tmp/" + name;
  const int fd = open(path.c_str(), O_RDWR | O_CREAT, 0600);
  if (fd < 0 || ftruncate(fd, static_cast<off_t>(c->map_bytes)) != 0) {
    if (fd >= 0) close(fd);
    delete c;
    return ncclSystemError;
  }
  void* p = mmap(nullptr, c->map_bytes, PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (p == MAP_FAILED) {
    delete c;
    return ncclSystemError;
  }
  c->base = static_cast<char*>(p);
  c->sh = reinterpret_cast<Shared*>(c->base);
  barrier(c, "init");
  if (rank == 0) unlink(path.c_str());  // every member has it mapped
  *out = c;
  return ncclSuccess;
}

size_t dsize(ncclDataType_t t) {
  switch (t) {
    case ncclInt8: case ncclUint8: return 1;
    case ncclFloat16: case ncclBfloat16: return 2;
    case ncclInt32: case ncclUint32: case ncclFloat32: return 4;
    case ncclInt64: case ncclUint64: case ncclFloat64: return 8;
    default: return 0;
  }
}

float bf2f(uint16_t h) {
  uint32_t u = uint32_t(h) << 16;
  float f;
  memcpy(&f, &u, 4);
  return f;
}

uint16_t f2bf(float f) {
  uint32_t u;
  memcpy(&u, &f, 4);
  if ((u & 0x7fffffffu) > 0x7f800000u) return uint16_t((u >> 16) | 0x40);  // NaN stays NaN
  u += 0x7fffu + ((u >> 16) & 1u);
  return uint16_t(u >> 16);
}

// out[i] = sum over members m (in order) of src_m[i]
ncclResult_t sum_into(ncclComm* c, size_t off_elems, size_t count, ncclDataType_t dt, void* out) {
  if (dt == ncclFloat32 || dt == ncclBfloat16) {
    std::vector<float> acc(count, 0.f);
    for (int m = 0; m < c->n; ++m) {
      const char* s = c->slot_of(m);
      if (dt == ncclFloat32) {
        const float* f = reinterpret_cast<const float*>(s) + off_elems;
        for (size_t i = 0; i < count; ++i) acc[i] += f[i];
      } else {
        const uint16_t* h = reinterpret_cast<const uint16_t*>(s) + off_elems;
        for (size_t i = 0; i < count; ++i) acc[i] += bf2f(h[i]);
      }
    }
    if (dt == ncclFloat32) {
      memcpy(out, acc.data(), count * 4);
    } else {
      uint16_t* o = static_cast<uint16_t*>(out);
      for (size_t i = 0; i < count; ++i) o[i] = f2bf(acc[i]);
    }
    return ncclSuccess;
  }
  if (dt == ncclInt32) {
    std::vector<int32_t> acc(count, 0);
    for (int m = 0; m < c->n; ++m) {
      const int32_t* s = reinterpret_cast<const int32_t*>(c->slot_of(m)) + off_elems;
      for (size_t i = 0; i < count; ++i) acc[i] += s[i];
    }
    memcpy(out, acc.data(), count * 4);
    return ncclSuccess;
  }
  return ncclInvalidArgument;
}

enum Kind { BCAST, REDUCE, ALLREDUCE, ALLGATHER, REDUCESCATTER, SEND, RECV };

struct Op {
  Kind k;
  const void* send;
  void* recv;
  size_t count;  // per-rank element count (all-gather: sendcount; reduce-scatter: recvcount)
  ncclDataType_t dt;
  int root;  // bcast / reduce root; send / recv peer
  ncclComm* c;
  cudaStream_t s;
};

const char* kind_name(Kind k) {
  static const char* n[] = {"broadcast", "reduce", "allreduce", "allgather", "reducescatter",
                            "send", "recv"};
  return n[k];
}

ncclResult_t cuda_ok(cudaError_t e) { return e == cudaSuccess ? ncclSuccess : ncclUnhandledCudaError; }

#define SHIM_TRY(x)                      \
  do {                                   \
    ncclResult_t r_ = (x);               \
    if (r_ != ncclSuccess) return r_;    \
  } while (0)

// TPSHIM_HOST_BUFFERS=1: buffers are host memory and streams are ignored (the CPU self-test
// of the shim's rendezvous and collective semantics, tests/test_ncclshim_cpu.py)
bool host_buffers() {
  static const bool h = getenv("TPSHIM_HOST_BUFFERS") && atoi(getenv("TPSHIM_HOST_BUFFERS")) != 0;
  return h;
}

ncclResult_t d2h(void* h, const void* d, size_t b, cudaStream_t s) {
  if (!b) return ncclSuccess;
  if (host_buffers()) {
    memmove(h, d, b);
    return ncclSuccess;
  }
  SHIM_TRY(cuda_ok(cudaMemcpyAsync(h, d, b, cudaMemcpyDeviceToHost, s)));
  return cuda_ok(cudaStreamSynchronize(s));
}

ncclResult_t h2d(void* d, const void* h, size_t b, cudaStream_t s) {
  if (!b) return ncclSuccess;
  if (host_buffers()) {
    memmove(d, h, b);
    return ncclSuccess;
  }
  SHIM_TRY(cuda_ok(cudaMemcpyAsync(d, h, b, cudaMemcpyHostToDevice, s)));
  return cuda_ok(cudaStreamSynchronize(s));
}

ncclResult_t run_collective(const Op& o) {
  ncclComm* c = o.c;
  const size_t es = dsize(o.dt);
  if (!es) return ncclInvalidArgument;
  const size_t in_elems = o.k == REDUCESCATTER ? o.count * c->n : o.count;
  if (in_elems * es > c->slot) {
    fprintf(stderr, "[ncclshim] %s of %zu bytes exceeds the %zu-byte slot (TPSHIM_SLOT_MB)\n",
            kind_name(o.k), in_elems * es, c->slot);
    return ncclInvalidArgument;
  }
  if (!host_buffers()) SHIM_TRY(cuda_ok(cudaStreamSynchronize(o.s)));
  char* mine = c->slot_of(c->rank);
  if (o.k != BCAST || c->rank == o.root) SHIM_TRY(d2h(mine, o.send, in_elems * es, o.s));
  barrier(c, kind_name(o.k));
  std::vector<char> tmp;
  switch (o.k) {
    case BCAST:
      SHIM_TRY(h2d(o.recv, c->slot_of(o.root), o.count * es, o.s));
      break;
    case REDUCE:
      if (c->rank == o.root) {
        tmp.resize(o.count * es);
        SHIM_TRY(sum_into(c, 0, o.count, o.dt, tmp.data()));
        SHIM_TRY(h2d(o.recv, tmp.data(), tmp.size(), o.s));
      }
      break;
    case ALLREDUCE:
      tmp.resize(o.count * es);
      SHIM_TRY(sum_into(c, 0, o.count, o.dt, tmp.data()));
      SHIM_TRY(h2d(o.recv, tmp.data(), tmp.size(), o.s));
      break;
    case ALLGATHER:
      for (int m = 0; m < c->n; ++m)
        SHIM_TRY(h2d(static_cast<char*>(o.recv) + size_t(m) * o.count * es, c->slot_of(m),
                     o.count * es, o.s));
      break;
    case REDUCESCATTER:
      tmp.resize(o.count * es);
      SHIM_TRY(sum_into(c, size_t(c->rank) * o.count, o.count, o.dt, tmp.data()));
      SHIM_TRY(h2d(o.recv, tmp.data(), tmp.size(), o.s));
      break;
    default:
      return ncclInternalError;
  }
  barrier(c, kind_name(o.k));  // slots free for the next operation
  return ncclSuccess;
}

// A group of point-to-point operations on one communicator: every member's sends land in its
// slot (one region per destination), then the receives read them.
ncclResult_t run_p2p(const std::vector<Op>& ops) {
  ncclComm* c = ops[0].c;
  const size_t region = c->slot / c->n;
  for (const Op& o : ops) {
    if (o.c != c) {
      fprintf(stderr, "[ncclshim] p2p group over several communicators is not supported\n");
      return ncclInvalidUsage;
    }
    if (o.count * dsize(o.dt) > region) return ncclInvalidArgument;
  }
  for (const Op& o : ops)
    if (o.k == SEND)
      SHIM_TRY(d2h(c->slot_of(c->rank) + size_t(o.root) * region, o.send, o.count * dsize(o.dt), o.s));
  barrier(c, "send/recv");
  for (const Op& o : ops)
    if (o.k == RECV)
      SHIM_TRY(h2d(o.recv, c->slot_of(o.root) + size_t(c->rank) * region, o.count * dsize(o.dt), o.s));
  barrier(c, "send/recv");
  return ncclSuccess;
}

thread_local int g_depth = 0;
thread_local std::vector<Op> g_ops;

ncclResult_t flush_group(std::vector<Op> ops) {
  std::vector<Op> p2p;
  for (const Op& o : ops) {
    if (o.k == SEND || o.k == RECV) {
      p2p.push_back(o);
      continue;
    }
    if (!p2p.empty()) {
      fprintf(stderr, "[ncclshim] collectives after send/recv in one group are not supported\n");
      return ncclInvalidUsage;
    }
    SHIM_TRY(run_collective(o));
  }
  if (!p2p.empty()) SHIM_TRY(run_p2p(p2p));
  return ncclSuccess;
}

ncclResult_t submit(const Op& o) {
  if (!o.c) return ncclInvalidArgument;
  if (g_depth > 0) {
    g_ops.push_back(o);
    return ncclSuccess;
  }
  return flush_group({o});
}

}  // namespace

extern "C" {

ncclResult_t ncclGetUniqueId(ncclUniqueId* id) {
  memset(id, 0, sizeof(*id));
  unsigned long long r = 0;
  FILE* f = fopen("/dev/urandom", "rb");
  if (f) {
    if (fread(&r, sizeof(r), 1, f) != 1) r = 0;
    fclose(f);
  }
  r ^= static_cast<unsigned long long>(std::chrono::steady_clock::now().time_since_epoch().count());
  snprintf(id->internal, sizeof(id->internal), "tpshim_%d_%llx", static_cast<int>(getpid()), r);
  return ncclSuccess;
}

ncclResult_t ncclCommInitRank(ncclComm_t* comm, int nranks, ncclUniqueId commId, int rank) {
  commId.internal[sizeof(commId.internal) - 1] = 0;
  if (strncmp(commId.internal, "tpshim_", 7) != 0) return ncclInvalidArgument;
  return open_comm(comm, commId.internal, nranks, rank);
}

ncclResult_t ncclCommSplit(ncclComm_t comm, int color, int key, ncclComm_t* newcomm,
                           ncclConfig_t* /*config*/) {
  if (!comm) return ncclInvalidArgument;
  comm->sh->split_color[comm->rank] = color;
  comm->sh->split_key[comm->rank] = key;
  barrier(comm, "split");
  int n = 0, pos = 0;
  for (int r = 0; r < comm->n; ++r) {
    if (color == NCCL_SPLIT_NOCOLOR || comm->sh->split_color[r] != color) continue;
    const int kr = comm->sh->split_key[r];
    if (kr < key || (kr == key && r < comm->rank)) ++pos;
    ++n;
  }
  barrier(comm, "split");  // the table is free again
  const int seq = comm->splits++;
  if (color == NCCL_SPLIT_NOCOLOR) {
    *newcomm = nullptr;
    return ncclSuccess;
  }
  return open_comm(newcomm, comm->name + "_s" + std::to_string(seq) + "c" + std::to_string(color),
                   n, pos);
}

ncclResult_t ncclCommDestroy(ncclComm_t comm) {
  if (!comm) return ncclSuccess;
  munmap(comm->base, comm->map_bytes);
  delete comm;
  return ncclSuccess;
}

ncclResult_t ncclCommAbort(ncclComm_t comm) { return ncclCommDestroy(comm); }

ncclResult_t ncclCommGetAsyncError(ncclComm_t comm, ncclResult_t* asyncError) {
  if (!comm) return ncclInvalidArgument;
  *asyncError = ncclSuccess;
  return ncclSuccess;
}

const char* ncclGetErrorString(ncclResult_t result) {
  switch (result) {
    case ncclSuccess: return "no error (ncclshim)";
    case ncclInvalidArgument: return "invalid argument (ncclshim)";
    case ncclInvalidUsage: return "invalid usage (ncclshim)";
    case ncclUnhandledCudaError: return "unhandled cuda error (ncclshim)";
    case ncclSystemError: return "system error (ncclshim)";
    default: return "error (ncclshim)";
  }
}

ncclResult_t ncclGroupStart() {
  ++g_depth;
  return ncclSuccess;
}

ncclResult_t ncclGroupEnd() {
  if (g_depth <= 0) return ncclInvalidUsage;
  if (--g_depth > 0) return ncclSuccess;
  std::vector<Op> ops;
  ops.swap(g_ops);
  return ops.empty() ? ncclSuccess : flush_group(std::move(ops));
}

ncclResult_t ncclBroadcast(const void* sendbuff, void* recvbuff, size_t count, ncclDataType_t datatype,
                           int root, ncclComm_t comm, cudaStream_t stream) {
  return submit({BCAST, sendbuff, recvbuff, count, datatype, root, comm, stream});
}

ncclResult_t ncclReduce(const void* sendbuff, void* recvbuff, size_t count, ncclDataType_t datatype,
                        ncclRedOp_t op, int root, ncclComm_t comm, cudaStream_t stream) {
  if (op != ncclSum) return ncclInvalidArgument;
  return submit({REDUCE, sendbuff, recvbuff, count, datatype, root, comm, stream});
}

ncclResult_t ncclAllReduce(const void* sendbuff, void* recvbuff, size_t count, ncclDataType_t datatype,
                           ncclRedOp_t op, ncclComm_t comm, cudaStream_t stream) {
  if (op != ncclSum) return ncclInvalidArgument;
  return submit({ALLREDUCE, sendbuff, recvbuff, count, datatype, 0, comm, stream});
}

ncclResult_t ncclReduceScatter(const void* sendbuff, void* recvbuff, size_t recvcount,
                               ncclDataType_t datatype, ncclRedOp_t op, ncclComm_t comm,
                               cudaStream_t stream) {
  if (op != ncclSum) return ncclInvalidArgument;
  return submit({REDUCESCATTER, sendbuff, recvbuff, recvcount, datatype, 0, comm, stream});
}

ncclResult_t ncclAllGather(const void* sendbuff, void* recvbuff, size_t sendcount,
                           ncclDataType_t datatype, ncclComm_t comm, cudaStream_t stream) {
  return submit({ALLGATHER, sendbuff, recvbuff, sendcount, datatype, 0, comm, stream});
}

ncclResult_t ncclSend(const void* sendbuff, size_t count, ncclDataType_t datatype, int peer,
                      ncclComm_t comm, cudaStream_t stream) {
  return submit({SEND, sendbuff, nullptr, count, datatype, peer, comm, stream});
}

ncclResult_t ncclRecv(void* recvbuff, size_t count, ncclDataType_t datatype, int peer,
                      ncclComm_t comm, cudaStream_t stream) {
  return submit({RECV, nullptr, recvbuff, count, datatype, peer, comm, stream});
}

}  // extern "C"
