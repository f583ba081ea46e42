// Internal declarations shared by the library's translation units.
#pragma once

#include <cuda_runtime.h>

#include <atomic>
#include <initializer_list>
#include <cstdint>
#include <memory>
#include <string>
#include <vector>

#include "../../include/tp_b200.h"

namespace tp {

// ---- errors ---------------------------------------------------------------------------
void set_error(const std::string& msg);
tp_status fail(tp_status s, const std::string& msg);

#define TP_CUDA(call)                                                                   \
  do {                                                                                  \
    cudaError_t e_ = (call);                                                            \
    if (e_ != cudaSuccess)                                                              \
      return ::tp::fail(TP_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_)); \
  } while (0)

#define TP_TRY(call)               \
  do {                             \
    tp_status s_ = (call);         \
    if (s_ != TP_OK) return s_;    \
  } while (0)

inline size_t dtype_size(tp_dtype t) { return t == TP_BF16 ? 2 : 4; }

// ---- tuning knobs (capi.cpp registry; tp_knob_set / tp_knob_get / tp_knobs) ---------------
// The effective value of a registered knob: tp_knob_set override, else the TP_* environment
// variable (read once), else the measured default. Unknown names abort in debug builds and
// return 0.
int knob(const char* name);

// ---- per-device one-time setup ---------------------------------------------------------
// Kernel attributes (cudaFuncSetAttribute) belong to a device context: set_smem_attr runs
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) once per (kernel, current device); callers
// on other threads block until it has been applied (a launch must never race ahead of it).
cudaError_t set_smem_attr(const void* kernel, int bytes);

// Number of live in-process multi-rank grids (TP_TRANSPORT_LOCAL, world > 1). While any exists,
// other ranks' kernels may share the device, so no GEMM may assume its whole persistent grid is
// co-resident (the split-K owner-wait / exchange spins on sibling clusters): it falls back to
// the last-arriver reduction.
extern std::atomic<int> g_shared_device_grids;

// ---- instrumentation ------------------------------------------------------------------
extern std::atomic<int64_t> g_launches;
extern unsigned long long* g_gemm_trace;
inline void count_launch(int n = 1) { g_launches.fetch_add(n, std::memory_order_relaxed); }
bool prof_on();
extern thread_local int t_rank;  // grid rank of the calling entry point (span tags)
// Opens a timed region for kernel class `cls` on `s`; returns a token for prof_end.
int prof_begin(int cls, cudaStream_t s, double flops);
void prof_end(int token, cudaStream_t s);

// Launch with programmatic stream serialization (PDL): the kernel may start while its
// predecessor drains and must call griddepcontrol.wait before touching dependent memory.
bool pdl_enabled();
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                       Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// ---- kernels (layout.cu) ------------------------------------------------------------------
tp_status launch_copy2d(const void* src, int64_t src_ld, void* dst, int64_t dst_ld, int64_t rows,
                        int64_t cols, size_t esz, cudaStream_t s);
// GeLU (exact erf form) over n elements: fwd z = y, y = gelu(y); bwd dz = dy * gelu'(z).
tp_status launch_gelu_fwd(void* y, void* z, size_t n, tp_dtype dt, cudaStream_t s);
// out = a + b elementwise (residual connections); out may alias a or b.
tp_status launch_add(const void* a, const void* b, void* out, size_t n, tp_dtype dt, cudaStream_t s);
tp_status launch_gelu_bwd(const void* dy, const void* z, void* dz, size_t n, tp_dtype dt,
                          cudaStream_t s);
// Deterministic two-pass column sums; scratch holds kColsumSlabs * cols floats.
constexpr int kColsumSlabs = 32;
tp_status launch_colsum(const void* src, int64_t rows, int64_t cols, int64_t ld, tp_dtype dt,
                        void* dst, float* scratch, cudaStream_t s);
tp_status launch_fill(void* dst, tp_dtype dt, int64_t rows, int64_t cols, int64_t ld,
                      uint64_t seed, int tensor_id, int kind, float scale, int64_t r0, int64_t c0,
                      int64_t gcols, cudaStream_t s);
// out[i] = sum_{j<n} in[j][i] (ascending j), fp32 accumulate; n <= 16.
tp_status launch_sum_n(const void* const* in, int n, void* out, size_t count, tp_dtype dt,
                       cudaStream_t s);
tp_status launch_memset(void* dst, size_t bytes, cudaStream_t s);

// ---- GEMM (gemm_sm100.cu, gemm_simt.cu) --------------------------------------------------
struct GemmArgs {
  int64_t M = 0, N = 0, K = 0;
  const void* A = nullptr;
  int64_t lda = 0;
  bool trans_a = false;  // A stored [K,M]
  const void* B = nullptr;
  int64_t ldb = 0;
  bool trans_b = false;  // B stored [N,K]
  const float* C = nullptr;
  int64_t ldc = 0;
  void* D = nullptr;
  int64_t ldd = 0;
  tp_dtype in_dtype = TP_BF16;
  tp_dtype out_dtype = TP_BF16;
  float alpha = 1.f;
  const void* bias = nullptr;
  void* ws = nullptr;    // split-K scratch (optional; no split-K without it)
  size_t ws_bytes = 0;
  int reserve_sms = 0;  // leave this many SMs free (a collective runs concurrently)
  // K-panels (fused peer SUMMA): the contraction runs over npanels panels of K each; panel p
  // reads A from Ap[p] and B from Bp[p] (same lda / ldb), accumulating in TMEM. npanels == 1
  // uses A / B. Only the CTA-pair kernel takes npanels > 1.
  int npanels = 1;
  const void* Ap[4] = {};
  const void* Bp[4] = {};
  // D row-panels (fused 1D reduce-scatter): rows [p d_rows, (p+1) d_rows) of the product go
  // to Dp[p] (row stride ldd), e.g. a slot in the owning rank's receive buffer. d_rows % 32 == 0.
  // dpanels == 1 uses D. Only the CTA-pair kernel takes dpanels > 1.
  int dpanels = 1;
  int64_t d_rows = 0;
  void* Dp[8] = {};
};
tp_status gemm(const GemmArgs& a, cudaStream_t s);         // dispatch + validation
// Two independent GEMMs: one grouped CTA-pair launch when both qualify, else two launches.
tp_status gemm_pair(const GemmArgs& a, const GemmArgs& b, cudaStream_t s);
// Up to 4 independent problems in one persistent CTA-pair launch (kernel level).
tp_status gemm_tc2_group(const GemmArgs* gs, int n, cudaStream_t s);
// Up to 4 independent GEMMs: one grouped launch when every problem is eligible, else in turn.
tp_status gemm_group(const GemmArgs* gs, int n, cudaStream_t s);
tp_status gemm_tc_bf16(const GemmArgs& a, cudaStream_t s);  // tcgen05, 1 CTA per tile
tp_status gemm_tc2_bf16(const GemmArgs& a, cudaStream_t s); // tcgen05 cta_group::2 pair tiles
bool gemm_tc2_supported(const GemmArgs& a);
// true when a grouped pair launch of these problems would split a long-K member (its tiles
// far longer than the group's per-cluster share, e.g. a token-long dW next to many short dX
// tiles): the dispatcher then launches them separately (TP_GEMM_GROUP_LONGK)
bool gemm_tc2_group_splits_member(const GemmArgs* gs, int n);
size_t gemm_tc2_ws_bytes();                                 // split-K scratch upper bound
tp_status gemm_simt_f32(const GemmArgs& a, cudaStream_t s); // FFMA
tp_status gemm_k0(const GemmArgs& a, cudaStream_t s);       // K == 0 epilogue only

// ---- communication ------------------------------------------------------------------------
// One communicator per grid line (group); `pos` is this rank's position in it.
class Comm {
 public:
  virtual ~Comm() = default;
  virtual int size() const = 0;
  virtual int pos() const = 0;
  // In place: at root `buf` is the source, elsewhere the destination.
  virtual tp_status bcast(void* buf, size_t count, tp_dtype dt, int root, cudaStream_t s) = 0;
  // recv (significant at root only) = sum over members of send.
  virtual tp_status reduce(const void* send, void* recv, size_t count, tp_dtype dt, int root,
                           cudaStream_t s) = 0;
  virtual tp_status allreduce(const void* send, void* recv, size_t count, tp_dtype dt,
                              cudaStream_t s) = 0;
  // recv = concat over members (ascending) of send [count each].
  virtual tp_status allgather(const void* send, void* recv, size_t count, tp_dtype dt,
                              cudaStream_t s) = 0;
  // recv [count] = slice `pos` of sum over members of send [size*count].
  virtual tp_status reducescatter(const void* send, void* recv, size_t count, tp_dtype dt,
                                  cudaStream_t s) = 0;
  // Cyclic shift along the line: recv [count] = send of member (pos + offset) mod size.
  // offset -1: the Ring Self-Attention's K / V pass (every member sends to its successor,
  // P:L606-612); offset +s: Cannon's "shift left / up by s". offset 0 copies.
  virtual tp_status shift(const void* send, void* recv, size_t count, tp_dtype dt, int offset,
                          cudaStream_t s) = 0;
  virtual tp_status group_start() { return TP_OK; }
  virtual tp_status group_end() { return TP_OK; }
  // Stream-ordered barrier: work after it on `s` starts only once every member's work before
  // it (on their streams) has completed.
  virtual tp_status barrier(cudaStream_t s) = 0;
  // Host-side all-gather of `bytes` per member (setup only: buffer registration).
  virtual tp_status host_allgather(const void* in, size_t bytes, void* out) = 0;
  // Failure detection (safe from another thread): an asynchronous transport error (NCCL:
  // ncclCommGetAsyncError), and abort, which makes blocked / future collectives return.
  virtual tp_status async_error() { return TP_OK; }
  virtual void abort() {}
};

struct NcclWorld;  // transport_nccl.cpp
std::unique_ptr<Comm> make_nccl_comm(NcclWorld* w, int color, int key, int size, int pos,
                                     tp_status* st);
NcclWorld* nccl_world_create(int world, int rank, const void* id128, tp_status* st);
std::unique_ptr<Comm> make_nccl_world_comm(NcclWorld* w);
void nccl_world_destroy(NcclWorld* w);
tp_status nccl_world_async_error(NcclWorld* w);
void nccl_world_abort(NcclWorld* w);
tp_status nccl_unique_id(void* id128);
// A 1-rank NCCL communicator of this process alone (size-1 grid lines in tp_axis_collective).
std::unique_ptr<Comm> make_nccl_self_comm(tp_status* st);

std::unique_ptr<Comm> make_local_comm(const void* id128, int world, const std::vector<int>& members,
                                      int pos, int device, tp_status* st);
tp_status local_unique_id(void* id128);

// Collective-contract check (capi.cpp): `kind` names the entry point; `words` its scalar
// arguments. TP_OK when disabled, at world == 1, or when every rank passed the same values.
enum ContractKind : uint64_t {
  kCallLinearFwd = 1, kCallLinearBwd, kCallLnFwd, kCallLnBwd, kCallRsaFwd, kCallRsaBwd,
  kCallAttnFwd, kCallAttnBwd
};
// d may be null (entry points without a linear desc). f32_word: a float's bit pattern.
uint64_t f32_word(float f);
tp_status contract_check(tp_grid* g, ContractKind kind, const tp_linear_desc* d,
                         std::initializer_list<uint64_t> words);

}  // namespace tp

// ---- the grid -----------------------------------------------------------------------------
struct tp_grid {
  tp_mode mode = TP_1D;
  int world = 1, rank = 0, q = 1, d = 1;
  int ndims = 1;
  int dims[3] = {1, 1, 1};
  int coords[3] = {0, 0, 0};
  int device = 0;
  tp_transport transport = TP_TRANSPORT_NONE;
  tp::NcclWorld* nccl = nullptr;
  std::unique_ptr<tp::Comm> axis[3];  // line along each axis (nullptr if size 1 or NONE)
  std::unique_ptr<tp::Comm> all;      // every rank (barriers, registration); nullptr if p == 1
  std::unique_ptr<tp::Comm> unit_axis[3];  // NCCL 1-rank comms for size-1 lines (lazy)
  // Symmetric registered buffers (tp_register_buffer): this rank's range and every rank's
  // pointer to its own copy, directly dereferenceable here (same process or CUDA IPC).
  struct RegBuf {
    char* base = nullptr;
    size_t bytes = 0;
    std::vector<char*> peer;
    std::vector<void*> ipc_opened;  // IPC mappings to close on deregistration
  };
  std::vector<RegBuf> regs;
  std::vector<int> peer_device;   // each rank's CUDA device (filled by tp_register_buffer)
  uint64_t staged_bytes = 0;      // bytes pulled from peers by staging copies (TP_FLAG_PEER_STAGED)
  std::vector<std::pair<std::string, void*>> ipc_cache;  // (peer rank + IPC handle) -> mapping
  // Pointer on `peer_rank` corresponding to `mine` (same offset in the same registered buffer),
  // or nullptr if `mine` is not inside a registered buffer.
  const void* peer_ptr(int peer_rank, const void* mine) const {
    const char* p = static_cast<const char*>(mine);
    for (const auto& r : regs)
      if (p >= r.base && p < r.base + r.bytes) return r.peer[peer_rank] + (p - r.base);
    return nullptr;
  }
  // Collective-contract check (tp_grid_set_contract_check): per-grid count of checked calls.
  bool contract_check = false;
  uint64_t contract_calls = 0;
  cudaStream_t comm_stream = nullptr;
  static constexpr int kEvents = 64;
  cudaEvent_t events[kEvents] = {};
  int next_event = 0;
  cudaEvent_t ev() {  // round-robin event pool (timing disabled)
    cudaEvent_t e = events[next_event];
    next_event = (next_event + 1) % kEvents;
    return e;
  }
  std::vector<int> group_members(int axis) const;
};
