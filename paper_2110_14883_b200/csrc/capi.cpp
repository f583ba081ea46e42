// The C ABI (include/tp_b200.h): argument validation, the grid / parallel context
// ("parallel context manager"), and dispatch into the per-mode schedules.
#include <cuda.h>
#include <nvtx3/nvToolsExt.h>
#include <cudaTypedefs.h>
#include <unistd.h>

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "sched.h"

namespace tp {

namespace {
thread_local std::string t_err;
}

void set_error(const std::string& msg) { t_err = msg; }

tp_status fail(tp_status s, const std::string& msg) {
  t_err = msg;
  return s;
}

std::atomic<int64_t> g_launches{0};

// ---- tuning knobs: every dispatch / kernel-variant choice the library makes from outside its
// own measurements, in one table (defaults = the measured choices, see DESIGN / profiles).
namespace {
struct KnobDef {
  const char* name;
  int def;
  const char* what;
};
constexpr KnobDef kKnobs[] = {
    {"TP_PDL", 1, "programmatic dependent launch for the GEMM kernels (0 off)"},
    {"TP_GEMM_KERNEL", 0, "force the GEMM kernel: 1 = 1-CTA tiles, 2 = CTA-pair tiles (0 auto)"},
    {"TP_GEMM_BN", 0, "force the pair tile width 128 / 256 (0 auto)"},
    {"TP_GEMM_MC", 0, "force a pair-kernel cluster: 2/3 = A/B multicast over 2 pairs, 4 = 2x2, 5 = K-split pair cluster (0/1 none)"},
    {"TP_GEMM_EPI_WARPS", 0, "force 4 or 8 epilogue warps in the pair kernel (0 auto)"},
    {"TP_GEMM_SPLITK", 1, "split-K in the pair kernel when tiles are few (0 off)"},
    {"TP_GEMM_SPLIT_OWNER", 1, "split-K owner-wait / exchange when all splits are co-resident (0 last-arriver)"},
    {"TP_GEMM_GROUP", 1, "independent products (dX, dW) as one grouped launch (0 separate)"},
    {"TP_GEMM_GROUP_BN", 256, "pair tile width of grouped launches"},
    {"TP_GEMM_GROUP_SPLIT", 1, "split-K inside grouped launches for long-K members (0 off)"},
    {"TP_GEMM_GROUP_LONGK", 1, "a group member the group would split-K (long K) makes the problems launch separately (0: keep the group)"},
    {"TP_GEMM_RASTER", 8, "pair-tile rows per raster band"},
    {"TP_GEMM_ABOX64", 0, "pair kernel: K-major A as two 64-row TMA boxes per k-block (measurement knob)"},
    {"TP_GEMM_L2PROMO", 3, "pair-kernel tensor maps' L2 promotion: 0 none, 1 64 B, 2 128 B, 3 256 B"},
    {"TP_GEMM_SCHED", 1, "longest-first unit-to-cluster schedule for pair launches with unequal units (0 round robin)"},
    {"TP_GEMM_EPI_DIAG", 0, "diagnostics (TP_TIMELINE builds only): pair-kernel epilogue skips its stores (1) or staging and stores (2)"},
    {"TP_GEMM_SCHED_EPI", 800, "per-unit epilogue cost (SM clocks) in the unit schedule's cost model"},
    {"TP_GEMM_WIDE", -1, "512x256 wide pair tiles: -1 auto (K >= 12288, >= #SMs tiles), 0 off, 1 wherever legal"},
    {"TP_GEMM_WIDE_RASTER", 8, "wide-tile rows per raster band"},
    {"TP_GEMM_WIDE_NP", 0, "wide tiles non-persistent (one tile per cluster; measured equal)"},
    {"TP_GEMM_NARROW", 1, "ragged last n-tile of <= 128 columns as a half-width pair tile (0 off)"},
    {"TP_GEMM_V1_BN", 0, "force the 1-CTA tile width 128 / 256 (0 auto)"},
    {"TP_GEMM_V1_TMA_STORE", 1, "1-CTA kernel TMA-store epilogue (0 per-element stores)"},
    {"TP_COMM_SMS", -1, "SMs a GEMM leaves to a collective running under it (-1 sized to the transfer)"},
    {"TP_FLASH", 1, "fused attention kernels (0 = two-pass through HBM)"},
    {"TP_RSA_FUSED", 1, "online-softmax ring for Ring Self-Attention in bf16 (0 two-pass)"},
    {"TP_FB_NODQ", 0, "diagnostics: the fused attention backward skips its dQ accumulation (wrong dQ)"},
};
constexpr int kNumKnobs = sizeof(kKnobs) / sizeof(kKnobs[0]);
struct KnobState {
  bool init = false, overridden = false, from_env = false;
  int value = 0;
};
std::mutex g_knob_mu;
KnobState g_knob[kNumKnobs];
int knob_index(const char* name) {
  for (int i = 0; i < kNumKnobs; ++i)
    if (std::strcmp(kKnobs[i].name, name) == 0) return i;
  return -1;
}
KnobState& knob_state(int i) {  // caller holds g_knob_mu
  KnobState& k = g_knob[i];
  if (!k.init) {
    const char* e = std::getenv(kKnobs[i].name);
    k.from_env = e != nullptr;
    k.value = e ? std::atoi(e) : kKnobs[i].def;
    k.init = true;
  }
  return k;
}
}  // namespace

int knob(const char* name) {
  const int i = knob_index(name);
  if (i < 0) return 0;
  std::lock_guard<std::mutex> lk(g_knob_mu);
  return knob_state(i).value;
}

// NVTX range over an entry point (host-side; nsys / ncu --nvtx show the library's calls)
struct NvtxRange {
  explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
  ~NvtxRange() { nvtxRangePop(); }
};
std::atomic<int> g_shared_device_grids{0};

cudaError_t set_smem_attr(const void* kernel, int bytes) {
  static std::mutex mu;
  static std::vector<std::pair<const void*, int>> done;
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  std::lock_guard<std::mutex> lk(mu);
  for (const auto& kv : done)
    if (kv.first == kernel && kv.second == dev) return cudaSuccess;
  e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
  if (e == cudaSuccess) done.emplace_back(kernel, dev);
  return e;
}

// ---- collective-contract check (tp_grid_set_contract_check) -----------------
namespace {
uint64_t fnv1a(uint64_t h, uint64_t w) {
  for (int b = 0; b < 8; ++b) {
    h ^= (w >> (8 * b)) & 0xffu;
    h *= 0x100000001b3ull;
  }
  return h;
}
}  // namespace

uint64_t f32_word(float f) {
  uint32_t u;
  std::memcpy(&u, &f, 4);
  return u;
}

tp_status contract_check(tp_grid* g, ContractKind kind, const tp_linear_desc* d,
                         std::initializer_list<uint64_t> words) {
  if (g) t_rank = g->rank;  // span tags (tp_prof_spans) of the work this call issues
  if (!g || !g->contract_check || !g->all || g->world <= 1) return TP_OK;
  const uint64_t call = g->contract_calls++;
  uint64_t h = 0xcbf29ce484222325ull;
  h = fnv1a(h, kind);
  h = fnv1a(h, call);
  if (d) {
    for (uint64_t w : {uint64_t(d->M), uint64_t(d->K), uint64_t(d->N), uint64_t(d->dtype),
                       uint64_t(d->split_1d), uint64_t(d->parity_3d), uint64_t(d->flags),
                       f32_word(d->alpha)})
      h = fnv1a(h, w);
  }
  for (uint64_t w : words) h = fnv1a(h, w);
  std::vector<uint64_t> all(g->world);
  TP_TRY(g->all->host_allgather(&h, sizeof(h), all.data()));
  for (int r = 0; r < g->world; ++r)
    if (all[r] != all[0])
      return fail(TP_ERR_ARG, "collective contract violated at checked call #" +
                                  std::to_string(call) + ": rank " + std::to_string(r) +
                                  " passed a different entry point / desc than rank 0 (this rank " +
                                  std::to_string(g->rank) + "); nothing was enqueued");
  return TP_OK;
}

// ---- instrumentation: events around GEMM launches --------------------------------------
namespace {
struct ProfRec {
  int cls;
  double flops;
  cudaEvent_t a, b;
  int rank;
};
std::mutex g_prof_mu;
std::vector<ProfRec> g_prof;
std::atomic<bool> g_prof_on{false};
}  // namespace

bool prof_on() { return g_prof_on.load(std::memory_order_relaxed); }
thread_local int t_rank = -1;

bool pdl_enabled() {
  const bool on = knob("TP_PDL") != 0;
  return on;
}

// Under CUDA-graph capture the record becomes an external event node, so the timestamps are
// taken on every replay of the graph (read them after each replay).
static void record_timing_event(cudaEvent_t e, cudaStream_t s) {
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &st) == cudaSuccess && st == cudaStreamCaptureStatusActive)
    cudaEventRecordWithFlags(e, s, cudaEventRecordExternal);
  else
    cudaEventRecord(e, s);
}

int prof_begin(int cls, cudaStream_t s, double flops) {
  if (!prof_on()) return -1;
  ProfRec r{cls, flops, nullptr, nullptr, t_rank};
  cudaEventCreate(&r.a);
  cudaEventCreate(&r.b);
  record_timing_event(r.a, s);
  std::lock_guard<std::mutex> lk(g_prof_mu);
  g_prof.push_back(r);
  return static_cast<int>(g_prof.size()) - 1;
}

void prof_end(int token, cudaStream_t s) {
  if (token < 0) return;
  cudaEvent_t b;
  {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    if (token >= static_cast<int>(g_prof.size())) return;
    b = g_prof[token].b;
  }
  record_timing_event(b, s);
}

// Decorator: every collective of a line communicator as a span of class 2 (tp_prof_spans).
namespace {
class TracedComm final : public Comm {
 public:
  explicit TracedComm(std::unique_ptr<Comm> c) : c_(std::move(c)) {}
  int size() const override { return c_->size(); }
  int pos() const override { return c_->pos(); }
  tp_status bcast(void* buf, size_t n, tp_dtype dt, int root, cudaStream_t s) override {
    return span(n, dt, s, [&] { return c_->bcast(buf, n, dt, root, s); });
  }
  tp_status reduce(const void* a, void* b, size_t n, tp_dtype dt, int root, cudaStream_t s) override {
    return span(n, dt, s, [&] { return c_->reduce(a, b, n, dt, root, s); });
  }
  tp_status allreduce(const void* a, void* b, size_t n, tp_dtype dt, cudaStream_t s) override {
    return span(n, dt, s, [&] { return c_->allreduce(a, b, n, dt, s); });
  }
  tp_status allgather(const void* a, void* b, size_t n, tp_dtype dt, cudaStream_t s) override {
    return span(n * c_->size(), dt, s, [&] { return c_->allgather(a, b, n, dt, s); });
  }
  tp_status reducescatter(const void* a, void* b, size_t n, tp_dtype dt, cudaStream_t s) override {
    return span(n * c_->size(), dt, s, [&] { return c_->reducescatter(a, b, n, dt, s); });
  }
  tp_status shift(const void* a, void* b, size_t n, tp_dtype dt, int off, cudaStream_t s) override {
    return span(n, dt, s, [&] { return c_->shift(a, b, n, dt, off, s); });
  }
  tp_status group_start() override { return c_->group_start(); }
  tp_status group_end() override { return c_->group_end(); }
  tp_status barrier(cudaStream_t s) override {
    return span(0, TP_BF16, s, [&] { return c_->barrier(s); });
  }
  tp_status host_allgather(const void* in, size_t bytes, void* out) override {
    return c_->host_allgather(in, bytes, out);
  }
  tp_status async_error() override { return c_->async_error(); }
  void abort() override { c_->abort(); }

 private:
  template <typename F>
  tp_status span(size_t n, tp_dtype dt, cudaStream_t s, F f) {
    const int tok = prof_begin(2, s, double(n) * double(dtype_size(dt)));
    const tp_status st = f();
    prof_end(tok, s);
    return st;
  }
  std::unique_ptr<Comm> c_;
};
std::unique_ptr<Comm> traced(std::unique_ptr<Comm> c) {
  return c ? std::unique_ptr<Comm>(new TracedComm(std::move(c))) : nullptr;
}
}  // namespace

}  // namespace tp

using namespace tp;

std::vector<int> tp_grid::group_members(int ax) const {
  std::vector<int> out;
  int c[3] = {coords[0], coords[1], coords[2]};
  for (int v = 0; v < dims[ax]; ++v) {
    c[ax] = v;
    int r = 0;
    for (int k = 0; k < ndims; ++k) r = r * dims[k] + c[k];
    out.push_back(r);
  }
  return out;
}

namespace {

int iroot(int p, int e) {
  for (int c = 1; c <= p; ++c) {
    int64_t v = 1;
    for (int k = 0; k < e; ++k) v *= c;
    if (v == p) return c;
    if (v > p) break;
  }
  return -1;
}

tp_status plan_grid(tp_grid* g, tp_mode mode, int world, int rank, int q, int d) {
  if (world < 1) return fail(TP_ERR_ARG, "world must be >= 1");
  if (rank < 0 || rank >= world) return fail(TP_ERR_ARG, "rank out of range");
  g->mode = mode;
  g->world = world;
  g->rank = rank;
  switch (mode) {
    case TP_1D:
      g->ndims = 1;
      g->dims[0] = world;
      g->q = world;
      g->d = 1;
      break;
    case TP_2D: {
      const int j = iroot(world, 2);
      if (j < 0) return fail(TP_ERR_CONSTRAINT, "2D needs p = j^2, got " + std::to_string(world));
      if (q > 0 && q != j) return fail(TP_ERR_CONSTRAINT, "2D: q*q != world");
      g->ndims = 2;
      g->dims[0] = g->dims[1] = j;
      g->q = j;
      g->d = 1;
      break;
    }
    case TP_2P5D: {
      if (d < 1 || world % d)
        return fail(TP_ERR_CONSTRAINT, "2.5D needs p = d*k^2 (p=" + std::to_string(world) +
                                           ", d=" + std::to_string(d) + ")");
      const int k = iroot(world / d, 2);
      if (k < 0)
        return fail(TP_ERR_CONSTRAINT, "2.5D needs p = d*k^2 (p=" + std::to_string(world) +
                                           ", d=" + std::to_string(d) + ")");
      if (q > 0 && q != k) return fail(TP_ERR_CONSTRAINT, "2.5D: d*q*q != world");
      g->ndims = 3;
      g->dims[0] = d;
      g->dims[1] = g->dims[2] = k;
      g->q = k;
      g->d = d;
      break;
    }
    case TP_3D: {
      const int l = iroot(world, 3);
      if (l < 0) return fail(TP_ERR_CONSTRAINT, "3D needs p = l^3, got " + std::to_string(world));
      if (q > 0 && q != l) return fail(TP_ERR_CONSTRAINT, "3D: q^3 != world");
      g->ndims = 3;
      g->dims[0] = g->dims[1] = g->dims[2] = l;
      g->q = l;
      g->d = 1;
      break;
    }
    default:
      return fail(TP_ERR_ARG, "unknown mode");
  }
  int r = rank;
  for (int k = g->ndims - 1; k >= 0; --k) {
    g->coords[k] = r % g->dims[k];
    r /= g->dims[k];
  }
  return TP_OK;
}

// Color of this rank's line along `ax`: the rank with that coordinate zeroed (unique per line).
int line_color(const tp_grid* g, int ax) {
  int c[3] = {g->coords[0], g->coords[1], g->coords[2]};
  c[ax] = 0;
  int r = 0;
  for (int k = 0; k < g->ndims; ++k) r = r * g->dims[k] + c[k];
  return r;
}

tp_status check_desc(const tp_grid* g, const tp_linear_desc* d) {
  if (!g) return fail(TP_ERR_ARG, "grid is null");
  if (!d) return fail(TP_ERR_ARG, "desc is null");
  if (d->dtype != TP_BF16 && d->dtype != TP_FP32) return fail(TP_ERR_ARG, "unknown dtype");
  return check_divisible(g, d);
}

tp_status plan_mode_sizes(tp_grid* g, const tp_linear_desc* d, size_t* ws, size_t* saved) {
  Run R;
  R.g = g;
  R.d = d;
  R.plan = true;
  TP_TRY(sched_fwd(R, nullptr, nullptr, nullptr, nullptr));
  size_t wf = R.ws.off, sf = R.saved.off;
  Run B;
  B.g = g;
  B.d = d;
  B.plan = true;
  // plan with every optional output present (the largest footprint)
  char dummy;
  TP_TRY(sched_bwd(B, nullptr, nullptr, nullptr, &dummy, &dummy, &dummy));
  *ws = std::max(wf, B.ws.off);
  *saved = sf;
  return TP_OK;
}

size_t align256(size_t v) { return (v + 255) & ~size_t(255); }

// TP_FLAG_GELU: the pre-activation Z (Y shard) lives in `saved` after the mode's own content,
// and the backward's dZ in `ws` after the mode's scratch.
struct GeluLayout {
  size_t saved_off = 0, ws_off = 0, bytes = 0, n = 0;
};

tp_status gelu_layout(tp_grid* g, const tp_linear_desc* d, GeluLayout* L) {
  size_t ws = 0, sv = 0;
  TP_TRY(plan_mode_sizes(g, d, &ws, &sv));
  Ext e;
  TP_TRY(extent(g, d, TP_TENSOR_Y, &e));
  L->n = size_t(e.rows) * size_t(e.cols);
  L->bytes = L->n * dtype_size(d->dtype);
  L->saved_off = align256(sv);
  L->ws_off = align256(ws);
  return TP_OK;
}

tp_status plan_sizes(tp_grid* g, const tp_linear_desc* d, size_t* ws, size_t* saved) {
  TP_TRY(plan_mode_sizes(g, d, ws, saved));
  if (d->flags & TP_FLAG_GELU) {
    GeluLayout L;
    TP_TRY(gelu_layout(g, d, &L));
    *ws = L.ws_off + L.bytes;
    *saved = L.saved_off + L.bytes;
  }
  return TP_OK;
}

}  // namespace

extern "C" {

const char* tp_status_string(tp_status s) {
  switch (s) {
    case TP_OK: return "TP_OK";
    case TP_ERR_CONSTRAINT: return "TP_ERR_CONSTRAINT";
    case TP_ERR_INDIVISIBLE: return "TP_ERR_INDIVISIBLE";
    case TP_ERR_SHAPE: return "TP_ERR_SHAPE";
    case TP_ERR_ARG: return "TP_ERR_ARG";
    case TP_ERR_CUDA: return "TP_ERR_CUDA";
    case TP_ERR_NCCL: return "TP_ERR_NCCL";
    case TP_ERR_WORKSPACE: return "TP_ERR_WORKSPACE";
    case TP_ERR_UNSUPPORTED: return "TP_ERR_UNSUPPORTED";
  }
  return "TP_ERR_UNKNOWN";
}

const char* tp_last_error(void) { return t_err.c_str(); }

const char* tp_version(void) { return "tp_b200 0.1 sm_100a"; }

tp_status tp_get_unique_id(tp_transport transport, void* id128) {
  if (!id128) return fail(TP_ERR_ARG, "id128 is null");
  switch (transport) {
    case TP_TRANSPORT_NCCL: return nccl_unique_id(id128);
    case TP_TRANSPORT_LOCAL: return local_unique_id(id128);
    case TP_TRANSPORT_NONE: std::memset(id128, 0, 128); return TP_OK;
  }
  return fail(TP_ERR_ARG, "unknown transport");
}

tp_status tp_grid_init(tp_grid** out, tp_mode mode, int world, int rank, int q, int d,
                       int cuda_device, tp_transport transport, const void* id128) {
  if (!out) return fail(TP_ERR_ARG, "grid out-pointer is null");
  *out = nullptr;
  if (mode != TP_2P5D) d = 1;
  auto g = std::make_unique<tp_grid>();
  TP_TRY(plan_grid(g.get(), mode, world, rank, q, d));
  g->device = cuda_device;
  g->transport = transport;
  if (transport == TP_TRANSPORT_NONE) {
    *out = g.release();
    return TP_OK;
  }
  if (transport != TP_TRANSPORT_NCCL && transport != TP_TRANSPORT_LOCAL)
    return fail(TP_ERR_ARG, "unknown transport");
  if (!id128) return fail(TP_ERR_ARG, "id128 is null");
  TP_CUDA(cudaSetDevice(cuda_device));
  TP_CUDA(cudaStreamCreateWithFlags(&g->comm_stream, cudaStreamNonBlocking));
  for (auto& e : g->events) TP_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  tp_status st = TP_OK;
  if (transport == TP_TRANSPORT_NCCL) {
    g->nccl = nccl_world_create(world, rank, id128, &st);
    if (st != TP_OK) return st;
  }
  for (int ax = 0; ax < g->ndims; ++ax) {
    if (g->dims[ax] == 1) continue;
    const int pos = g->coords[ax];
    if (transport == TP_TRANSPORT_NCCL)
      g->axis[ax] = make_nccl_comm(g->nccl, line_color(g.get(), ax), pos, g->dims[ax], pos, &st);
    else
      g->axis[ax] = make_local_comm(id128, world, g->group_members(ax), pos, cuda_device, &st);
    if (st != TP_OK) {
      tp_grid_destroy(g.release());
      return st;
    }
    g->axis[ax] = traced(std::move(g->axis[ax]));
  }
  if (world > 1) {  // all ranks: barriers of the fused peer-memory path, buffer registration
    if (transport == TP_TRANSPORT_NCCL) {
      g->all = make_nccl_world_comm(g->nccl);
    } else {
      std::vector<int> everyone(world);
      for (int r = 0; r < world; ++r) everyone[r] = r;
      g->all = make_local_comm(id128, world, everyone, rank, cuda_device, &st);
      if (st != TP_OK) {
        tp_grid_destroy(g.release());
        return st;
      }
    }
  }
  g->all = traced(std::move(g->all));
  if (transport == TP_TRANSPORT_LOCAL && world > 1) g_shared_device_grids.fetch_add(1);
  *out = g.release();
  return TP_OK;
}

tp_status tp_grid_coords(const tp_grid* g, int coords[3]) {
  if (!g || !coords) return fail(TP_ERR_ARG, "null argument");
  for (int k = 0; k < 3; ++k) coords[k] = k < g->ndims ? g->coords[k] : 0;
  return TP_OK;
}

tp_status tp_grid_dims(const tp_grid* g, int dims[3], int* ndims) {
  if (!g || !dims || !ndims) return fail(TP_ERR_ARG, "null argument");
  for (int k = 0; k < 3; ++k) dims[k] = k < g->ndims ? g->dims[k] : 1;
  *ndims = g->ndims;
  return TP_OK;
}

tp_status tp_grid_group(const tp_grid* g, int axis, int* members) {
  if (!g || !members) return fail(TP_ERR_ARG, "null argument");
  if (axis < 0 || axis >= g->ndims) return fail(TP_ERR_ARG, "axis out of range");
  auto m = g->group_members(axis);
  std::memcpy(members, m.data(), m.size() * sizeof(int));
  return TP_OK;
}

tp_status tp_axis_collective(tp_grid* g, int axis, tp_collective op, const void* send, void* recv,
                             size_t count, tp_dtype dt, int arg, void* stream) {
  tp::NvtxRange nvtx_("tp_axis_collective");
  if (!g) return fail(TP_ERR_ARG, "tp_axis_collective: null grid");
  if (axis < 0 || axis >= g->ndims) return fail(TP_ERR_ARG, "tp_axis_collective: axis out of range");
  if (dt != TP_BF16 && dt != TP_FP32) return fail(TP_ERR_ARG, "tp_axis_collective: dtype");
  if (op < TP_COLL_BCAST || op > TP_COLL_SHIFT) return fail(TP_ERR_ARG, "tp_axis_collective: op");
  if (count && (!recv || (op != TP_COLL_BCAST && !send)))
    return fail(TP_ERR_ARG, "tp_axis_collective: null buffer");
  const int n = g->dims[axis];
  if ((op == TP_COLL_BCAST || op == TP_COLL_REDUCE) && (arg < 0 || arg >= n))
    return fail(TP_ERR_ARG, "tp_axis_collective: root out of range");
  TP_CUDA(cudaSetDevice(g->device));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Comm* c = g->axis[axis].get();
  if (!c && n == 1 && g->transport == TP_TRANSPORT_NCCL) {
    if (!g->unit_axis[axis]) {
      tp_status st = TP_OK;
      g->unit_axis[axis] = make_nccl_self_comm(&st);
      if (st != TP_OK) return st;
    }
    c = g->unit_axis[axis].get();
  }
  if (!c) {  // a size-1 line without a communicator: the identity
    if (n != 1) return fail(TP_ERR_ARG, "tp_axis_collective: grid has no transport");
    if (op != TP_COLL_BCAST && count && send != recv)
      TP_CUDA(cudaMemcpyAsync(recv, send, count * dtype_size(dt), cudaMemcpyDeviceToDevice, s));
    return TP_OK;
  }
  switch (op) {
    case TP_COLL_BCAST: return c->bcast(recv, count, dt, arg, s);
    case TP_COLL_REDUCE: return c->reduce(send, recv, count, dt, arg, s);
    case TP_COLL_ALLREDUCE: return c->allreduce(send, recv, count, dt, s);
    case TP_COLL_ALLGATHER: return c->allgather(send, recv, count, dt, s);
    case TP_COLL_REDUCESCATTER: return c->reducescatter(send, recv, count, dt, s);
    case TP_COLL_SHIFT: return c->shift(send, recv, count, dt, arg, s);
  }
  return fail(TP_ERR_ARG, "tp_axis_collective: op");
}

tp_status tp_grid_check(const tp_grid* g) {
  if (!g) return fail(TP_ERR_ARG, "tp_grid_check: null grid");
  if (g->nccl) TP_TRY(nccl_world_async_error(g->nccl));
  for (const auto& a : g->axis)
    if (a) TP_TRY(a->async_error());
  return TP_OK;
}

tp_status tp_grid_abort(tp_grid* g) {
  if (!g) return fail(TP_ERR_ARG, "tp_grid_abort: null grid");
  for (auto& a : g->axis)
    if (a) a->abort();
  for (auto& a : g->unit_axis)
    if (a) a->abort();
  if (g->nccl) nccl_world_abort(g->nccl);
  return TP_OK;
}

tp_status tp_knob_set(const char* name, int value) {
  const int i = name ? knob_index(name) : -1;
  if (i < 0) return fail(TP_ERR_ARG, std::string("tp_knob_set: unknown knob ") + (name ? name : "(null)"));
  std::lock_guard<std::mutex> lk(g_knob_mu);
  KnobState& k = knob_state(i);
  k.value = value;
  k.overridden = true;
  return TP_OK;
}

tp_status tp_knob_get(const char* name, int* value) {
  const int i = name ? knob_index(name) : -1;
  if (i < 0 || !value) return fail(TP_ERR_ARG, "tp_knob_get: unknown knob or null output");
  std::lock_guard<std::mutex> lk(g_knob_mu);
  *value = knob_state(i).value;
  return TP_OK;
}

tp_status tp_knobs(char* buf, size_t cap, size_t* needed) {
  std::string j = "[";
  {
    std::lock_guard<std::mutex> lk(g_knob_mu);
    for (int i = 0; i < kNumKnobs; ++i) {
      const KnobState& k = knob_state(i);
      j += std::string(i ? "," : "") + "{\"name\":\"" + kKnobs[i].name + "\",\"value\":" +
           std::to_string(k.value) + ",\"default\":" + std::to_string(kKnobs[i].def) +
           ",\"source\":\"" + (k.overridden ? "api" : k.from_env ? "env" : "default") +
           "\",\"what\":\"" + kKnobs[i].what + "\"}";
    }
  }
  j += "]";
  if (needed) *needed = j.size() + 1;
  if (buf && cap) {
    const size_t n = std::min(cap - 1, j.size());
    std::memcpy(buf, j.data(), n);
    buf[n] = 0;
  }
  return TP_OK;
}

tp_status tp_grid_set_contract_check(tp_grid* g, int enable) {
  if (!g) return fail(TP_ERR_ARG, "null grid");
  g->contract_check = enable != 0;
  g->contract_calls = 0;
  return TP_OK;
}

tp_status tp_grid_destroy(tp_grid* g) {
  if (!g) return TP_OK;
  if (g->transport == TP_TRANSPORT_LOCAL && g->world > 1 && g->all) g_shared_device_grids.fetch_sub(1);
  if (g->comm_stream) cudaStreamSynchronize(g->comm_stream);
  for (auto& kv : g->ipc_cache) cudaIpcCloseMemHandle(kv.second);
  g->ipc_cache.clear();
  g->regs.clear();
  for (auto& a : g->axis) a.reset();
  for (auto& a : g->unit_axis) a.reset();
  g->all.reset();
  if (g->nccl) nccl_world_destroy(g->nccl);
  for (auto& e : g->events)
    if (e) cudaEventDestroy(e);
  if (g->comm_stream) cudaStreamDestroy(g->comm_stream);
  delete g;
  return TP_OK;
}

tp_status tp_shard_extent(const tp_grid* g, const tp_linear_desc* d, tp_tensor tensor,
                          int64_t* row0, int64_t* rows, int64_t* col0, int64_t* cols) {
  TP_TRY(check_desc(g, d));
  if (!row0 || !rows || !col0 || !cols) return fail(TP_ERR_ARG, "null output");
  Ext e;
  TP_TRY(extent(g, d, tensor, &e));
  *row0 = e.r0;
  *rows = e.rows;
  *col0 = e.c0;
  *cols = e.cols;
  return TP_OK;
}

tp_status tp_workspace_size(const tp_grid* g, const tp_linear_desc* d, size_t* ws_bytes,
                            size_t* saved_bytes) {
  TP_TRY(check_desc(g, d));
  if (!ws_bytes || !saved_bytes) return fail(TP_ERR_ARG, "null output");
  return plan_sizes(const_cast<tp_grid*>(g), d, ws_bytes, saved_bytes);
}

static tp_status ready_to_run(tp_grid* g, const tp_linear_desc* d, size_t ws_bytes, void* ws,
                              const void* saved, size_t* need_saved) {
  TP_TRY(check_desc(g, d));
  if (g->world > 1 && g->transport == TP_TRANSPORT_NONE)
    return fail(TP_ERR_ARG, "transport NONE can only compute when world == 1");
  size_t need_ws = 0;
  TP_TRY(plan_sizes(g, d, &need_ws, need_saved));
  if (ws_bytes < need_ws || (need_ws && !ws))
    return fail(TP_ERR_WORKSPACE, "ws_bytes " + std::to_string(ws_bytes) + " < required " +
                                      std::to_string(need_ws));
  if (*need_saved && !saved) return fail(TP_ERR_WORKSPACE, "saved buffer required");
  return TP_OK;
}

static void begin_run(Run& R, tp_grid* g, const tp_linear_desc* d, void* ws, void* saved,
                      cudaStream_t s) {
  R.g = g;
  R.d = d;
  R.s = s;
  const bool serial = (d->flags & TP_FLAG_SERIAL) || !g->comm_stream;
  R.cs = serial ? s : g->comm_stream;
  R.ws.base = static_cast<char*>(ws);
  R.saved.base = static_cast<char*>(saved);
}

tp_status tp_linear_fwd(tp_grid* g, const tp_linear_desc* d, const void* x, const void* w,
                        const void* bias, void* y, void* saved, void* ws, size_t ws_bytes,
                        void* stream) {
  tp::NvtxRange nvtx_("tp_linear_fwd");
  if (!g || !d) return fail(TP_ERR_ARG, "tp_linear_fwd: null grid or desc");
  TP_TRY(contract_check(g, kCallLinearFwd, d, {uint64_t(bias != nullptr)}));
  size_t need_saved = 0;
  TP_TRY(ready_to_run(g, d, ws_bytes, ws, saved, &need_saved));
  if ((d->M && d->K && !x) || (d->K && d->N && !w) || (d->M && d->N && !y))
    return fail(TP_ERR_ARG, "null shard pointer");
  TP_CUDA(cudaSetDevice(g->device));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Run R;
  begin_run(R, g, d, ws, saved, s);
  if (R.cs != s) {
    cudaEvent_t e = g->ev();
    TP_CUDA(cudaEventRecord(e, s));
    TP_CUDA(cudaStreamWaitEvent(R.cs, e, 0));
  }
  tp_status st = sched_fwd(R, x, w, bias, y);
  if (R.cs != s) {
    cudaEvent_t e = g->ev();
    cudaEventRecord(e, R.cs);
    cudaStreamWaitEvent(s, e, 0);
  }
  if (st == TP_OK && (d->flags & TP_FLAG_GELU)) {  // Y = gelu(Z); Z kept for the backward
    GeluLayout L;
    TP_TRY(gelu_layout(g, d, &L));
    if (L.n) TP_TRY(launch_gelu_fwd(y, static_cast<char*>(saved) + L.saved_off, L.n, d->dtype, s));
  }
  return st;
}

tp_status tp_linear_bwd(tp_grid* g, const tp_linear_desc* d, const void* dy, const void* x,
                        const void* w, const void* saved, void* dx, void* dw, void* dbias, void* ws,
                        size_t ws_bytes, void* stream) {
  tp::NvtxRange nvtx_("tp_linear_bwd");
  if (!g || !d) return fail(TP_ERR_ARG, "tp_linear_bwd: null grid or desc");
  TP_TRY(contract_check(g, kCallLinearBwd, d,
                        {uint64_t(dx != nullptr), uint64_t(dbias != nullptr)}));
  size_t need_saved = 0;
  TP_TRY(ready_to_run(g, d, ws_bytes, ws, saved, &need_saved));
  if ((d->M && d->N && !dy) || (d->K && d->N && !dw) || (d->M && d->K && !x) ||
      (d->K && d->N && !w))
    return fail(TP_ERR_ARG, "null shard pointer");
  TP_CUDA(cudaSetDevice(g->device));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Run R;
  begin_run(R, g, d, ws, const_cast<void*>(saved), s);
  if (R.cs != s) {
    cudaEvent_t e = g->ev();
    TP_CUDA(cudaEventRecord(e, s));
    TP_CUDA(cudaStreamWaitEvent(R.cs, e, 0));
  }
  if (d->flags & TP_FLAG_GELU) {  // dZ = dY * gelu'(Z), then the linear backward with dZ
    GeluLayout L;
    TP_TRY(gelu_layout(g, d, &L));
    void* dz = static_cast<char*>(ws) + L.ws_off;
    if (L.n)
      TP_TRY(launch_gelu_bwd(dy, static_cast<const char*>(saved) + L.saved_off, dz, L.n,
                             d->dtype, s));
    dy = dz;
    if (R.cs != s) {  // the comm stream must see dZ too
      cudaEvent_t e = g->ev();
      TP_CUDA(cudaEventRecord(e, s));
      TP_CUDA(cudaStreamWaitEvent(R.cs, e, 0));
    }
  }
  tp_status st = sched_bwd(R, dy, x, w, dx, dw, dbias);
  if (R.cs != s) {
    cudaEvent_t e = g->ev();
    cudaEventRecord(e, R.cs);
    cudaStreamWaitEvent(s, e, 0);
  }
  return st;
}

static tp_status pack_common(const tp_grid* g, const tp_linear_desc* d, tp_tensor t, bool pack,
                             const void* src, void* dst, void* stream) {
  TP_TRY(check_desc(g, d));
  Ext e;
  TP_TRY(extent(g, d, t, &e));
  if (e.rows * e.cols == 0) return TP_OK;
  if (!src || !dst) return fail(TP_ERR_ARG, "null pointer");
  const int64_t gcols = (t == TP_TENSOR_X) ? d->K : d->N;
  const size_t esz = dtype_size(d->dtype);
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (g->transport != TP_TRANSPORT_NONE) TP_CUDA(cudaSetDevice(g->device));
  if (pack) {
    const char* base = static_cast<const char*>(src) + (e.r0 * gcols + e.c0) * esz;
    return launch_copy2d(base, gcols, dst, e.cols, e.rows, e.cols, esz, s);
  }
  char* base = static_cast<char*>(dst) + (e.r0 * gcols + e.c0) * esz;
  return launch_copy2d(src, e.cols, base, gcols, e.rows, e.cols, esz, s);
}

tp_status tp_pack(const tp_grid* g, const tp_linear_desc* d, tp_tensor t, const void* global,
                  void* shard, void* stream) {
  tp::NvtxRange nvtx_("tp_pack");
  return pack_common(g, d, t, true, global, shard, stream);
}

tp_status tp_unpack(const tp_grid* g, const tp_linear_desc* d, tp_tensor t, const void* shard,
                    void* global, void* stream) {
  tp::NvtxRange nvtx_("tp_unpack");
  return pack_common(g, d, t, false, shard, global, stream);
}

tp_status tp_gemm(int trans_a, int trans_b, int64_t M, int64_t N, int64_t K, tp_dtype in_dtype,
                  const void* A, int64_t lda, const void* B, int64_t ldb, const float* C,
                  int64_t ldc, void* D, int64_t ldd, tp_dtype out_dtype, float alpha,
                  const void* bias, void* ws, size_t ws_bytes, void* stream) {
  tp::NvtxRange nvtx_("tp_gemm");
  if (in_dtype != TP_BF16 && in_dtype != TP_FP32) return fail(TP_ERR_ARG, "in_dtype");
  if (out_dtype != TP_BF16 && out_dtype != TP_FP32) return fail(TP_ERR_ARG, "out_dtype");
  GemmArgs a;
  a.M = M;
  a.N = N;
  a.K = K;
  a.A = A;
  a.lda = lda;
  a.trans_a = trans_a != 0;
  a.B = B;
  a.ldb = ldb;
  a.trans_b = trans_b != 0;
  a.C = C;
  a.ldc = ldc;
  a.D = D;
  a.ldd = ldd;
  a.in_dtype = in_dtype;
  a.out_dtype = out_dtype;
  a.alpha = alpha;
  a.bias = bias;
  a.ws = ws;
  a.ws_bytes = ws ? ws_bytes : 0;
  return gemm(a, static_cast<cudaStream_t>(stream));
}

size_t tp_gemm_ws_bytes(void) { return gemm_tc2_ws_bytes(); }

tp_status tp_colsum(const void* src, int64_t rows, int64_t cols, int64_t ld, tp_dtype dtype,
                    void* dst, void* stream) {
  if (rows < 0 || cols < 0 || ld < cols) return fail(TP_ERR_SHAPE, "colsum shape");
  if (!dst || (rows && cols && !src)) return fail(TP_ERR_ARG, "null pointer");
  // fp32 scratch: a small, cached per-thread device buffer
  thread_local float* scratch = nullptr;
  thread_local int64_t cap = 0;
  if (cap < cols) {
    if (scratch) cudaFree(scratch);
    TP_CUDA(cudaMalloc(&scratch, kColsumSlabs * std::max<int64_t>(cols, 1024) * sizeof(float)));
    cap = std::max<int64_t>(cols, 1024);
  }
  return launch_colsum(src, rows, cols, ld, dtype, dst, scratch, static_cast<cudaStream_t>(stream));
}

tp_status tp_fill(void* dst, tp_dtype dtype, int64_t rows, int64_t cols, int64_t ld, uint64_t seed,
                  int tensor_id, int kind, float scale, int64_t g_row0, int64_t g_col0,
                  int64_t g_cols, void* stream) {
  if (rows < 0 || cols < 0 || ld < cols) return fail(TP_ERR_SHAPE, "fill shape");
  if (!dst && rows && cols) return fail(TP_ERR_ARG, "null pointer");
  if (kind != 0 && kind != 1) return fail(TP_ERR_ARG, "kind must be 0 (uniform) or 1 (ternary)");
  if (g_col0 + cols > g_cols) return fail(TP_ERR_SHAPE, "block exceeds global columns");
  return launch_fill(dst, dtype, rows, cols, ld, seed, tensor_id, kind, scale, g_row0, g_col0,
                     g_cols, static_cast<cudaStream_t>(stream));
}

tp_status tp_l2_flush(void* scratch, size_t bytes, void* stream) {
  if (!scratch) return fail(TP_ERR_ARG, "null pointer");
  TP_CUDA(cudaMemsetAsync(scratch, static_cast<int>(g_launches.load() & 0xFF), bytes,
                          static_cast<cudaStream_t>(stream)));
  return TP_OK;
}

tp_status tp_prof_enable(int on) {
  g_prof_on.store(on != 0);
  return TP_OK;
}

tp_status tp_prof_reset(void) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  for (auto& r : g_prof) {
    cudaEventSynchronize(r.b);
    cudaEventDestroy(r.a);
    cudaEventDestroy(r.b);
  }
  g_prof.clear();
  return TP_OK;
}

tp_status tp_prof_read(int cls, double* total_ms, int64_t* launches, double* flops) {
  if (!total_ms || !launches || !flops) return fail(TP_ERR_ARG, "null output");
  std::lock_guard<std::mutex> lk(g_prof_mu);
  double ms = 0, fl = 0;
  int64_t n = 0;
  for (auto& r : g_prof) {
    if (r.cls != cls) continue;
    TP_CUDA(cudaEventSynchronize(r.b));
    float e = 0;
    TP_CUDA(cudaEventElapsedTime(&e, r.a, r.b));
    ms += e;
    fl += r.flops;
    ++n;
  }
  *total_ms = ms;
  *launches = n;
  *flops = fl;
  return TP_OK;
}

tp_status tp_prof_spans(int max, tp_span* out, int* n) {
  if (!n || (max > 0 && !out)) return fail(TP_ERR_ARG, "tp_prof_spans: null output");
  std::lock_guard<std::mutex> lk(g_prof_mu);
  *n = static_cast<int>(g_prof.size());
  if (g_prof.empty()) return TP_OK;
  for (auto& r : g_prof) TP_CUDA(cudaEventSynchronize(r.b));
  // the earliest start: every other start is measured from it
  size_t first = 0;
  for (size_t i = 1; i < g_prof.size(); ++i) {
    float d = 0;
    TP_CUDA(cudaEventElapsedTime(&d, g_prof[first].a, g_prof[i].a));
    if (d < 0) first = i;
  }
  for (int i = 0; i < *n && i < max; ++i) {
    const ProfRec& r = g_prof[i];
    float a = 0, b = 0;
    TP_CUDA(cudaEventElapsedTime(&a, g_prof[first].a, r.a));
    TP_CUDA(cudaEventElapsedTime(&b, g_prof[first].a, r.b));
    out[i] = tp_span{r.cls, r.rank, a, b, r.flops};
  }
  return TP_OK;
}

int64_t tp_launch_count(void) { return g_launches.load(); }

// ---- symmetric buffer registration (fused peer-memory path) ------------------------------
namespace {
struct RegRecord {
  cudaIpcMemHandle_t handle;
  uint64_t offset;  // ptr - allocation base
  uint64_t ptr;     // raw pointer (usable as-is by ranks of the same process)
  int64_t pid;
  int32_t device;
  int32_t pad;
};

tp_status alloc_range(const void* ptr, void** base) {
  static PFN_cuMemGetAddressRange_v3020 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuMemGetAddressRange_v3020>(p);
  });
  if (!fn) return fail(TP_ERR_CUDA, "cuMemGetAddressRange unavailable");
  CUdeviceptr b = 0;
  size_t sz = 0;
  if (fn(&b, &sz, reinterpret_cast<CUdeviceptr>(ptr)) != CUDA_SUCCESS)
    return fail(TP_ERR_ARG, "tp_register_buffer: not a device allocation");
  *base = reinterpret_cast<void*>(b);
  return TP_OK;
}
}  // namespace

tp_status tp_register_buffer(tp_grid* g, void* ptr, size_t bytes) {
  tp::NvtxRange nvtx_("tp_register_buffer");
  if (!g || !ptr || !bytes) return fail(TP_ERR_ARG, "tp_register_buffer: null argument");
  tp_grid::RegBuf rb;
  rb.base = static_cast<char*>(ptr);
  rb.bytes = bytes;
  rb.peer.assign(g->world, nullptr);
  rb.peer[g->rank] = rb.base;
  if (g->world > 1) {
    if (!g->all) return fail(TP_ERR_ARG, "tp_register_buffer: grid has no transport");
    TP_CUDA(cudaSetDevice(g->device));
    RegRecord mine{};
    mine.ptr = reinterpret_cast<uint64_t>(ptr);
    mine.pid = static_cast<int64_t>(getpid());
    mine.device = g->device;
    if (g->transport == TP_TRANSPORT_NCCL) {
      void* base = nullptr;
      TP_TRY(alloc_range(ptr, &base));
      TP_CUDA(cudaIpcGetMemHandle(&mine.handle, base));
      mine.offset = static_cast<uint64_t>(static_cast<char*>(ptr) - static_cast<char*>(base));
    }
    std::vector<RegRecord> all(g->world);
    TP_TRY(g->all->host_allgather(&mine, sizeof(RegRecord), all.data()));
    g->peer_device.assign(g->world, g->device);
    for (int r = 0; r < g->world; ++r) g->peer_device[r] = all[r].device;
    for (int r = 0; r < g->world; ++r) {
      if (r == g->rank) continue;
      if (all[r].pid == mine.pid) {  // same process (LOCAL transport / threads): share directly
        rb.peer[r] = reinterpret_cast<char*>(all[r].ptr);
        if (all[r].device != g->device) {
          cudaError_t e = cudaDeviceEnablePeerAccess(all[r].device, 0);
          if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
            return fail(TP_ERR_CUDA, std::string("peer access: ") + cudaGetErrorString(e));
          cudaGetLastError();
        }
        continue;
      }
      std::string key = std::to_string(r) + ":" +
                        std::string(reinterpret_cast<const char*>(&all[r].handle), sizeof(cudaIpcMemHandle_t));
      void* mapped = nullptr;
      for (auto& kv : g->ipc_cache)
        if (kv.first == key) mapped = kv.second;
      if (!mapped) {
        TP_CUDA(cudaIpcOpenMemHandle(&mapped, all[r].handle, cudaIpcMemLazyEnablePeerAccess));
        g->ipc_cache.emplace_back(key, mapped);
      }
      rb.peer[r] = static_cast<char*>(mapped) + all[r].offset;
    }
  }
  g->regs.push_back(std::move(rb));
  return TP_OK;
}

tp_status tp_peer_staged_bytes(const tp_grid* g, uint64_t* bytes) {
  if (!g || !bytes) return fail(TP_ERR_ARG, "tp_peer_staged_bytes: null argument");
  *bytes = g->staged_bytes;
  return TP_OK;
}

tp_status tp_deregister_all(tp_grid* g) {
  if (!g) return fail(TP_ERR_ARG, "grid is null");
  if (g->comm_stream) cudaStreamSynchronize(g->comm_stream);
  g->regs.clear();  // IPC mappings stay cached until tp_grid_destroy (cheap re-registration)
  return TP_OK;
}

tp_status tp_gemm_trace(unsigned long long* buf) {
  tp::g_gemm_trace = buf;
  return TP_OK;
}

}  // extern "C"

// ------------------------------------------------------------------------ analytic cost model
// Communication the schedules leave exposed (not hidden under a GEMM), one layer fwd + bwd, per
// rank: every collective costs its received bytes / link_gbs, every GEMM its flops / peak, and a
// collective that runs under a GEMM costs only what exceeds that GEMM (sched.cpp's overlap
// structure: SUMMA's next-step broadcast / previous-step reduce under each step's GEMM, 1D's
// AR(dX) under dW, 3D's row-block pipeline with AG(W) / AG(dY)-remainder / the last reduce /
// RS(dW) exposed; the depth collectives of 2.5D are exposed).
// Peer bytes of the fused owner-computes path per rank, layer fwd + bwd (sched.cpp fused_ab /
// fused_abt_atb / fused3_fwd / fused3_bwd): direct TMA panels are re-read once per 256-wide
// output tile they feed; staged, each distinct remote shard crosses once.
static void fused_peer_bytes(tp_mode mode, const tp_linear_desc* d, int q, int dd, double* direct,
                             double* staged) {
  *direct = *staged = 0;
  if (q < 2) return;
  const double M = double(d->M), K = double(d->K), N = double(d->N);
  const double e = d->dtype == TP_BF16 ? 2.0 : 4.0;
  auto t = [](double x) { return std::ceil(x / 256.0); };
  if ((mode == TP_2D || mode == TP_2P5D) && !(d->flags & (TP_FLAG_W25_DEPTH_SHARDED | TP_FLAG_SOLOMONIK))) {
    const double mb = M / (double(dd) * q), kq = K / q, nq = N / q, r = q - 1;
    *direct = r * (t(nq) * mb * kq + t(mb) * kq * nq)           // Y = sum_t X[i,t] W[t,j]
            + r * (t(kq) * mb * nq + t(mb) * kq * nq)           // dX = sum_t dY[i,t] W[j,t]^T
            + r * (t(nq) * mb * kq + t(kq) * mb * nq);          // dW = sum_t X[t,i]^T dY[t,j]
    *staged = r * (mb * kq + kq * nq) + r * (2 * mb * nq + kq * nq + mb * kq);
  } else if (mode == TP_3D && q == 2) {
    const double l = q, mb = M / (l * l), kl = K / l, kb = K / (l * l), nl = N / l;
    *direct = l * l * t(nl) * mb * kb + (l * l - 1) * t(mb) * kb * nl                 // forward
            + l * (l * t(kb) * mb * nl + l * t(mb) * kb * nl)                        // dX blocks
            + l * l * (t(nl) * mb * kb + t(kb) * mb * nl);                           // dW
    *staged = l * mb * kl + (l * l - 1) * kb * nl
            + l * mb * nl + (l * l - 1) * kb * nl + (l * l - 1) * mb * kl + (l * l - 1) * mb * nl;
  }
  *direct *= e;
  *staged *= e;
}

static double exposed_comm_us(tp_mode mode, const tp_linear_desc* d, int q, int dd, double p,
                              double peak_tflops, double link_gbs) {
  const double M = double(d->M), K = double(d->K), N = double(d->N);
  const double e = d->dtype == TP_BF16 ? 2.0 : 4.0;
  auto tl = [&](double elems) { return elems * e / (link_gbs * 1e9) * 1e6; };
  auto tf = [&](double m, double n, double k) { return 2.0 * m * n * k / (peak_tflops * 1e12) * 1e6; };
  auto over = [](double comm, double gemm) { return comm > gemm ? comm - gemm : 0.0; };
  double x = 0;
  switch (mode) {
    case TP_1D:
      if (d->split_1d == 0)  // bwd: AR(dX) [M,K] under the dW GEMM (K x N/p x M)
        x = over(tl(2.0 * (p - 1) / p * M * K), tf(K, N / p, M));
      else                   // fwd: AR(Y) [M,N] after the only GEMM
        x = tl(2.0 * (p - 1) / p * M * N);
      break;
    case TP_2D:
    case TP_2P5D: {
      const bool solo = d->flags & TP_FLAG_SOLOMONIK;
      const double mb = solo ? M / q : M / (double(dd) * q), kq = K / q, nq = N / q;
      const int steps = solo ? q / dd : q;
      // a broadcast panel is received by the q-1 non-roots: (q-1)/q of the steps per rank
      const double f = double(q - 1) / q;
      const double sx = mb * kq * f, sw = kq * nq * f, sy = mb * nq;
      const double rx = mb * kq, rw = kq * nq;  // reduce partials: every rank's time
      // fwd (AB): first step's X and W panels, then step t+1's under step t's GEMM
      x += tl(sx + sw);
      for (int t = 0; t + 1 < steps; ++t) x += over(tl(sx + sw), tf(mb, nq, kq));
      // ABT: W panel k+1 and reduce k-1 under GEMM k; first W and last reduce exposed
      x += tl(sw);
      for (int k = 0; k < steps; ++k)
        x += over(tl((k + 1 < steps ? sw : 0) + (k > 0 ? rx : 0)), tf(mb, kq, nq));
      x += tl(rx);
      // ATB: X panel k+1 and reduce k-1 under GEMM k
      x += tl(sx);
      for (int k = 0; k < steps; ++k)
        x += over(tl((k + 1 < steps ? sx : 0) + (k > 0 ? rw : 0)), tf(kq, nq, mb));
      x += tl(rw);
      if (mode == TP_2P5D && dd > 1) {
        if (solo) x += tl(2.0 * (dd - 1) / dd * sy) + tl(rx) + tl(rw);  // AR(Y), bcast dX, dW
        else if (d->flags & TP_FLAG_W25_DEPTH_SHARDED)
          x += 2.0 * tl(double(dd - 1) / dd * rw);                       // AG(W) + RS(dW)
        else
          x += tl(2.0 * (dd - 1) / dd * rw);                              // AR(dW)
      }
      break;
    }
    case TP_3D: {
      const double l = q, mb = M / (l * l), kl = K / l, kb = K / (l * l), nl = N / l;
      // fwd: AG(W) exposed; AG(X)'s remote blocks under block 0; reduce j under block j+1; last
      x += tl((l - 1) * kb * nl);
      x += over(tl((l - 1) * mb * kl), tf(mb, nl, kl));
      for (int i = 1; i < q; ++i) x += over(tl(mb * nl), tf(mb, nl, kl));
      x += tl(mb * nl);
      // bwd: AG(dY) remote blocks under dX block 0; reduce j under dX block j+1; the last dX
      // reduce under the dW GEMM; RS(dW) exposed
      x += over(tl((l - 1) * mb * nl), tf(mb, kl, nl));
      for (int i = 1; i < q; ++i) x += over(tl(mb * kl), tf(mb, kl, nl));
      x += over(tl(mb * kl), tf(kl, nl, l * mb));
      x += tl((l - 1) / l * kl * nl);
      break;
    }
  }
  return x;
}

// the paper's Table row next to what the library's schedules move,
// per-GPU link bytes, flops and at-rest shard sizes, and the roofline times.
// Written independently of oracle/closed_forms.py (tests compare the two).
extern "C" tp_status tp_cost_model(tp_mode mode, int world, int q, int d, const tp_linear_desc* desc,
                                   double peak_tflops, double link_gbs, tp_cost* out) {
  if (!desc || !out) return tp::fail(TP_ERR_ARG, "tp_cost_model: null desc or out");
  tp_grid g;
  TP_TRY(plan_grid(&g, mode, world, 0, q, d));
  TP_TRY(check_desc(&g, desc));
  const double M = double(desc->M), K = double(desc->K), N = double(desc->N);
  const double Sx = M * K, Sw = K * N, Sy = M * N, p = world;
  const double e = desc->dtype == TP_BF16 ? 2.0 : 4.0;
  const int j = g.q, dd = g.d;
  const bool row = desc->split_1d != 0;
  double cannon_acc = 0;  // Cannon backward accumulator elements (fp32 on the wire)
  tp_cost c{};
  switch (mode) {
    case TP_1D:  // col: AR of dX in bwd; row: AR of Y in fwd (one ring AR per layer, A3)
      c.paper_elems = 2.0 * (p - 1) * (row ? Sy : Sx);
      c.counted_elems = c.paper_elems;
      c.mem_x = row ? Sx / p : Sx;
      c.mem_w = Sw / p;
      c.mem_y = row ? Sy : Sy / p;
      break;
    case TP_2D:  // SUMMA: fwd bcast X,W; bwd bcast W + reduce dX, bcast X + reduce dW (A4)
      c.paper_elems = 3.0 * (j - 1) * (Sx + Sw);
      c.counted_elems = c.paper_elems;
      // Cannon (oracle/cannon.py): forward skew (q-1)/q + (q-1) unit shifts of X and W; backward
      // (reading N7) the same for W / X plus q accumulator shifts and the delivery (q-1)/q
      if (desc->flags & TP_FLAG_CANNON) {
        cannon_acc = (j + (j - 1.0) / j) * (Sx + Sw);
        c.counted_elems = 2.0 * ((j - 1.0) / j + (j - 1)) * (Sx + Sw) + cannon_acc;
      }
      c.mem_x = Sx / p;
      c.mem_w = Sw / p;
      c.mem_y = Sy / p;
      break;
    case TP_2P5D:  // d planes of SUMMA on S_x/d rows + depth AR(dW) or AG(W)+RS(dW) (A6, A11)
      if (desc->flags & TP_FLAG_SOLOMONIK) {
        // N5 (oracle/solomonik.py closed_form_volume): the q/d steps of every layer move
        // (q-1)(S_x+S_w)/d per product; depth AR of Y, depth bcasts of dX and dW. The Table has
        // no row for this scheme: paper_elems = the paper's 2.5D row, for comparison.
        c.paper_elems = 3.0 * (j - 1) * (Sx / dd + Sw);
        c.counted_elems = 3.0 * (j - 1) * (Sx + Sw) + 2.0 * (dd - 1) * Sy + (dd - 1) * (Sx + Sw);
        c.mem_x = Sx / (double(j) * j);
        c.mem_w = Sw / (double(j) * j);
        c.mem_y = Sy / (double(j) * j);
        break;
      }
      c.paper_elems = 3.0 * (j - 1) * (Sx / dd + Sw);
      c.counted_elems = dd * 3.0 * (j - 1) * (Sx / dd + Sw) + 2.0 * (dd - 1) * Sw;
      if (desc->flags & TP_FLAG_CANNON) {  // per plane as in 2D (reading N7), + the depth term
        cannon_acc = dd * (j + (j - 1.0) / j) * (Sx / dd + Sw);
        c.counted_elems = dd * 2.0 * ((j - 1.0) / j + (j - 1)) * (Sx / dd + Sw) + cannon_acc +
                          2.0 * (dd - 1) * Sw;
      }
      c.mem_x = Sx / p;
      c.mem_w = (desc->flags & TP_FLAG_W25_DEPTH_SHARDED) ? Sw / p : Sw / (double(j) * j);
      c.mem_y = Sy / p;
      break;
    case TP_3D:  // AG X, AG W, RS Y; AG dY, RS dX, RS dW: each tensor moves twice (A10)
      c.paper_elems = 2.0 * (j - 1) / j * (Sx + Sw + Sy);
      c.counted_elems = 2.0 * (j - 1) * (Sx + Sw + Sy);
      c.mem_x = Sx / p;
      c.mem_w = Sw / p;
      c.mem_y = Sy / p;
      break;
    default:
      return tp::fail(TP_ERR_ARG, "tp_cost_model: unknown mode");
  }
  // Cannon's backward carries fp32 accumulators: those elements cost 4 bytes
  c.link_bytes = (c.counted_elems - cannon_acc) / p * e + cannon_acc / p * 4.0;
  c.flops = 6.0 * M * K * N / p;
  if (peak_tflops > 0) c.t_tensor_us = c.flops / (peak_tflops * 1e12) * 1e6;
  if (link_gbs > 0) c.t_link_us = c.link_bytes / (link_gbs * 1e9) * 1e6;
  c.t_roof_us = c.t_tensor_us > c.t_link_us ? c.t_tensor_us : c.t_link_us;
  if (peak_tflops > 0 && link_gbs > 0 && world > 1)
    c.t_exposed_us = exposed_comm_us(mode, desc, j, dd, p, peak_tflops, link_gbs);
  fused_peer_bytes(mode, desc, j, dd, &c.fused_direct_bytes, &c.fused_staged_bytes);
  *out = c;
  return TP_OK;
}

// ------------------------------------------------------------------------------- LayerNorm
extern "C" tp_status tp_layernorm_ws_size(const tp_grid* g, const tp_linear_desc* d, tp_tensor t,
                                          size_t* ws_bytes) {
  if (!g || !d || !ws_bytes) return tp::fail(TP_ERR_ARG, "tp_layernorm_ws_size: null argument");
  return tp::layernorm_ws_bytes(g, d, t, ws_bytes);
}

extern "C" tp_status tp_layernorm_fwd(tp_grid* g, const tp_linear_desc* d, tp_tensor t, float eps,
                                      const void* x, const void* gamma, const void* beta, void* y,
                                      float* stats, void* ws, size_t ws_bytes, void* stream) {
  tp::NvtxRange nvtx_("tp_layernorm_fwd");
  if (!g || !d) return tp::fail(TP_ERR_ARG, "tp_layernorm_fwd: null grid or desc");
  TP_TRY(tp::contract_check(g, tp::kCallLnFwd, d, {uint64_t(t), tp::f32_word(eps),
                                                   uint64_t(stats != nullptr)}));
  if (d->dtype != TP_BF16 && d->dtype != TP_FP32) return tp::fail(TP_ERR_ARG, "unknown dtype");
  TP_CUDA(cudaSetDevice(g->device));
  return tp::layernorm_fwd(g, d, t, eps, x, gamma, beta, y, stats, ws, ws_bytes,
                           static_cast<cudaStream_t>(stream));
}

extern "C" tp_status tp_layernorm_bwd(tp_grid* g, const tp_linear_desc* d, tp_tensor t,
                                      const void* dy, const void* x, const void* gamma,
                                      const float* stats, void* dx, void* dgamma, void* dbeta,
                                      void* ws, size_t ws_bytes, void* stream) {
  tp::NvtxRange nvtx_("tp_layernorm_bwd");
  if (!g || !d) return tp::fail(TP_ERR_ARG, "tp_layernorm_bwd: null grid or desc");
  TP_TRY(tp::contract_check(g, tp::kCallLnBwd, d, {uint64_t(t), uint64_t(dgamma != nullptr),
                                                   uint64_t(dbeta != nullptr)}));
  if (d->dtype != TP_BF16 && d->dtype != TP_FP32) return tp::fail(TP_ERR_ARG, "unknown dtype");
  TP_CUDA(cudaSetDevice(g->device));
  return tp::layernorm_bwd(g, d, t, dy, x, gamma, stats, dx, dgamma, dbeta, ws, ws_bytes,
                           static_cast<cudaStream_t>(stream));
}

// ----------------------------------------------------------------------- Ring Self-Attention
extern "C" tp_status tp_rsa_ws_size(const tp_grid* g, const tp_rsa_desc* d, size_t* ws_bytes) {
  if (!ws_bytes) return tp::fail(TP_ERR_ARG, "tp_rsa_ws_size: null ws_bytes");
  return tp::rsa_ws_bytes(g, d, ws_bytes);
}

extern "C" tp_status tp_rsa_fwd(tp_grid* g, const tp_rsa_desc* d, const void* q, const void* k,
                                const void* v, void* out, float* lse, void* ws, size_t ws_bytes,
                                void* stream) {
  tp::NvtxRange nvtx_("tp_rsa_fwd");
  if (!g || !d) return tp::fail(TP_ERR_ARG, "tp_rsa_fwd: null grid or desc");
  TP_TRY(tp::contract_check(g, tp::kCallRsaFwd, nullptr,
                            {uint64_t(d->seq), uint64_t(d->d_k), uint64_t(d->heads),
                             uint64_t(d->dtype), tp::f32_word(d->scale)}));
  TP_CUDA(cudaSetDevice(g->device));
  return tp::rsa_fwd(g, d, q, k, v, out, ws, ws_bytes, static_cast<cudaStream_t>(stream), lse);
}

extern "C" tp_status tp_rsa_bwd(tp_grid* g, const tp_rsa_desc* d, const void* q, const void* k,
                                const void* v, const void* out, const float* lse, const void* dout,
                                void* dq, void* dk, void* dv, void* ws, size_t ws_bytes,
                                void* stream) {
  tp::NvtxRange nvtx_("tp_rsa_bwd");
  if (!g || !d) return tp::fail(TP_ERR_ARG, "tp_rsa_bwd: null grid or desc");
  TP_TRY(tp::contract_check(g, tp::kCallRsaBwd, nullptr,
                            {uint64_t(d->seq), uint64_t(d->d_k), uint64_t(d->heads),
                             uint64_t(d->dtype), tp::f32_word(d->scale)}));
  TP_CUDA(cudaSetDevice(g->device));
  return tp::rsa_bwd(g, d, q, k, v, dout, dq, dk, dv, ws, ws_bytes, static_cast<cudaStream_t>(stream),
                      out, lse);
}

// ---------------------------------------------------------------- multi-head attention core
extern "C" tp_status tp_attention_ws_size(const tp_grid* g, const tp_linear_desc* d, int64_t seq,
                                          int64_t heads, size_t* ws_bytes) {
  if (!ws_bytes) return tp::fail(TP_ERR_ARG, "tp_attention_ws_size: null ws_bytes");
  return tp::attention_ws_bytes(g, d, seq, heads, ws_bytes);
}

extern "C" tp_status tp_attention_fwd(tp_grid* g, const tp_linear_desc* d, int64_t seq,
                                      int64_t heads, float scale, const void* qkv, void* out,
                                      float* lse, void* ws, size_t ws_bytes, void* stream) {
  tp::NvtxRange nvtx_("tp_attention_fwd");
  if (!g) return tp::fail(TP_ERR_ARG, "tp_attention_fwd: null grid");
  TP_TRY(tp::contract_check(g, tp::kCallAttnFwd, d,
                            {uint64_t(seq), uint64_t(heads), tp::f32_word(scale)}));
  TP_CUDA(cudaSetDevice(g->device));
  return tp::attention_fwd(g, d, seq, heads, scale, qkv, out, lse, ws, ws_bytes,
                           static_cast<cudaStream_t>(stream));
}

extern "C" tp_status tp_attention_bwd(tp_grid* g, const tp_linear_desc* d, int64_t seq,
                                      int64_t heads, float scale, const void* qkv, const void* out,
                                      const float* lse, const void* dout, void* dqkv, void* ws,
                                      size_t ws_bytes, void* stream) {
  tp::NvtxRange nvtx_("tp_attention_bwd");
  if (!g) return tp::fail(TP_ERR_ARG, "tp_attention_bwd: null grid");
  TP_TRY(tp::contract_check(g, tp::kCallAttnBwd, d,
                            {uint64_t(seq), uint64_t(heads), tp::f32_word(scale)}));
  TP_CUDA(cudaSetDevice(g->device));
  return tp::attention_bwd(g, d, seq, heads, scale, qkv, out, lse, dout, dqkv, ws, ws_bytes,
                           static_cast<cudaStream_t>(stream));
}

extern "C" tp_status tp_add(const void* a, const void* b, void* out, size_t n, tp_dtype dt,
                            void* stream) {
  if (n && (!a || !b || !out)) return tp::fail(TP_ERR_ARG, "tp_add: null pointer");
  if (dt != TP_BF16 && dt != TP_FP32) return tp::fail(TP_ERR_ARG, "tp_add: dtype");
  return tp::launch_add(a, b, out, n, dt, static_cast<cudaStream_t>(stream));
}

namespace tp { extern volatile unsigned* g_flash_dbg; }
// tools only: progress markers of the fused attention kernel's first CTA (mapped host memory)
extern "C" tp_status tp_flash_debug(unsigned* host_mapped) {
  tp::g_flash_dbg = host_mapped;
  return TP_OK;
}
