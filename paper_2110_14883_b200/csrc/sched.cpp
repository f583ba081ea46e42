// Per-mode schedules of the tensor-parallel linear layer: which collective moves which shard,
// which local GEMM runs where, on which stream, in which order (SURVEY 8(a) a-3 .. a-13).
//
// Streams and overlap (a-13): all compute runs on the caller's stream `s`; collectives run on
// the grid's communication stream `cs`, ordered with events only (no host sync). SUMMA panels
// are double-buffered: the broadcast for step t+2 is issued into the buffer step t has
// finished with, so step t+1's transfer overlaps step t's GEMM; the reduce of step k's
// partial overlaps step k+1's GEMM. In 3D the reduce-scatter of dX overlaps the dW GEMM.
// Every collective's root uses its own shard in place (no staging copy).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "sched.h"

namespace tp {
namespace {

// ---- extents -----------------------------------------------------------------------------
bool divides(int64_t a, int64_t b) { return b > 0 && a % b == 0; }

struct Ctx {
  Run& R;
  tp_grid* g;
  const tp_linear_desc* d;
  tp_dtype dt;
  size_t esz;
  explicit Ctx(Run& r) : R(r), g(r.g), d(r.d), dt(r.d->dtype), esz(dtype_size(r.d->dtype)) {}

  void* ws(size_t elems, size_t es = 0) { return R.ws.take(elems * (es ? es : esz)); }
  void* sv(size_t elems) { return R.saved.take(elems * esz); }

  cudaEvent_t record(cudaStream_t st) {
    cudaEvent_t e = g->ev();
    cudaEventRecord(e, st);
    return e;
  }
  tp_status order(cudaStream_t from, cudaStream_t to) {  // `to` waits for work so far on `from`
    if (from == to) return TP_OK;
    TP_CUDA(cudaStreamWaitEvent(to, record(from), 0));
    return TP_OK;
  }
  // D[M,N] = alpha * (op(A).op(B) + C) + bias
  tp_status mm(int64_t M, int64_t N, int64_t K, const void* A, bool ta, const void* B, bool tb,
               void* D, tp_dtype out, float alpha, const float* C, const void* bias) {
    return gemm(args(M, N, K, A, ta, B, tb, D, out, alpha, C, bias), R.s);
  }
  // two independent products (a layer's dX and dW) -> one grouped launch when possible
  tp_status mm2(const GemmArgs& a, const GemmArgs& b) { return gemm_pair(a, b, R.s); }
  GemmArgs args(int64_t M, int64_t N, int64_t K, const void* A, bool ta, const void* B, bool tb,
                void* D, tp_dtype out, float alpha, const float* C, const void* bias) {
    GemmArgs a;
    a.M = M;
    a.N = N;
    a.K = K;
    a.A = A;
    a.trans_a = ta;
    a.lda = ta ? M : K;
    a.B = B;
    a.trans_b = tb;
    a.ldb = tb ? K : N;
    a.C = C;
    a.ldc = N;
    a.D = D;
    a.ldd = N;
    a.in_dtype = dt;
    a.out_dtype = out;
    a.alpha = alpha;
    a.bias = bias;
    a.ws = gws;
    a.ws_bytes = gws_bytes;
    a.reserve_sms = comm_sms(2.0 * double(M) * double(N) * double(K));
    return a;
  }
  // Bytes this rank's collectives move on `cs` while the next GEMM runs (set by the schedule
  // right before the GEMM it overlaps; 0 = nothing in flight under it).
  double ovb = 0;
  // SMs the GEMM leaves to the collective running under it, sized to the transfer: none when
  // nothing overlaps or the transport needs no SMs (LOCAL: copy engines + small sum kernels);
  // over NCCL, enough channels (one CTA each, ~40 GB/s per channel over NVLink 5) for the
  // transfer to finish within the GEMM at ~1.4 PFLOP/s, 2..16 (the NCCL communicators are
  // created with maxCTAs = 16). TP_COMM_SMS=n forces n.
  int comm_sms(double gemm_flops) const {
    if (g->world == 1 || R.cs == R.s || ovb <= 0) return 0;
    const int forced = knob("TP_COMM_SMS");
    if (forced >= 0) return forced;
    if (g->transport != TP_TRANSPORT_NCCL) return 0;
    const double t = std::max(gemm_flops / 1.4e15, 1e-6);
    const int k = static_cast<int>(std::ceil(ovb / (40e9 * t)));
    return std::min(16, std::max(2, k));
  }
  // ---- peer-panel staging (TP_FLAG_PEER_STAGED, or peers on another GPU): a fused panel GEMM
  // reads a local copy of every staged peer shard, pulled once by the copy engine on `cs`
  char* stage_base = nullptr;
  size_t stage_cap = 0, stage_used = 0;
  bool stage_copies = false;
  std::vector<std::pair<const void*, const void*>> staged;  // peer pointer -> local copy
  void carve_stage(size_t bytes) {
    stage_base = static_cast<char*>(R.ws.take(bytes));
    stage_cap = bytes;
  }
  bool must_stage(int owner) const {
    if (owner == g->rank) return false;
    if (d->flags & TP_FLAG_PEER_STAGED) return true;
    return owner < static_cast<int>(g->peer_device.size()) && g->peer_device[owner] != g->device;
  }
  // `owner`'s copy of the registered shard `mine` (bytes long) as this rank reads it: the peer
  // pointer, or (staged) a local copy. Call after the barrier that marks the shards ready.
  const void* shard(int owner, const void* mine, size_t bytes, tp_status* st) {
    const void* p = g->peer_ptr(owner, mine);
    if (!p || !must_stage(owner)) return p;
    for (const auto& kv : staged)
      if (kv.first == p) return kv.second;
    const size_t off = (stage_used + 255) & ~size_t(255);
    if (off + bytes > stage_cap) {
      *st = fail(TP_ERR_WORKSPACE, "peer staging: workspace too small");
      return nullptr;
    }
    char* dst = stage_base + off;
    stage_used = off + bytes;
    if (!stage_copies) {
      if (order(R.s, R.cs) != TP_OK) {
        *st = TP_ERR_CUDA;
        return nullptr;
      }
      stage_copies = true;
    }
    if (cudaMemcpyAsync(dst, p, bytes, cudaMemcpyDefault, R.cs) != cudaSuccess) {
      *st = fail(TP_ERR_CUDA, "peer staging copy failed");
      return nullptr;
    }
    g->staged_bytes += bytes;
    staged.emplace_back(p, dst);
    return dst;
  }
  // the panel GEMMs on `s` wait for the staging copies issued so far
  tp_status stage_done() {
    if (!stage_copies) return TP_OK;
    stage_copies = false;
    return order(R.cs, R.s);
  }
  // split-K scratch shared by this schedule's GEMMs (they run in order on `s`)
  void* gws = nullptr;
  size_t gws_bytes = 0;
  void carve_gemm_scratch() {
    if (dt != TP_BF16) return;
    gws_bytes = gemm_tc2_ws_bytes();
    gws = R.ws.take(gws_bytes);
  }
  // column sums of a [rows, cols] shard into out (dtype dt); fp32 scratch from ws
  float* colsum_scratch(int64_t cols) { return static_cast<float*>(ws(size_t(kColsumSlabs) * cols, 4)); }
  tp_status colsum(const void* src, int64_t rows, int64_t cols, void* out, float* scratch) {
    return launch_colsum(src, rows, cols, cols, dt, out, scratch, R.s);
  }
};

}  // namespace

tp_status check_divisible(const tp_grid* g, const tp_linear_desc* d) {
  const int64_t M = d->M, K = d->K, N = d->N;
  const int p = g->world, q = g->q, dd = g->d;
  auto bad = [&](const char* what, int64_t a, int64_t b) {
    return fail(TP_ERR_INDIVISIBLE, std::string(what) + "=" + std::to_string(a) +
                                         " not divisible by " + std::to_string(b));
  };
  if (M < 0 || K < 0 || N < 0) return fail(TP_ERR_SHAPE, "negative dimension");
  switch (g->mode) {
    case TP_1D:
      if (d->split_1d == 0 && !divides(N, p)) return bad("1D col: N", N, p);
      if (d->split_1d == 1 && !divides(K, p)) return bad("1D row: K", K, p);
      if (d->split_1d != 0 && d->split_1d != 1) return fail(TP_ERR_ARG, "split_1d must be 0 or 1");
      break;
    case TP_2D:
      if (!divides(M, q)) return bad("M", M, q);
      if (!divides(K, q)) return bad("K", K, q);
      if (!divides(N, q)) return bad("N", N, q);
      break;
    case TP_2P5D: {
      const bool sh = d->flags & TP_FLAG_W25_DEPTH_SHARDED;
      if (d->flags & TP_FLAG_SOLOMONIK) {  // replicated layers, depth-split SUMMA steps (N5)
        if (d->flags & (TP_FLAG_W25_DEPTH_SHARDED | TP_FLAG_CANNON | TP_FLAG_PEER_FUSED))
          return fail(TP_ERR_ARG, "TP_FLAG_SOLOMONIK excludes W25_DEPTH_SHARDED, CANNON, PEER_FUSED");
        if (q % dd)
          return fail(TP_ERR_CONSTRAINT, "Solomonik 2.5D: q = " + std::to_string(q) +
                                             " not divisible by d = " + std::to_string(dd));
        if (!divides(M, q)) return bad("M", M, q);
        if (!divides(K, q)) return bad("K", K, q);
        if (!divides(N, q)) return bad("N", N, q);
        break;
      }
      if (!divides(M, int64_t(dd) * q)) return bad("M", M, int64_t(dd) * q);
      if (!divides(N, q)) return bad("N", N, q);
      if (!divides(K, sh ? int64_t(q) * dd : q)) return bad("K", K, sh ? int64_t(q) * dd : q);
      break;
    }
    case TP_3D:
      if (!divides(M, int64_t(q) * q)) return bad("M", M, int64_t(q) * q);
      if (!divides(K, int64_t(q) * q)) return bad("K", K, int64_t(q) * q);
      if (!divides(N, q)) return bad("N", N, q);
      if (d->parity_3d != 0 && d->parity_3d != 1) return fail(TP_ERR_ARG, "parity_3d must be 0 or 1");
      break;
  }
  return TP_OK;
}

tp_status extent(const tp_grid* g, const tp_linear_desc* d, int tensor, Ext* e) {
  TP_TRY(check_divisible(g, d));
  if (tensor < TP_TENSOR_X || tensor > TP_TENSOR_BIAS) return fail(TP_ERR_ARG, "unknown tensor");
  const int64_t M = d->M, K = d->K, N = d->N;
  const int64_t fr[4] = {M, K, M, 1}, fc[4] = {K, N, N, N};
  auto set = [&](int64_t r0, int64_t rows, int64_t c0, int64_t cols) {
    e->r0 = r0;
    e->rows = rows;
    e->c0 = c0;
    e->cols = cols;
    return TP_OK;
  };
  const int* c = g->coords;
  switch (g->mode) {
    case TP_1D: {
      const int64_t r = c[0], p = g->world;
      if (d->split_1d == 0) {
        if (tensor == TP_TENSOR_X) return set(0, M, 0, K);
        if (tensor == TP_TENSOR_W) return set(0, K, r * N / p, N / p);
        if (tensor == TP_TENSOR_Y) return set(0, M, r * N / p, N / p);
        return set(0, 1, r * N / p, N / p);
      }
      if (tensor == TP_TENSOR_X) return set(0, M, r * K / p, K / p);
      if (tensor == TP_TENSOR_W) return set(r * K / p, K / p, 0, N);
      return set(0, fr[tensor], 0, fc[tensor]);
    }
    case TP_2D: {
      const int64_t i = c[0], j = c[1], q = g->q;
      if (tensor == TP_TENSOR_X) return set(i * M / q, M / q, j * K / q, K / q);
      if (tensor == TP_TENSOR_W) return set(i * K / q, K / q, j * N / q, N / q);
      if (tensor == TP_TENSOR_Y) return set(i * M / q, M / q, j * N / q, N / q);
      return set(0, 1, j * N / q, N / q);
    }
    case TP_2P5D: {
      const int64_t dep = c[0], i = c[1], j = c[2], q = g->q, dd = g->d;
      if (d->flags & TP_FLAG_SOLOMONIK) {  // the 2D block layout on every layer
        if (tensor == TP_TENSOR_X) return set(i * M / q, M / q, j * K / q, K / q);
        if (tensor == TP_TENSOR_W) return set(i * K / q, K / q, j * N / q, N / q);
        if (tensor == TP_TENSOR_Y) return set(i * M / q, M / q, j * N / q, N / q);
        return set(0, 1, j * N / q, N / q);
      }
      const int64_t mb = M / (dd * q);
      if (tensor == TP_TENSOR_X) return set((dep * q + i) * mb, mb, j * K / q, K / q);
      if (tensor == TP_TENSOR_W) {
        if (d->flags & TP_FLAG_W25_DEPTH_SHARDED) {
          const int64_t h = K / (q * dd);
          return set(i * K / q + dep * h, h, j * N / q, N / q);
        }
        return set(i * K / q, K / q, j * N / q, N / q);
      }
      if (tensor == TP_TENSOR_Y) return set((dep * q + i) * mb, mb, j * N / q, N / q);
      return set(0, 1, j * N / q, N / q);
    }
    case TP_3D: {
      const int64_t l = g->q, a = c[0];
      int64_t b = c[1], cc = c[2];
      if (d->parity_3d == 1) std::swap(b, cc);  // parity 1: roles of axes b and c swap
      const int64_t mb = M / (l * l), kb = K / (l * l);
      if (tensor == TP_TENSOR_X) return set((a * l + cc) * mb, mb, b * K / l, K / l);
      if (tensor == TP_TENSOR_W) return set((b * l + a) * kb, kb, cc * N / l, N / l);
      if (tensor == TP_TENSOR_Y) return set((a * l + b) * mb, mb, cc * N / l, N / l);
      return set(0, 1, cc * N / l, N / l);
    }
  }
  return fail(TP_ERR_ARG, "bad mode");
}

namespace {

// =========================================================================== 1D (a-3, a-4)
// ---- fused 1D reduce-scatter + all-gather over peer memory (TP_FLAG_PEER_FUSED, SURVEY
// 8(f) NEXT-1 for 1D: "RS fused into the GEMM epilogue (partial tiles stored to the peer)").
// The product whose partial sums the collective path all-reduces (1D column bwd: dX = sum_r
// dY_r W_r^T; 1D row fwd: Y = sum_r X_r W_r) is computed in full on every rank, but the GEMM
// epilogue stores the rows of block o straight into owner o's receive slot r (peer memory,
// D row-panels); owner o sums its p slots in rank order (fp32) into its row block of the
// output and every rank then copies the other row blocks from their owners. Moves the bytes
// of a ring reduce-scatter + all-gather (= the all-reduce) without collective kernels; the
// partials never round-trip through the sender's HBM. Needs `ws` (receive slots) and the
// output registered (tp_register_buffer), 2 <= p <= 8, (rows / p) % 32 == 0.
bool fused1d_ok(Ctx& C, const void* rx, const void* out, int64_t rows, int64_t cols) {
  const int p = C.g->world;
  if (!(C.d->flags & TP_FLAG_PEER_FUSED) || C.dt != TP_BF16 || !C.g->all || p < 2 || p > 8)
    return false;
  if (rows % p || (rows / p) % 32 || rows <= 128 || cols % 8) return false;
  return rx && out && C.g->peer_ptr(C.g->rank, rx) && C.g->peer_ptr(C.g->rank, out);
}

tp_status fused_rs_ag(Ctx& C, GemmArgs a, const GemmArgs* other, void* rx, void* out, int64_t rows,
                      int64_t cols) {
  const tp_grid* g = C.g;
  const int p = g->world, r = g->rank;
  const int64_t b = rows / p;
  const size_t blk = size_t(b) * cols * C.esz;
  a.dpanels = p;
  a.d_rows = b;
  a.ldd = cols;
  for (int o = 0; o < p; ++o)
    a.Dp[o] = const_cast<char*>(static_cast<const char*>(g->peer_ptr(o, rx))) + r * blk;
  a.D = a.Dp[0];
  a.reserve_sms = 0;
  TP_TRY(g->all->barrier(C.R.s));  // every owner's receive slots are free
  if (other) TP_TRY(gemm_pair(a, *other, C.R.s));
  else TP_TRY(gemm(a, C.R.s));
  TP_TRY(g->all->barrier(C.R.s));  // every partial has landed
  const void* in[8];
  for (int o = 0; o < p; ++o) in[o] = static_cast<const char*>(rx) + o * blk;
  TP_TRY(launch_sum_n(in, p, static_cast<char*>(out) + r * blk, size_t(b) * cols, C.dt, C.R.s));
  TP_TRY(g->all->barrier(C.R.s));  // every owner has summed its block
  for (int o = 0; o < p; ++o)
    if (o != r)
      TP_CUDA(cudaMemcpyAsync(static_cast<char*>(out) + o * blk,
                              static_cast<const char*>(g->peer_ptr(o, out)) + o * blk, blk,
                              cudaMemcpyDefault, C.R.s));
  return g->all->barrier(C.R.s);   // nobody overwrites a block a peer still reads
}

tp_status fwd_1d(Ctx& C, const void* x, const void* w, const void* bias, void* y) {
  const tp_linear_desc* d = C.d;
  const int p = C.g->world, r = C.g->coords[0];
  const int64_t M = d->M, K = d->K, N = d->N;
  if (d->split_1d == 0) {  // column-parallel: Y_r = X.W_r, no communication
    if (C.R.plan) return TP_OK;
    return C.mm(M, N / p, K, x, false, w, false, y, C.dt, d->alpha, nullptr, bias);
  }
  // row-parallel: Y = AR_p(X_r.W_r); bias enters once, on rank 0's partial
  const int64_t Kl = K / p;
  void* P = p > 1 ? C.ws(M * N) : y;
  if (C.R.plan) return TP_OK;
  if (p > 1 && fused1d_ok(C, P, y, M, N))
    return fused_rs_ag(C, C.args(M, N, Kl, x, false, w, false, nullptr, C.dt, d->alpha, nullptr,
                                 r == 0 ? bias : nullptr), nullptr, P, y, M, N);
  TP_TRY(C.mm(M, N, Kl, x, false, w, false, P, C.dt, d->alpha, nullptr, r == 0 ? bias : nullptr));
  if (p > 1) {
    TP_TRY(C.order(C.R.s, C.R.cs));
    TP_TRY(C.g->axis[0]->allreduce(P, y, M * N, C.dt, C.R.cs));
  }
  return TP_OK;
}

tp_status bwd_1d(Ctx& C, const void* dy, const void* x, const void* w, void* dx, void* dw,
                 void* dbias) {
  const tp_linear_desc* d = C.d;
  const int p = C.g->world;
  const int64_t M = d->M, K = d->K, N = d->N;
  if (d->split_1d == 0) {
    const int64_t Nl = N / p;
    void* P = (dx && p > 1) ? C.ws(M * K) : dx;
    float* scratch = dbias ? C.colsum_scratch(Nl) : nullptr;
    if (C.R.plan) return TP_OK;
    if (dx && p == 1) {  // no collective to overlap: dX and dW as one grouped launch
      TP_TRY(C.mm2(C.args(M, K, Nl, dy, false, w, true, dx, C.dt, d->alpha, nullptr, nullptr),
                   C.args(K, Nl, M, x, true, dy, false, dw, C.dt, d->alpha, nullptr, nullptr)));
      if (dbias) TP_TRY(C.colsum(dy, M, Nl, dbias, scratch));
      return TP_OK;
    }
    if (dx && fused1d_ok(C, P, dx, M, K)) {  // dX by the fused reduce-scatter + all-gather
      const GemmArgs gw = C.args(K, Nl, M, x, true, dy, false, dw, C.dt, d->alpha, nullptr, nullptr);
      TP_TRY(fused_rs_ag(C, C.args(M, K, Nl, dy, false, w, true, nullptr, C.dt, d->alpha, nullptr,
                                   nullptr), &gw, P, dx, M, K));
      if (dbias) TP_TRY(C.colsum(dy, M, Nl, dbias, scratch));
      return TP_OK;
    }
    if (dx) {  // dX = AR_p(dY_r . W_r^T): the column split's only collective
      TP_TRY(C.mm(M, K, Nl, dy, false, w, true, P, C.dt, d->alpha, nullptr, nullptr));
      if (p > 1) {
        TP_TRY(C.order(C.R.s, C.R.cs));
        TP_TRY(C.g->axis[0]->allreduce(P, dx, M * K, C.dt, C.R.cs));
      }
    }
    // dW_r = X^T . dY_r overlaps the all-reduce
    C.ovb = (dx && p > 1) ? 2.0 * (p - 1) / p * double(M) * double(K) * C.esz : 0.0;
    TP_TRY(C.mm(K, Nl, M, x, true, dy, false, dw, C.dt, d->alpha, nullptr, nullptr));
    C.ovb = 0;
    if (dbias) TP_TRY(C.colsum(dy, M, Nl, dbias, scratch));
    return TP_OK;
  }
  const int64_t Kl = K / p;
  float* scratch = dbias ? C.colsum_scratch(N) : nullptr;
  if (C.R.plan) return TP_OK;
  const GemmArgs gw = C.args(Kl, N, M, x, true, dy, false, dw, C.dt, d->alpha, nullptr, nullptr);
  if (dx)  // row-parallel backward is communication-free: dX_r and dW_r in one launch
    TP_TRY(C.mm2(C.args(M, Kl, N, dy, false, w, true, dx, C.dt, d->alpha, nullptr, nullptr), gw));
  else
    TP_TRY(gemm(gw, C.R.s));
  if (dbias) TP_TRY(C.colsum(dy, M, N, dbias, scratch));
  return TP_OK;
}

// =========================================================================== 2D / 2.5D
struct Plane {
  Comm* row;    // line along j (fixed i): X panels move here, dX partials reduce here
  Comm* col;    // line along i (fixed j): W panels move here, dW partials reduce here
  Comm* depth;  // 2.5D depth line (nullptr for 2D or d == 1)
  int i, j, q, d;
  int64_t mb, kq, nq;
  int t0, t1;  // SUMMA steps this rank's layer runs: all (q), or Solomonik's [dep q/d, +q/d)
};

Plane plane_of(Ctx& C) {
  Plane P{};
  const tp_grid* g = C.g;
  P.q = g->q;
  if (g->mode == TP_2D) {
    P.i = g->coords[0];
    P.j = g->coords[1];
    P.col = g->axis[0].get();
    P.row = g->axis[1].get();
    P.depth = nullptr;
    P.d = 1;
  } else {
    P.i = g->coords[1];
    P.j = g->coords[2];
    P.depth = g->axis[0].get();
    P.col = g->axis[1].get();
    P.row = g->axis[2].get();
    P.d = g->d;
  }
  P.mb = C.d->M / (int64_t(P.d) * P.q);
  if (C.g->mode == TP_2P5D && (C.d->flags & TP_FLAG_SOLOMONIK)) {  // layers replicate, steps split
    P.mb = C.d->M / P.q;
    P.t0 = g->coords[0] * (P.q / P.d);
    P.t1 = P.t0 + P.q / P.d;
  } else {
    P.t0 = 0;
    P.t1 = P.q;
  }
  P.kq = C.d->K / P.q;
  P.nq = C.d->N / P.q;
  return P;
}

// SUMMA "AB" (a-5): for t: bcast X[i,t] along row i, W[t,j] along column j; Y += X_t W_t.
tp_status summa_ab(Ctx& C, const Plane& P, const void* x, const void* W, const void* bias, void* y) {
  const float alpha = C.d->alpha;
  if (P.q == 1 && P.t1 - P.t0 == 1) {
    if (C.R.plan) return TP_OK;
    return C.mm(P.mb, P.nq, P.kq, x, false, W, false, y, C.dt, alpha, nullptr, bias);
  }
  void* bx[2] = {C.ws(P.mb * P.kq), C.ws(P.mb * P.kq)};
  void* bw[2] = {C.ws(P.kq * P.nq), C.ws(P.kq * P.nq)};
  float* acc = static_cast<float*>(C.ws(P.mb * P.nq, 4));
  if (C.R.plan) return TP_OK;
  cudaEvent_t ready[2] = {};
  auto xpan = [&](int t) { return P.j == t ? const_cast<void*>(x) : bx[t & 1]; };
  auto wpan = [&](int t) { return P.i == t ? const_cast<void*>(W) : bw[t & 1]; };
  auto issue = [&](int t) -> tp_status {
    TP_TRY(P.row->group_start());
    TP_TRY(P.row->bcast(xpan(t), P.mb * P.kq, C.dt, t, C.R.cs));
    TP_TRY(P.col->bcast(wpan(t), P.kq * P.nq, C.dt, t, C.R.cs));
    TP_TRY(P.row->group_end());
    ready[t & 1] = C.record(C.R.cs);
    return TP_OK;
  };
  TP_TRY(issue(P.t0));
  if (P.t0 + 1 < P.t1) TP_TRY(issue(P.t0 + 1));
  const double panels = double(P.mb * P.kq + P.kq * P.nq) * C.esz;
  for (int t = P.t0; t < P.t1; ++t) {
    TP_CUDA(cudaStreamWaitEvent(C.R.s, ready[t & 1], 0));
    const bool last = t == P.t1 - 1;
    C.ovb = last ? 0.0 : panels;  // step t+1's broadcasts run under this GEMM
    TP_TRY(C.mm(P.mb, P.nq, P.kq, xpan(t), false, wpan(t), false, last ? y : acc,
                last ? C.dt : TP_FP32, last ? alpha : 1.f, t > P.t0 ? acc : nullptr,
                last ? bias : nullptr));
    C.ovb = 0;
    if (t + 2 < P.t1) {
      TP_TRY(C.order(C.R.s, C.R.cs));  // panel buffers of step t are free again
      TP_TRY(issue(t + 2));
    }
  }
  return TP_OK;
}

// Cannon's forward (TP_FLAG_CANNON; "SUMMA and Cannon"): skew
// row i of X left by i and column j of W up by j, then q steps of (GEMM, shift X left by 1,
// W up by 1). Each step's shifts run on the comm stream under the step's GEMM (double
// buffers); oracle/cannon.py is the reference schedule.
tp_status cannon_ab(Ctx& C, const Plane& P, const void* x, const void* W, const void* bias, void* y) {
  const float alpha = C.d->alpha;
  if (P.q == 1) {
    if (C.R.plan) return TP_OK;
    return C.mm(P.mb, P.nq, P.kq, x, false, W, false, y, C.dt, alpha, nullptr, bias);
  }
  void* bx[2] = {C.ws(P.mb * P.kq), C.ws(P.mb * P.kq)};
  void* bw[2] = {C.ws(P.kq * P.nq), C.ws(P.kq * P.nq)};
  float* acc = static_cast<float*>(C.ws(P.mb * P.nq, 4));
  if (C.R.plan) return TP_OK;
  // skew (every member of a row shares i, of a column shares j: collective-consistent)
  TP_TRY(C.order(C.R.s, C.R.cs));
  const void* cx = x;
  const void* cw = W;
  int ix = 0, iw = 0;
  if (P.i) {
    TP_TRY(P.row->shift(x, bx[0], P.mb * P.kq, C.dt, P.i, C.R.cs));
    cx = bx[0];
    ix = 1;
  }
  if (P.j) {
    TP_TRY(P.col->shift(W, bw[0], P.kq * P.nq, C.dt, P.j, C.R.cs));
    cw = bw[0];
    iw = 1;
  }
  TP_TRY(C.order(C.R.cs, C.R.s));
  for (int t = 0; t < P.q; ++t) {
    const bool last = t == P.q - 1;
    cudaEvent_t moved = nullptr;
    void* nx = bx[ix];
    void* nw = bw[iw];
    if (!last) {  // next blocks move while this step's GEMM runs
      TP_TRY(C.order(C.R.s, C.R.cs));  // the previous GEMM is done with the buffers we refill
      TP_TRY(P.row->shift(cx, nx, P.mb * P.kq, C.dt, 1, C.R.cs));
      TP_TRY(P.col->shift(cw, nw, P.kq * P.nq, C.dt, 1, C.R.cs));
      moved = C.record(C.R.cs);
    }
    C.ovb = last ? 0.0 : double(P.mb * P.kq + P.kq * P.nq) * C.esz;  // next shifts under it
    TP_TRY(C.mm(P.mb, P.nq, P.kq, cx, false, cw, false, last ? y : acc, last ? C.dt : TP_FP32,
                last ? alpha : 1.f, t > 0 ? acc : nullptr, last ? bias : nullptr));
    C.ovb = 0;
    if (!last) {
      TP_CUDA(cudaStreamWaitEvent(C.R.s, moved, 0));
      cx = nx;
      cw = nw;
      ix ^= 1;
      iw ^= 1;
    }
  }
  return TP_OK;
}

// Cannon's backward (TP_FLAG_CANNON; reading N7, oracle/cannon.cannon_bwd): one product, the
// operand `B` circulating along `bline` (skew by `bskew`, then +1 per step) and the fp32
// accumulator along `aline` (+1 after every step, then a delivery shift by `deliver`).
//   ABT (dX = dY W^T): part_t = dY . W_t^T   [mb, kq]  W along the column, acc along the row
//   ATB (dW = X^T dY): part_t = X_t^T . dY   [kq, nq]  X along the row, acc along the column
// Step t: the GEMM writes part_t (fp32) while the accumulator of step t-1 and the operand of
// step t+1 travel on the comm stream; acc_t = part_t + acc_{t-1} (fp32 add), then shifted.
tp_status cannon_bwd_product(Ctx& C, const Plane& P, bool abt, const void* stat, const void* B,
                             void* out) {
  const int q = P.q;
  Comm* bline = abt ? P.col : P.row;
  Comm* aline = abt ? P.row : P.col;
  const int bskew = abt ? P.j : P.i;
  const int deliver = abt ? -P.i : -P.j;
  const int64_t bsz = abt ? P.kq * P.nq : P.mb * P.kq;   // circulating operand (dtype)
  const int64_t am = abt ? P.mb : P.kq, an = abt ? P.kq : P.nq;  // accumulator [am, an]
  const int64_t asz = am * an;
  void* bb[2] = {C.ws(bsz), C.ws(bsz)};
  float* part[2] = {static_cast<float*>(C.ws(asz, 4)), static_cast<float*>(C.ws(asz, 4))};
  float* recv[2] = {static_cast<float*>(C.ws(asz, 4)), static_cast<float*>(C.ws(asz, 4))};
  if (C.R.plan) return TP_OK;
  TP_TRY(C.order(C.R.s, C.R.cs));
  const void* cb = B;
  int ib = 0;
  if (bskew) {
    TP_TRY(bline->shift(B, bb[0], bsz, C.dt, bskew, C.R.cs));
    cb = bb[0];
    ib = 1;
  }
  TP_TRY(C.order(C.R.cs, C.R.s));
  cudaEvent_t acc_in = nullptr;
  for (int t = 0; t < q; ++t) {
    const bool last = t == q - 1;
    cudaEvent_t moved = nullptr;
    void* nb = bb[ib];
    if (!last) {  // the next operand block moves while this step's GEMM runs
      TP_TRY(C.order(C.R.s, C.R.cs));
      TP_TRY(bline->shift(cb, nb, bsz, C.dt, 1, C.R.cs));
      moved = C.record(C.R.cs);
    }
    float* pt = part[t & 1];
    C.ovb = double(last ? 0 : bsz) * C.esz + double(t > 0 ? asz : 0) * 4;
    if (abt)
      TP_TRY(C.mm(P.mb, P.kq, P.nq, stat, false, cb, true, pt, TP_FP32, 1.f, nullptr, nullptr));
    else
      TP_TRY(C.mm(P.kq, P.nq, P.mb, cb, true, stat, false, pt, TP_FP32, 1.f, nullptr, nullptr));
    C.ovb = 0;
    if (t > 0) {  // + the accumulator that arrived from the neighbour
      TP_CUDA(cudaStreamWaitEvent(C.R.s, acc_in, 0));
      TP_TRY(launch_add(pt, recv[(t - 1) & 1], pt, size_t(asz), TP_FP32, C.R.s));
    }
    TP_TRY(C.order(C.R.s, C.R.cs));
    TP_TRY(aline->shift(pt, recv[t & 1], asz, TP_FP32, 1, C.R.cs));
    acc_in = C.record(C.R.cs);
    if (!last) {
      TP_CUDA(cudaStreamWaitEvent(C.R.s, moved, 0));
      cb = nb;
      ib ^= 1;
    }
  }
  // deliver: the accumulator of this rank's block sits `deliver` positions away
  float* fin = recv[(q - 1) & 1];
  if (deliver % q) {
    float* dst = part[0];  // free: every step's reads of it completed before the last shift
    TP_TRY(aline->shift(fin, dst, asz, TP_FP32, deliver, C.R.cs));
    fin = dst;
  }
  TP_TRY(C.order(C.R.cs, C.R.s));
  // out = alpha * acc in the layer dtype (the GEMM epilogue with K = 0)
  return C.mm(am, an, 0, nullptr, false, nullptr, false, out, C.dt, C.d->alpha, fin, nullptr);
}

// SUMMA "ABT" (a-6): dX[i,k] = reduce_row( dY[i,j] . W[k,j]^T ), W panels down the columns.
tp_status summa_abt(Ctx& C, const Plane& P, const void* dy, const void* W, void* dx) {
  const float alpha = C.d->alpha;
  if (P.q == 1) {
    if (C.R.plan) return TP_OK;
    return C.mm(P.mb, P.kq, P.nq, dy, false, W, true, dx, C.dt, alpha, nullptr, nullptr);
  }
  void* bw[2] = {C.ws(P.kq * P.nq), C.ws(P.kq * P.nq)};
  void* bp[2] = {C.ws(P.mb * P.kq), C.ws(P.mb * P.kq)};
  if (C.R.plan) return TP_OK;
  cudaEvent_t ready[2] = {};
  auto wpan = [&](int k) { return P.i == k ? const_cast<void*>(W) : bw[k & 1]; };
  auto issue = [&](int k) -> tp_status {
    TP_TRY(P.col->bcast(wpan(k), P.kq * P.nq, C.dt, k, C.R.cs));
    ready[k & 1] = C.record(C.R.cs);
    return TP_OK;
  };
  TP_TRY(issue(P.t0));
  if (P.t0 + 1 < P.t1) TP_TRY(issue(P.t0 + 1));
  for (int k = P.t0; k < P.t1; ++k) {
    TP_CUDA(cudaStreamWaitEvent(C.R.s, ready[k & 1], 0));
    void* part = P.j == k ? dx : bp[k & 1];  // the root reduces in place into dX
    // under this GEMM: step k+1's W broadcast and step k-1's partial reduce
    C.ovb = double(k + 1 < P.t1 ? P.kq * P.nq : 0) * C.esz + double(k > P.t0 ? P.mb * P.kq : 0) * C.esz;
    TP_TRY(C.mm(P.mb, P.kq, P.nq, dy, false, wpan(k), true, part, C.dt, alpha, nullptr, nullptr));
    C.ovb = 0;
    TP_TRY(C.order(C.R.s, C.R.cs));
    TP_TRY(P.row->reduce(part, dx, P.mb * P.kq, C.dt, k, C.R.cs));
    if (k + 2 < P.t1) TP_TRY(issue(k + 2));
  }
  return TP_OK;
}

// SUMMA "ATB" (a-7): dW[k,j] = reduce_col( X[i,k]^T . dY[i,j] ), X panels along the rows.
tp_status summa_atb(Ctx& C, const Plane& P, const void* x, const void* dy, void* dwt) {
  const float alpha = C.d->alpha;
  if (P.q == 1) {
    if (C.R.plan) return TP_OK;
    return C.mm(P.kq, P.nq, P.mb, x, true, dy, false, dwt, C.dt, alpha, nullptr, nullptr);
  }
  void* bx[2] = {C.ws(P.mb * P.kq), C.ws(P.mb * P.kq)};
  void* bp[2] = {C.ws(P.kq * P.nq), C.ws(P.kq * P.nq)};
  if (C.R.plan) return TP_OK;
  cudaEvent_t ready[2] = {};
  auto xpan = [&](int k) { return P.j == k ? const_cast<void*>(x) : bx[k & 1]; };
  auto issue = [&](int k) -> tp_status {
    TP_TRY(P.row->bcast(xpan(k), P.mb * P.kq, C.dt, k, C.R.cs));
    ready[k & 1] = C.record(C.R.cs);
    return TP_OK;
  };
  TP_TRY(issue(P.t0));
  if (P.t0 + 1 < P.t1) TP_TRY(issue(P.t0 + 1));
  for (int k = P.t0; k < P.t1; ++k) {
    TP_CUDA(cudaStreamWaitEvent(C.R.s, ready[k & 1], 0));
    void* part = P.i == k ? dwt : bp[k & 1];
    C.ovb = double(k + 1 < P.t1 ? P.mb * P.kq : 0) * C.esz + double(k > P.t0 ? P.kq * P.nq : 0) * C.esz;
    TP_TRY(C.mm(P.kq, P.nq, P.mb, xpan(k), true, dy, false, part, C.dt, alpha, nullptr, nullptr));
    C.ovb = 0;
    TP_TRY(C.order(C.R.s, C.R.cs));
    TP_TRY(P.col->reduce(part, dwt, P.kq * P.nq, C.dt, k, C.R.cs));
    if (k + 2 < P.t1) TP_TRY(issue(k + 2));
  }
  return TP_OK;
}

// =========================================================================== fused peer SUMMA
// TP_FLAG_PEER_FUSED. Owner computes: every output block is ONE panel
// GEMM whose q K-panels are TMA-loaded straight from the shards of the ranks that own them
// (registered symmetric buffers, NVLink peer memory across GPUs):
//   Y[i,j]  = sum_t X[i,t] . W[t,j]        panels from ranks (i,t) and (t,j)
//   dX[i,j] = sum_n dY[i,n] . W[j,n]^T     panels from ranks (i,n) and (j,n)
//   dW[i,j] = sum_m X[m,i]^T . dY[m,j]     panels from ranks (m,i) and (m,j)
// SUMMA's q broadcasts become TMA reads inside the GEMM and its q reduces disappear (the
// whole contraction accumulates in TMEM); two stream-ordered barriers bracket the reads.
int plane_rank(const tp_grid* g, const Plane& P, int i, int j) {
  const int base = g->mode == TP_2P5D ? g->coords[0] * P.q * P.q : 0;
  return base + i * P.q + j;
}

bool fused_ok(Ctx& C, const Plane& P, std::initializer_list<const void*> shards,
              std::initializer_list<int64_t> rows) {
  if (!(C.d->flags & TP_FLAG_PEER_FUSED) || C.dt != TP_BF16 || !C.g->all) return false;
  if (C.g->mode == TP_2P5D && (C.d->flags & TP_FLAG_W25_DEPTH_SHARDED)) return false;
  if (P.q < 2 || P.q > 4) return false;
  if (P.kq % 8 || P.nq % 8) return false;  // TMA row strides
  for (int64_t r : rows)
    if (r <= 128) return false;  // CTA-pair kernel only (panels)
  for (const void* s : shards)
    if (!s || !C.g->peer_ptr(C.g->rank, s)) return false;
  return true;
}

tp_status fused_barrier(Ctx& C) { return C.g->all->barrier(C.R.s); }

// Panel t of A / B is the whole shard A_shard / B_shard of rank a_owner(t) / b_owner(t), of
// a_bytes / b_bytes (staged copies when the owner's shard must be pulled).
GemmArgs panel_args(Ctx& C, const Plane& P, int64_t M, int64_t N, int64_t K, bool ta, bool tb,
                    void* D, float alpha, const void* bias, const void* A_shard,
                    const void* B_shard, int (*a_owner)(const Plane&, int), int (*b_owner)(const Plane&, int),
                    size_t a_bytes, size_t b_bytes, tp_status* st) {
  GemmArgs a = C.args(M, N, K, nullptr, ta, nullptr, tb, D, C.dt, alpha, nullptr, bias);
  a.reserve_sms = 0;
  a.ws = nullptr;
  a.ws_bytes = 0;
  a.npanels = P.q;
  for (int t = 0; t < P.q; ++t) {
    a.Ap[t] = C.shard(a_owner(P, t), A_shard, a_bytes, st);
    a.Bp[t] = C.shard(b_owner(P, t), B_shard, b_bytes, st);
  }
  a.A = a.Ap[0];
  a.B = a.Bp[0];
  return a;
}

// owners of panel t, as global ranks, for the three products (P carries this rank's i, j)
thread_local const tp_grid* t_grid = nullptr;
int own_x_it(const Plane& P, int t) { return plane_rank(t_grid, P, P.i, t); }   // X[i,t]
int own_w_tj(const Plane& P, int t) { return plane_rank(t_grid, P, t, P.j); }   // W[t,j]
int own_dy_it(const Plane& P, int t) { return plane_rank(t_grid, P, P.i, t); }  // dY[i,t]
int own_w_jt(const Plane& P, int t) { return plane_rank(t_grid, P, P.j, t); }   // W[j,t]
int own_x_ti(const Plane& P, int t) { return plane_rank(t_grid, P, t, P.i); }   // X[t,i]
int own_dy_tj(const Plane& P, int t) { return plane_rank(t_grid, P, t, P.j); }  // dY[t,j]

tp_status fused_ab(Ctx& C, const Plane& P, const void* x, const void* w, const void* bias, void* y) {
  if (C.R.plan) return TP_OK;
  t_grid = C.g;
  TP_TRY(fused_barrier(C));  // every owner's shards are written
  tp_status st = TP_OK;
  GemmArgs a = panel_args(C, P, P.mb, P.nq, P.kq, false, false, y, C.d->alpha, bias, x, w, own_x_it,
                          own_w_tj, P.mb * P.kq * C.esz, P.kq * P.nq * C.esz, &st);
  TP_TRY(st);
  TP_TRY(C.stage_done());
  TP_TRY(gemm(a, C.R.s));
  return fused_barrier(C);   // every reader is done before anyone overwrites its shards
}

tp_status fused_abt_atb(Ctx& C, const Plane& P, const void* dy, const void* x, const void* w,
                        void* dx, void* dwt) {
  if (C.R.plan) return TP_OK;
  t_grid = C.g;
  const float alpha = C.d->alpha;
  TP_TRY(fused_barrier(C));
  tp_status st = TP_OK;
  const size_t xb = P.mb * P.kq * C.esz, wb = P.kq * P.nq * C.esz, yb = P.mb * P.nq * C.esz;
  GemmArgs gw = panel_args(C, P, P.kq, P.nq, P.mb, true, false, dwt, alpha, nullptr, x, dy,
                           own_x_ti, own_dy_tj, xb, yb, &st);
  TP_TRY(st);
  if (dx) {
    GemmArgs gx = panel_args(C, P, P.mb, P.kq, P.nq, false, true, dx, alpha, nullptr, dy, w,
                             own_dy_it, own_w_jt, yb, wb, &st);
    TP_TRY(st);
    TP_TRY(C.stage_done());
    TP_TRY(gemm_pair(gx, gw, C.R.s));  // both products in one grouped launch
  } else {
    TP_TRY(C.stage_done());
    TP_TRY(gemm(gw, C.R.s));
  }
  return fused_barrier(C);
}

// ---- fused depth-sharded 2.5D (TP_FLAG_W25_DEPTH_SHARDED + TP_FLAG_PEER_FUSED; the north
// star's 1/p weight layout). W[t,j] is split by rows over the d planes: rank (e,t,j) holds rows
// e hq .. e hq + hq - 1 of it (hq = K/(q d)), so each K-panel of the 2D product splits into d
// sub-panels read from d planes:
//   Y[dep,i,j]            = sum_t sum_e X[dep,i,t][:, e hq : +hq] . W_e[t,j]      (q d panels)
//   dX[dep,i,j][:, e hq:] = sum_n dY[dep,i,n] . W_e[j,n]^T                        (d GEMMs, q panels)
//   dW_dep[i,j]           = sum_e sum_m X[e,m,i][:, dep hq : +hq]^T . dY[e,m,j]  (q d panels)
// The depth all-gather of W (forward) and reduce-scatter of dW (backward) disappear: the peer
// panels cover them. Needs q d <= 4 (the kernel's K-panels), hq % 8 == 0 (16-byte sub-panel
// offsets) and > 128 output rows per product (CTA-pair kernel).
bool fused25_ok(Ctx& C, const Plane& P, std::initializer_list<const void*> shards,
                std::initializer_list<int64_t> rows) {
  if (!(C.d->flags & TP_FLAG_PEER_FUSED) || C.dt != TP_BF16 || !C.g->all) return false;
  if (C.g->mode != TP_2P5D || !(C.d->flags & TP_FLAG_W25_DEPTH_SHARDED) || P.d < 2) return false;
  if (P.q * P.d > 4) return false;
  const int64_t hq = P.kq / P.d;
  if (hq % 8 || P.kq % 8 || P.nq % 8) return false;
  for (int64_t r : rows)
    if (r <= 128) return false;
  for (const void* sh : shards)
    if (!sh || !C.g->peer_ptr(C.g->rank, sh)) return false;
  return true;
}

int rank25(const Plane& P, int e, int i, int j) { return e * P.q * P.q + i * P.q + j; }

GemmArgs panel_base(Ctx& C, int64_t M, int64_t N, int64_t K, bool ta, bool tb, void* D,
                    const void* bias, int64_t lda, int64_t ldb, int64_t ldd) {
  GemmArgs a = C.args(M, N, K, nullptr, ta, nullptr, tb, D, C.dt, C.d->alpha, nullptr, bias);
  a.reserve_sms = 0;
  a.ws = nullptr;
  a.ws_bytes = 0;
  a.lda = lda;
  a.ldb = ldb;
  a.ldd = ldd;
  return a;
}

tp_status fused25_fwd(Ctx& C, const Plane& P, const void* x, const void* w, const void* bias, void* y) {
  if (C.R.plan) return TP_OK;
  const tp_grid* g = C.g;
  const int dep = g->coords[0];
  const int64_t hq = P.kq / P.d;
  TP_TRY(fused_barrier(C));  // every owner's shards are written
  tp_status st = TP_OK;
  const size_t xb = P.mb * P.kq * C.esz, wb = hq * P.nq * C.esz;
  GemmArgs a = panel_base(C, P.mb, P.nq, hq, false, false, y, bias, P.kq, P.nq, P.nq);
  a.npanels = P.q * P.d;
  int k = 0;
  for (int t = 0; t < P.q; ++t)
    for (int e = 0; e < P.d; ++e, ++k) {
      a.Ap[k] = static_cast<const char*>(C.shard(rank25(P, dep, P.i, t), x, xb, &st)) + e * hq * C.esz;
      a.Bp[k] = C.shard(rank25(P, e, t, P.j), w, wb, &st);
    }
  TP_TRY(st);
  a.A = a.Ap[0];
  a.B = a.Bp[0];
  TP_TRY(C.stage_done());
  TP_TRY(gemm(a, C.R.s));
  return fused_barrier(C);   // every reader is done before anyone overwrites its shards
}

tp_status fused25_bwd(Ctx& C, const Plane& P, const void* dy, const void* x, const void* w,
                      void* dx, void* dw) {
  if (C.R.plan) return TP_OK;
  const tp_grid* g = C.g;
  const int dep = g->coords[0];
  const int64_t hq = P.kq / P.d;
  GemmArgs gs[1 + 4];  // dW + up to d = 4 dX column blocks (q d <= 4)
  int n = 0;
  TP_TRY(fused_barrier(C));
  tp_status st = TP_OK;
  const size_t xb = P.mb * P.kq * C.esz, yb = P.mb * P.nq * C.esz, wb = hq * P.nq * C.esz;
  // dW_dep[i,j] [hq, nq]: contraction over every plane's batch rows
  GemmArgs gw = panel_base(C, hq, P.nq, P.mb, true, false, dw, nullptr, P.kq, P.nq, P.nq);
  gw.npanels = P.q * P.d;
  int k = 0;
  for (int e = 0; e < P.d; ++e)
    for (int m = 0; m < P.q; ++m, ++k) {
      gw.Ap[k] = static_cast<const char*>(C.shard(rank25(P, e, m, P.i), x, xb, &st)) + dep * hq * C.esz;
      gw.Bp[k] = C.shard(rank25(P, e, m, P.j), dy, yb, &st);
    }
  gw.A = gw.Ap[0];
  gw.B = gw.Bp[0];
  gs[n++] = gw;
  if (dx) {
    for (int e = 0; e < P.d; ++e) {  // dX column block e: [mb, hq] at column e hq
      GemmArgs gx = panel_base(C, P.mb, hq, P.nq, false, true,
                               static_cast<char*>(dx) + e * hq * C.esz, nullptr, P.nq, P.nq, P.kq);
      gx.npanels = P.q;
      for (int t = 0; t < P.q; ++t) {
        gx.Ap[t] = C.shard(rank25(P, dep, P.i, t), dy, yb, &st);
        gx.Bp[t] = C.shard(rank25(P, e, P.j, t), w, wb, &st);
      }
      gx.A = gx.Ap[0];
      gx.B = gx.Bp[0];
      gs[n++] = gx;
    }
  }
  TP_TRY(st);
  TP_TRY(C.stage_done());
  for (int i0 = 0; i0 < n; i0 += 4)  // grouped launches of up to four problems
    TP_TRY(gemm_group(gs + i0, std::min(4, n - i0), C.R.s));
  return fused_barrier(C);
}

// ---- Solomonik-style 2.5D (TP_FLAG_SOLOMONIK, reading N5; oracle/
// solomonik.py): every layer holds the 2D block layout, layer dep runs SUMMA steps [t0, t1).
// Forward: the layer's partial Y (bias on layer 0 only) all-reduced over depth. Backward: the
// layer reduces dX[i,k] / dW[k,j] for its k's; every rank then receives its own block by a
// depth broadcast from the layer that owns its column (dX) / row (dW) index.
bool solomonik(const Ctx& C) { return C.g->mode == TP_2P5D && (C.d->flags & TP_FLAG_SOLOMONIK); }

tp_status fwd_solomonik(Ctx& C, const Plane& P, const void* x, const void* w, const void* bias, void* y) {
  void* yp = P.d > 1 ? C.ws(P.mb * P.nq) : y;
  TP_TRY(summa_ab(C, P, x, w, C.g->coords[0] == 0 ? bias : nullptr, yp));
  if (C.R.plan || P.d == 1) return TP_OK;
  TP_TRY(C.order(C.R.s, C.R.cs));
  return P.depth->allreduce(yp, y, P.mb * P.nq, C.dt, C.R.cs);
}

tp_status bwd_solomonik(Ctx& C, const Plane& P, const void* dy, const void* x, const void* w,
                        void* dx, void* dw, void* dbias) {
  float* scratch = dbias ? C.colsum_scratch(P.nq) : nullptr;
  void* dbt = (dbias && P.q > 1) ? C.ws(P.nq) : nullptr;
  if (dx) TP_TRY(summa_abt(C, P, dy, w, dx));
  TP_TRY(summa_atb(C, P, x, dy, dw));
  if (C.R.plan) return TP_OK;
  if (P.d > 1) {
    const int span = P.q / P.d;  // steps per layer: block index k is reduced on layer k / span
    TP_TRY(C.order(C.R.s, C.R.cs));
    if (dx) TP_TRY(P.depth->bcast(dx, P.mb * P.kq, C.dt, P.j / span, C.R.cs));
    TP_TRY(P.depth->bcast(dw, P.kq * P.nq, C.dt, P.i / span, C.R.cs));
  }
  if (dbias) {  // dY is replicated over depth: column sums reduced along the column only
    TP_TRY(C.colsum(dy, P.mb, P.nq, dbt ? dbt : dbias, scratch));
    if (dbt) {
      TP_TRY(C.order(C.R.s, C.R.cs));
      TP_TRY(P.col->allreduce(dbt, dbias, P.nq, C.dt, C.R.cs));
    }
  }
  return TP_OK;
}

tp_status fwd_2d(Ctx& C, const void* x, const void* w, const void* bias, void* y) {
  Plane P = plane_of(C);
  if (solomonik(C)) return fwd_solomonik(C, P, x, w, bias, y);
  if (fused_ok(C, P, {x, w}, {P.mb})) return fused_ab(C, P, x, w, bias, y);
  if (fused25_ok(C, P, {x, w}, {P.mb, P.kq / P.d})) return fused25_fwd(C, P, x, w, bias, y);
  const void* W = w;
  if (C.g->mode == TP_2P5D && (C.d->flags & TP_FLAG_W25_DEPTH_SHARDED) && P.d > 1) {
    // depth-sharded W: all-gather the depth pieces of W[i,j] (row-contiguous) into `saved`
    void* Wfull = C.sv(P.kq * P.nq);
    if (!C.R.plan) {
      TP_TRY(P.depth->allgather(w, Wfull, (P.kq / P.d) * P.nq, C.dt, C.R.cs));
      TP_TRY(C.order(C.R.cs, C.R.s));
    }
    W = Wfull;
  }
  if (C.d->flags & TP_FLAG_CANNON) return cannon_ab(C, P, x, W, bias, y);
  return summa_ab(C, P, x, W, bias, y);
}

tp_status bwd_2d(Ctx& C, const void* dy, const void* x, const void* w, const void* saved, void* dx,
                 void* dw, void* dbias) {
  Plane P = plane_of(C);
  if (solomonik(C)) return bwd_solomonik(C, P, dy, x, w, dx, dw, dbias);
  const bool sharded = C.g->mode == TP_2P5D && (C.d->flags & TP_FLAG_W25_DEPTH_SHARDED) && P.d > 1;
  const void* W = sharded ? saved : w;
  const bool depth = P.d > 1;
  void* dwt = depth ? C.ws(P.kq * P.nq) : dw;
  float* scratch = dbias ? C.colsum_scratch(P.nq) : nullptr;
  void* db_t[2] = {dbias ? C.ws(P.nq) : nullptr, dbias ? C.ws(P.nq) : nullptr};
  // the two SUMMA chains carve separate buffers so both pipelines can stay in flight
  const bool fused_sh = sharded && fused25_ok(C, P, {x, w, dy}, {P.mb, P.kq / P.d});
  if (sharded && !fused_sh && !C.R.plan && fused25_ok(C, P, {x, w}, {P.mb, P.kq / P.d})) {
    // the forward ran fused (no depth-gathered W in `saved`) but dY is not a registered
    // buffer: gather W here for the collective backward
    TP_TRY(C.order(C.R.s, C.R.cs));
    TP_TRY(P.depth->allgather(w, const_cast<void*>(saved), (P.kq / P.d) * P.nq, C.dt, C.R.cs));
    TP_TRY(C.order(C.R.cs, C.R.s));
  }
  if (fused_sh) {
    TP_TRY(fused25_bwd(C, P, dy, x, w, dx, dw));  // dW comes out as this plane's depth shard
  } else if (!sharded && fused_ok(C, P, {x, w, dy}, {P.mb, P.kq})) {
    TP_TRY(fused_abt_atb(C, P, dy, x, w, dx, dwt));
  } else if (P.q == 1 && dx) {  // one-rank plane: both products local and independent
    if (!C.R.plan)
      TP_TRY(C.mm2(C.args(P.mb, P.kq, P.nq, dy, false, W, true, dx, C.dt, C.d->alpha, nullptr, nullptr),
                   C.args(P.kq, P.nq, P.mb, x, true, dy, false, dwt, C.dt, C.d->alpha, nullptr, nullptr)));
  } else if (C.d->flags & TP_FLAG_CANNON) {  // NEXT-4: Cannon's backward (reading N7)
    if (dx) TP_TRY(cannon_bwd_product(C, P, true, dy, W, dx));
    TP_TRY(cannon_bwd_product(C, P, false, dy, x, dwt));
  } else {
    if (dx) TP_TRY(summa_abt(C, P, dy, W, dx));
    TP_TRY(summa_atb(C, P, x, dy, dwt));
  }
  if (C.R.plan) return TP_OK;
  if (depth && !fused_sh) {  // 2.5D: sum the planes' dW partials over depth (a-8)
    TP_TRY(C.order(C.R.s, C.R.cs));
    if (sharded)
      TP_TRY(P.depth->reducescatter(dwt, dw, (P.kq / P.d) * P.nq, C.dt, C.R.cs));
    else
      TP_TRY(P.depth->allreduce(dwt, dw, P.kq * P.nq, C.dt, C.R.cs));
  }
  if (dbias) {  // db[j] = sum over the ranks holding column block j (a-12)
    const bool need_col = P.q > 1, need_dep = depth;
    void* first = (need_col || need_dep) ? db_t[0] : dbias;
    TP_TRY(C.colsum(dy, P.mb, P.nq, first, scratch));
    if (need_col || need_dep) {
      TP_TRY(C.order(C.R.s, C.R.cs));
      const void* cur = first;
      if (need_col) {
        void* dst = need_dep ? db_t[1] : dbias;
        TP_TRY(P.col->allreduce(cur, dst, P.nq, C.dt, C.R.cs));
        cur = dst;
      }
      if (need_dep) TP_TRY(P.depth->allreduce(cur, dbias, P.nq, C.dt, C.R.cs));
    }
  }
  return TP_OK;
}

// =========================================================================== 3D (a-9, a-10)
struct Cube {
  Comm *cx, *cw, *cy;  // X-gather / W-gather / Y-scatter lines
  int ys_coord;         // this rank's coordinate along the Y-scatter axis
  int xg_coord;         // ... and along the X-gather axis
  int64_t l, mb, ml, kb, kl, nl;
};

Cube cube_of(Ctx& C) {
  const tp_grid* g = C.g;
  Cube Q{};
  const int ax_x = C.d->parity_3d == 0 ? 2 : 1;  // parity 0: X over c, Y over b
  const int ax_y = C.d->parity_3d == 0 ? 1 : 2;
  Q.cx = g->axis[ax_x].get();
  Q.cw = g->axis[0].get();
  Q.cy = g->axis[ax_y].get();
  Q.ys_coord = g->coords[ax_y];
  Q.xg_coord = g->coords[ax_x];
  Q.l = g->q;
  Q.mb = C.d->M / (Q.l * Q.l);
  Q.ml = C.d->M / Q.l;
  Q.kb = C.d->K / (Q.l * Q.l);
  Q.kl = C.d->K / Q.l;
  Q.nl = C.d->N / Q.l;
  return Q;
}

// ---- fused peer 3D (TP_FLAG_PEER_FUSED), owner computes, l = 2.
// Write the rank as (a, u, v): a = coords[0] (the W axis), u = X's column-block coordinate
// (b at parity 0, c at parity 1), v = the other. Then (extent table)
//   X(a,u,v) = rows (a l + v) M/l^2, cols u K/l;  W(a,u,v) = rows (u l + a) K/l^2, cols v N/l;
//   Y(a,u,v) = rows (a l + u) M/l^2, cols v N/l,
// and every output shard is ONE GEMM over l^2 (or l) K-panels read from the owners' shards:
//   Y  = sum_{u',a''} X(a,u',u)[:, a'' K/l^2 +: K/l^2] . W(a'',u',v)
//   dX[:, a'' K/l^2 +: K/l^2] = sum_{v'} dY(a,v,v') . W(a'',u,v')^T        (l problems)
//   dW = sum_{a',v'} X(a',u,v')[:, a K/l^2 +: K/l^2]^T . dY(a',v',v)
// Balanced (M N K / l^3 flops per rank, as the collective schedule) and collective-free; it
// reads (l-1)/l of X plus (l^2-1)/l^2 of the W column block -- more W bytes than AG+RS when
// W dominates, fewer passes through HBM (no gathered copies, no partials).
int cube_rank(const tp_grid* g, int parity, int a, int u, int v) {
  const int l = g->q;
  return parity == 0 ? (a * l + u) * l + v : (a * l + v) * l + u;
}

struct Cube3 {
  int a, u, v, par;
};

Cube3 cube3_of(const Ctx& C) {
  const tp_grid* g = C.g;
  Cube3 r;
  r.par = C.d->parity_3d;
  r.a = g->coords[0];
  r.u = r.par == 0 ? g->coords[1] : g->coords[2];
  r.v = r.par == 0 ? g->coords[2] : g->coords[1];
  return r;
}

bool fused3_ok(Ctx& C, const Cube& Q, std::initializer_list<const void*> shards) {
  if (!(C.d->flags & TP_FLAG_PEER_FUSED) || C.dt != TP_BF16 || !C.g->all || Q.l != 2) return false;
  if (Q.mb <= 128 || Q.kb <= 128) return false;           // CTA-pair kernel (fwd/dX and dW rows)
  if (Q.kb % 8 || Q.nl % 8 || Q.kl % 8) return false;     // TMA bases / strides (16 bytes)
  for (const void* s : shards)
    if (!s || !C.g->peer_ptr(C.g->rank, s)) return false;
  return true;
}

GemmArgs fused_args(Ctx& C, int64_t M, int64_t N, int64_t K, bool ta, bool tb, void* D,
                    int64_t lda, int64_t ldb, int64_t ldd, const void* bias) {
  GemmArgs a = C.args(M, N, K, nullptr, ta, nullptr, tb, D, C.dt, C.d->alpha, nullptr, bias);
  a.lda = lda;
  a.ldb = ldb;
  a.ldd = ldd;
  a.reserve_sms = 0;
  a.ws = nullptr;
  a.ws_bytes = 0;
  return a;
}

const void* at_col(const void* p, int64_t col, size_t esz) {
  return static_cast<const char*>(p) + col * static_cast<int64_t>(esz);
}

tp_status fused3_fwd(Ctx& C, const Cube& Q, const void* x, const void* w, const void* bias, void* y) {
  if (C.R.plan) return TP_OK;
  const tp_grid* g = C.g;
  const Cube3 r = cube3_of(C);
  const int l = static_cast<int>(Q.l);
  TP_TRY(fused_barrier(C));  // every owner's shards are written
  tp_status st = TP_OK;
  const size_t xb = Q.mb * Q.kl * C.esz, wb = Q.kb * Q.nl * C.esz;
  GemmArgs a = fused_args(C, Q.mb, Q.nl, Q.kb, false, false, y, Q.kl, Q.nl, Q.nl, bias);
  a.npanels = l * l;
  for (int u2 = 0; u2 < l; ++u2)
    for (int a2 = 0; a2 < l; ++a2) {
      const int p = u2 * l + a2;
      a.Ap[p] = at_col(C.shard(cube_rank(g, r.par, r.a, u2, r.u), x, xb, &st), a2 * Q.kb, C.esz);
      a.Bp[p] = C.shard(cube_rank(g, r.par, a2, u2, r.v), w, wb, &st);
    }
  TP_TRY(st);
  a.A = a.Ap[0];
  a.B = a.Bp[0];
  TP_TRY(C.stage_done());
  TP_TRY(gemm(a, C.R.s));
  return fused_barrier(C);   // every reader is done before anyone overwrites its shards
}

tp_status fused3_bwd(Ctx& C, const Cube& Q, const void* dy, const void* x, const void* w, void* dx,
                     void* dw, void* dbias, float* scratch, void* db_t) {
  if (C.R.plan) return TP_OK;
  const tp_grid* g = C.g;
  const Cube3 r = cube3_of(C);
  const int l = static_cast<int>(Q.l);
  GemmArgs gs[4];
  int n = 0;
  TP_TRY(fused_barrier(C));
  tp_status st = TP_OK;
  const size_t xb = Q.mb * Q.kl * C.esz, wb = Q.kb * Q.nl * C.esz, yb = Q.mb * Q.nl * C.esz;
  if (dx) {
    for (int a2 = 0; a2 < l; ++a2) {  // dX column sub-block a2 needs W rows owned by (a2,u,*)
      GemmArgs& d = gs[n++];
      d = fused_args(C, Q.mb, Q.kb, Q.nl, false, true, static_cast<char*>(dx) + a2 * Q.kb * C.esz,
                     Q.nl, Q.nl, Q.kl, nullptr);
      d.npanels = l;
      for (int v2 = 0; v2 < l; ++v2) {
        d.Ap[v2] = C.shard(cube_rank(g, r.par, r.a, r.v, v2), dy, yb, &st);
        d.Bp[v2] = C.shard(cube_rank(g, r.par, a2, r.u, v2), w, wb, &st);
      }
      d.A = d.Ap[0];
      d.B = d.Bp[0];
    }
  }
  GemmArgs& e = gs[n++];
  e = fused_args(C, Q.kb, Q.nl, Q.mb, true, false, dw, Q.kl, Q.nl, Q.nl, nullptr);
  e.npanels = l * l;
  for (int a1 = 0; a1 < l; ++a1)
    for (int v2 = 0; v2 < l; ++v2) {
      const int p = a1 * l + v2;
      e.Ap[p] = at_col(C.shard(cube_rank(g, r.par, a1, r.u, v2), x, xb, &st), r.a * Q.kb, C.esz);
      e.Bp[p] = C.shard(cube_rank(g, r.par, a1, v2, r.v), dy, yb, &st);
    }
  TP_TRY(st);
  e.A = e.Ap[0];
  e.B = e.Bp[0];
  TP_TRY(C.stage_done());
  TP_TRY(gemm_group(gs, n, C.R.s));  // the dX sub-blocks and dW in one persistent launch
  TP_TRY(fused_barrier(C));
  if (dbias) {  // db[v] = sum over the l^2 ranks holding column block v (axes a and u)
    void* db_u = static_cast<char*>(db_t) + ((Q.nl * C.esz + 255) & ~int64_t(255));
    TP_TRY(C.colsum(dy, Q.mb, Q.nl, db_t, scratch));
    TP_TRY(C.order(C.R.s, C.R.cs));
    TP_TRY(Q.cy->allreduce(db_t, db_u, Q.nl, C.dt, C.R.cs));
    TP_TRY(Q.cw->allreduce(db_u, dbias, Q.nl, C.dt, C.R.cs));
  }
  return TP_OK;
}

tp_status fwd_3d(Ctx& C, const void* x, const void* w, const void* bias, void* y) {
  Cube Q = cube_of(C);
  const float alpha = C.d->alpha;
  if (Q.l > 1 && fused3_ok(C, Q, {x, w})) return fused3_fwd(C, Q, x, w, bias, y);
  if (Q.l == 1) {
    if (C.R.plan) return TP_OK;
    return C.mm(C.d->M, C.d->N, C.d->K, x, false, w, false, y, C.dt, alpha, nullptr, bias);
  }
  void* Xg = C.sv(Q.ml * Q.kl);  // X[a,b] [M/l, K/l], kept for backward
  void* Wg = C.sv(Q.kl * Q.nl);  // W[b,c] [K/l, N/l]
  void* P = C.ws(Q.ml * Q.nl);
  if (C.R.plan) return TP_OK;
  // Pipelined by the row blocks of the gathered X (block j = X-gather member j's shard):
  //   cs: AG(W), then AG(X);   s: block `own` (this rank's own X rows: no wait for AG(X)),
  //   then the others; every block's partial P_j is reduced to Y-scatter member j (RS(P) over
  //   the Y line = one reduce per row block) while the next block's GEMM runs.
  // Exposed: AG(W) and the last block's reduce (vs AG(X) + AG(W) + the whole RS).
  // Every member of a Y line has the same `own` (the X-gather coordinate), so the lines' reduce
  // sequences agree.
  const int l = static_cast<int>(Q.l), own = Q.xg_coord;
  TP_TRY(C.order(C.R.s, C.R.cs));
  TP_TRY(Q.cw->allgather(w, Wg, Q.kb * Q.nl, C.dt, C.R.cs));
  cudaEvent_t ev_w = C.record(C.R.cs);
  TP_TRY(Q.cx->allgather(x, Xg, Q.mb * Q.kl, C.dt, C.R.cs));
  cudaEvent_t ev_x = C.record(C.R.cs);
  TP_CUDA(cudaStreamWaitEvent(C.R.s, ev_w, 0));
  for (int i = 0; i < l; ++i) {
    const int blk = (own + i) % l;
    if (i == 1) TP_CUDA(cudaStreamWaitEvent(C.R.s, ev_x, 0));
    const void* A = blk == own ? x : static_cast<const char*>(Xg) + blk * Q.mb * Q.kl * C.esz;
    void* Pb = static_cast<char*>(P) + blk * Q.mb * Q.nl * C.esz;
    C.ovb = i == 0 ? double((l - 1) * Q.mb * Q.kl) * C.esz : double(Q.mb * Q.nl) * C.esz;
    TP_TRY(C.mm(Q.mb, Q.nl, Q.kl, A, false, Wg, false, Pb, C.dt, alpha, nullptr,
                Q.ys_coord == 0 ? bias : nullptr));
    C.ovb = 0;
    TP_TRY(C.order(C.R.s, C.R.cs));
    TP_TRY(Q.cy->reduce(Pb, y, Q.mb * Q.nl, C.dt, blk, C.R.cs));
  }
  return TP_OK;
}

tp_status bwd_3d(Ctx& C, const void* dy, const void* x, const void* w, const void* saved, void* dx,
                 void* dw, void* dbias) {
  Cube Q = cube_of(C);
  const float alpha = C.d->alpha;
  if (Q.l == 1) {
    float* scratch = dbias ? C.colsum_scratch(C.d->N) : nullptr;
    if (C.R.plan) return TP_OK;
    const int64_t M = C.d->M, K = C.d->K, N = C.d->N;
    const GemmArgs gw = C.args(K, N, M, x, true, dy, false, dw, C.dt, alpha, nullptr, nullptr);
    if (dx)
      TP_TRY(C.mm2(C.args(M, K, N, dy, false, w, true, dx, C.dt, alpha, nullptr, nullptr), gw));
    else
      TP_TRY(gemm(gw, C.R.s));
    if (dbias) TP_TRY(C.colsum(dy, M, N, dbias, scratch));
    return TP_OK;
  }
  if (fused3_ok(C, Q, {x, w, dy})) {
    float* scr = dbias ? C.colsum_scratch(Q.nl) : nullptr;
    void* dbt = dbias ? C.ws(2 * ((Q.nl + 255) & ~int64_t(255))) : nullptr;  // two temporaries
    return fused3_bwd(C, Q, dy, x, w, dx, dw, dbias, scr, dbt);
  }
  const char* sv = static_cast<const char*>(saved);
  const void* Xg = sv;
  const void* Wg = sv ? sv + (((Q.ml * Q.kl * C.esz) + 255) & ~size_t(255)) : nullptr;
  if (!C.R.plan && fused3_ok(C, Q, {x, w})) {
    // the forward ran fused and left no gathered X / W in `saved`: gather them now
    TP_TRY(Q.cx->group_start());
    TP_TRY(Q.cx->allgather(x, const_cast<void*>(Xg), Q.mb * Q.kl, C.dt, C.R.cs));
    TP_TRY(Q.cw->allgather(w, const_cast<void*>(Wg), Q.kb * Q.nl, C.dt, C.R.cs));
    TP_TRY(Q.cx->group_end());
    TP_TRY(C.order(C.R.cs, C.R.s));  // the dX blocks below read W[b,c] without further waits
  }
  void* dYg = C.ws(Q.ml * Q.nl);
  void* Px = dx ? C.ws(Q.ml * Q.kl) : nullptr;
  void* Pw = C.ws(Q.kl * Q.nl);
  float* scratch = dbias ? C.colsum_scratch(Q.nl) : nullptr;
  void* dbt = dbias ? C.ws(Q.nl) : nullptr;
  if (C.R.plan) return TP_OK;
  // dY[a,c] = AG(dY over the Y line); block j comes from Y-line member j. The dX partial is
  // pipelined by those row blocks: block `ys` (this rank's own dY rows) first, without waiting
  // for the gather; each block's partial is reduced to X-line member j (RS(Px) over the X line =
  // one reduce per row block) under the next GEMM; the dW GEMM needs all of dY[a,c] and its
  // reduce-scatter over the W line is the one exposed collective.
  const int l = static_cast<int>(Q.l), ys = Q.ys_coord;
  TP_TRY(C.order(C.R.s, C.R.cs));
  TP_TRY(Q.cy->allgather(dy, dYg, Q.mb * Q.nl, C.dt, C.R.cs));
  cudaEvent_t ev_dy = C.record(C.R.cs);
  if (dx) {
    for (int i = 0; i < l; ++i) {
      const int blk = (ys + i) % l;
      if (i == 1) TP_CUDA(cudaStreamWaitEvent(C.R.s, ev_dy, 0));
      const void* A = blk == ys ? dy : static_cast<const char*>(dYg) + blk * Q.mb * Q.nl * C.esz;
      void* Pb = static_cast<char*>(Px) + blk * Q.mb * Q.kl * C.esz;
      C.ovb = i == 0 ? double((l - 1) * Q.mb * Q.nl) * C.esz : double(Q.mb * Q.kl) * C.esz;
      TP_TRY(C.mm(Q.mb, Q.kl, Q.nl, A, false, Wg, true, Pb, C.dt, alpha, nullptr, nullptr));
      C.ovb = 0;
      TP_TRY(C.order(C.R.s, C.R.cs));
      TP_TRY(Q.cx->reduce(Pb, dx, Q.mb * Q.kl, C.dt, blk, C.R.cs));
    }
  }
  TP_CUDA(cudaStreamWaitEvent(C.R.s, ev_dy, 0));
  C.ovb = dx ? double(Q.mb * Q.kl) * C.esz : 0.0;  // the last dX block's reduce
  TP_TRY(C.mm(Q.kl, Q.nl, Q.ml, Xg, true, dYg, false, Pw, C.dt, alpha, nullptr, nullptr));
  C.ovb = 0;
  if (dbias) TP_TRY(C.colsum(dYg, Q.ml, Q.nl, dbt, scratch));
  TP_TRY(C.order(C.R.s, C.R.cs));
  TP_TRY(Q.cw->reducescatter(Pw, dw, Q.kb * Q.nl, C.dt, C.R.cs));
  if (dbias) TP_TRY(Q.cw->allreduce(dbt, dbias, Q.nl, C.dt, C.R.cs));
  return TP_OK;
}

}  // namespace

// Upper bound of the peer shards one fused call may stage (every panel's whole shard; 256 B
// alignment slack each). 0 when the call cannot take a fused panel path.
size_t stage_bound(Ctx& C, bool fwd) {
  if (!(C.d->flags & TP_FLAG_PEER_FUSED) || C.g->world == 1 || C.dt != TP_BF16) return 0;
  double elems = 0, shards = 0;
  if (C.g->mode == TP_2D || C.g->mode == TP_2P5D) {
    const Plane P = plane_of(C);
    const double q = P.q, d = P.d, mb = P.mb, kq = P.kq, nq = P.nq;
    if (fwd) {
      elems = q * mb * kq + q * kq * nq;
      shards = q + q * d;
    } else {
      elems = (q + q * d) * mb * nq + q * kq * nq + q * d * mb * kq;
      shards = 2 * q + 3 * q * d;
    }
  } else if (C.g->mode == TP_3D) {
    const Cube Q = cube_of(C);
    const double l = Q.l, mb = Q.mb, kl = Q.kl, kb = Q.kb, nl = Q.nl;
    if (fwd) {
      elems = l * mb * kl + l * l * kb * nl;
      shards = l + l * l;
    } else {
      elems = l * mb * nl + l * l * kb * nl + l * l * mb * kl + l * l * mb * nl;
      shards = l + 3 * l * l;
    }
  }
  return static_cast<size_t>(elems) * C.esz + static_cast<size_t>(shards) * 256;
}

tp_status sched_fwd(Run& R, const void* x, const void* w, const void* bias, void* y) {
  Ctx C(R);
  C.carve_gemm_scratch();
  if (const size_t sb = stage_bound(C, true)) C.carve_stage(sb);
  switch (R.g->mode) {
    case TP_1D: return fwd_1d(C, x, w, bias, y);
    case TP_2D:
    case TP_2P5D: return fwd_2d(C, x, w, bias, y);
    case TP_3D: return fwd_3d(C, x, w, bias, y);
  }
  return fail(TP_ERR_ARG, "bad mode");
}

tp_status sched_bwd(Run& R, const void* dy, const void* x, const void* w, void* dx, void* dw,
                    void* dbias) {
  Ctx C(R);
  C.carve_gemm_scratch();
  if (const size_t sb = stage_bound(C, false)) C.carve_stage(sb);
  const void* saved = R.saved.base;
  switch (R.g->mode) {
    case TP_1D: return bwd_1d(C, dy, x, w, dx, dw, dbias);
    case TP_2D:
    case TP_2P5D: return bwd_2d(C, dy, x, w, saved, dx, dw, dbias);
    case TP_3D: return bwd_3d(C, dy, x, w, saved, dx, dw, dbias);
  }
  return fail(TP_ERR_ARG, "bad mode");
}

}  // namespace tp
