// Ring Self-Attention forward (sequence parallelism; P:L596-615,
// S:L361-414): Q, K, V are split along the sequence over the p ranks of a 1D grid (ring =
// grid axis 0); for every (batch, head) problem h a rank holds rows [r b, (r+1) b) of
// Q_h, K_h, V_h [s, d] (b = s / p) and produces the same rows of softmax(Q_h K_h^T scale) V_h.
//
// Schedule (the paper's, reading N3: scores are assembled before the softmax, then V
// circulates), per chunk of heads whose fp32 score rows fit the workspace budget:
//   pass 1: p steps; at step t the rank holds the K block that originated on rank
//           j = (r - t) mod p and writes S[:, j b : (j+1) b] = scale Q K_j^T (tcgen05 GEMM,
//           fp32 out); then every rank sends that block to its successor (ring shift,
//           double-buffered; N-1 shifts);
//   softmax over each assembled row [s] (fp32, max-subtracted) -> P (bf16 for the tensor
//           cores, fp32 in fp32 mode);
//   pass 2: p steps over the V ring; O += P[:, j b : (j+1) b] V_j with the fp32 accumulator
//           in the GEMM's C input; the last step writes O in the output dtype.
// Traffic: every score is written (fp32), read by the softmax, written as P and read by the
// PV GEMM; the ring moves 2 (p-1) s d elements per head.
#include <cuda_bf16.h>

#include <algorithm>
#include <cstdlib>
#include <cmath>

#include "sched.h"
#include "tp_internal.h"

namespace tp {
namespace {

constexpr size_t kScoreBudget = size_t(1) << 30;  // fp32 score rows per head chunk (bytes)

template <typename T>
__device__ __forceinline__ void st_out(T* p, float v) {
  if constexpr (sizeof(T) == 2) *reinterpret_cast<__nv_bfloat16*>(p) = __float2bfloat16_rn(v);
  else *p = v;
}

__device__ __forceinline__ float wmax(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float wsum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Row-resident softmax: 256 threads hold one fp32 row of VPT float4 each (s <= 1024 * VPT).
template <typename T, int VPT>
__global__ void __launch_bounds__(256) softmax_rows(const float* __restrict__ S, int64_t rows,
                                                    int64_t s, T* __restrict__ P) {
  __shared__ float red[8];
  __shared__ float bc;
  const int64_t r = blockIdx.x;
  if (r >= rows) return;
  const int64_t nvec = s / 4;
  const float4* row = reinterpret_cast<const float4*>(S + r * s);
  float4 v[VPT];
  float m = -INFINITY;
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const int64_t k = threadIdx.x + int64_t(i) * 256;
    if (k < nvec) {
      v[i] = __ldg(row + k);
      m = fmaxf(m, fmaxf(fmaxf(v[i].x, v[i].y), fmaxf(v[i].z, v[i].w)));
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  m = wmax(m);
  if (lane == 0) red[warp] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = red[0];
    for (int w = 1; w < 8; ++w) t = fmaxf(t, red[w]);
    bc = t;
  }
  __syncthreads();
  m = bc;
  float z = 0.f;
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const int64_t k = threadIdx.x + int64_t(i) * 256;
    if (k < nvec) {
      v[i].x = __expf(v[i].x - m);
      v[i].y = __expf(v[i].y - m);
      v[i].z = __expf(v[i].z - m);
      v[i].w = __expf(v[i].w - m);
      z += (v[i].x + v[i].y) + (v[i].z + v[i].w);
    }
  }
  z = wsum(z);
  __syncthreads();
  if (lane == 0) red[warp] = z;
  __syncthreads();
  if (threadIdx.x == 0) {
    float t = 0.f;
    for (int w = 0; w < 8; ++w) t += red[w];
    bc = 1.f / t;
  }
  __syncthreads();
  const float inv = bc;
  T* out = P + r * s;
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const int64_t k = threadIdx.x + int64_t(i) * 256;
    if (k < nvec) {
      st_out(out + 4 * k, v[i].x * inv);
      st_out(out + 4 * k + 1, v[i].y * inv);
      st_out(out + 4 * k + 2, v[i].z * inv);
      st_out(out + 4 * k + 3, v[i].w * inv);
    }
  }
}

// General softmax: one warp per row, three passes over the row.
template <typename T>
__global__ void softmax_rows_warp(const float* __restrict__ S, int64_t rows, int64_t s,
                                  T* __restrict__ P) {
  const int64_t r = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const float* row = S + r * s;
  float m = -INFINITY;
  for (int64_t c = lane; c < s; c += 32) m = fmaxf(m, row[c]);
  m = wmax(m);
  float z = 0.f;
  for (int64_t c = lane; c < s; c += 32) z += __expf(row[c] - m);
  const float inv = 1.f / wsum(z);
  for (int64_t c = lane; c < s; c += 32) st_out(P + r * s + c, __expf(row[c] - m) * inv);
}

tp_status launch_softmax(const float* S, int64_t rows, int64_t s, tp_dtype dt, void* P,
                         cudaStream_t st) {
  if (!rows || !s) return TP_OK;
  const bool vec = (s % 4 == 0) && (reinterpret_cast<uintptr_t>(S) % 16 == 0);
  const int64_t nvec = s / 4;
  const unsigned R = static_cast<unsigned>(rows);
#define SM(T, VP) softmax_rows<T, VP><<<R, 256, 0, st>>>(S, rows, s, static_cast<T*>(P))
#define SM_T(T)                                        \
  if (nvec <= 256) SM(T, 1);                           \
  else if (nvec <= 512) SM(T, 2);                      \
  else if (nvec <= 1024) SM(T, 4);                     \
  else if (nvec <= 2048) SM(T, 8);                     \
  else SM(T, 16)
  if (vec && nvec <= 4096) {
    if (dt == TP_BF16) {
      SM_T(__nv_bfloat16);
    } else {
      SM_T(float);
    }
  } else {
    const unsigned G = static_cast<unsigned>((rows * 32 + 255) / 256);
    if (dt == TP_BF16)
      softmax_rows_warp<__nv_bfloat16><<<G, 256, 0, st>>>(S, rows, s, static_cast<__nv_bfloat16*>(P));
    else
      softmax_rows_warp<float><<<G, 256, 0, st>>>(S, rows, s, static_cast<float*>(P));
  }
#undef SM_T
#undef SM
  count_launch();
  TP_CUDA(cudaGetLastError());
  return TP_OK;
}

// dS = scale * P * (dP - rowsum(P * dP)) per row (in place over P); dP fp32.
template <typename T>
__global__ void rsa_dscore(T* __restrict__ P, const float* __restrict__ dP, int64_t rows, int64_t s,
                           float scale) {
  const int64_t r = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  T* pr = P + r * s;
  const float* dr = dP + r * s;
  // a zero probability contributes nothing (and marks the padding columns, whose dP is -inf)
  float dsum = 0.f;
  for (int64_t c = lane; c < s; c += 32) {
    float pv;
    if constexpr (sizeof(T) == 2) pv = __bfloat162float(pr[c]);
    else pv = pr[c];
    if (pv != 0.f) dsum += pv * dr[c];
  }
  dsum = wsum(dsum);
  for (int64_t c = lane; c < s; c += 32) {
    float pv;
    if constexpr (sizeof(T) == 2) pv = __bfloat162float(pr[c]);
    else pv = pr[c];
    st_out(pr + c, pv != 0.f ? scale * pv * (dr[c] - dsum) : 0.f);
  }
}

// Padding columns of the score rows (block offset >= b of each bp-wide block) := -inf.
__global__ void rsa_fill_pad(float* __restrict__ S, int64_t rows, int64_t ls, int64_t b, int64_t bp) {
  const int64_t pad = bp - b, nblk = ls / bp;
  const int64_t n = rows * nblk * pad;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t o = i % pad, j = (i / pad) % nblk, r = i / (pad * nblk);
    S[r * ls + j * bp + b + o] = -INFINITY;
  }
}

template <typename T>
__global__ void rsa_cast(const float* __restrict__ src, int64_t n, T* __restrict__ dst) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) st_out(dst + i, src[i]);
}

struct RsaPlan {
  int p = 1, r = 0;
  int64_t s = 0, b = 0, d = 0, heads = 0, chunk = 1;
  // score rows are stored as p blocks of bp >= b columns (bp = b rounded up to 8) so that every
  // block starts 16-byte aligned and every row stride is a TMA-legal multiple of 8 elements
  // (ragged sequences, e.g. ViT's 197 tokens); the bp - b padding columns hold -inf scores and
  // zero probabilities. ls = p bp is the row stride of S and P.
  int64_t bp = 0, ls = 0;
  int64_t fchunk = 0;  // heads per online-softmax ring launch (0: two-pass only)
  size_t esz = 2;
};

tp_status rsa_plan(const tp_grid* g, const tp_rsa_desc* d, RsaPlan* P) {
  if (!g || !d) return fail(TP_ERR_ARG, "rsa: null grid or desc");
  if (g->mode != TP_1D) return fail(TP_ERR_CONSTRAINT, "rsa: the ring is a 1D grid (TP_1D)");
  if (d->dtype != TP_BF16 && d->dtype != TP_FP32) return fail(TP_ERR_ARG, "rsa: unknown dtype");
  if (d->seq < 0 || d->d_k < 0 || d->heads < 0) return fail(TP_ERR_SHAPE, "rsa: negative size");
  P->p = g->world;
  P->r = g->rank;
  if (d->seq % P->p)
    return fail(TP_ERR_INDIVISIBLE, "rsa: sequence " + std::to_string(d->seq) +
                                        " not divisible by the ring size " + std::to_string(P->p));
  P->s = d->seq;
  P->b = d->seq / P->p;
  P->d = d->d_k;
  P->heads = d->heads;
  P->esz = dtype_size(d->dtype);
  P->bp = (P->b + 7) / 8 * 8;
  P->ls = P->bp * P->p;
  const size_t per_head = size_t(P->b) * size_t(P->ls) * 4;
  P->chunk = per_head ? std::max<int64_t>(1, std::min<int64_t>(d->heads, kScoreBudget / per_head)) : 1;
  if (P->chunk < 1) P->chunk = 1;
  // the online-softmax ring keeps no score rows: all heads in one launch per ring step
  P->fchunk = flash_supported(P->d, d->dtype) ? std::max<int64_t>(1, std::min<int64_t>(d->heads, 65535)) : 0;
  return TP_OK;
}

tp_status fill_pad(const RsaPlan& P, float* S, int64_t rows, cudaStream_t s) {
  if (P.bp == P.b || !rows) return TP_OK;
  const int64_t n = rows * P.p * (P.bp - P.b);
  const unsigned G = static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, 148 * 8));
  rsa_fill_pad<<<G, 256, 0, s>>>(S, rows, P.ls, P.b, P.bp);
  count_launch();
  TP_CUDA(cudaGetLastError());
  return TP_OK;
}

struct RsaWs {
  float* S = nullptr;       // [chunk, b, s] fp32 scores
  void* Pm = nullptr;       // [chunk, b, s] probabilities (dtype)
  void* kv[2] = {};         // ring buffers [chunk, b, d] (dtype)
  float* acc = nullptr;     // [chunk, b, d] fp32 output accumulator
  float* facc = nullptr;    // online-softmax ring: [fchunk, b, d] fp32 unnormalised O
  void* fk[2] = {};         //   K ring buffers [fchunk, b, d] (dtype)
  void* vv[2] = {};         //   V ring buffers [fchunk, b, d] (dtype)
  float* ml = nullptr;      //   [fchunk, b, 2] fp32 running row max / sum
  void* gemm_ws = nullptr;  // split-K scratch
  size_t gemm_ws_bytes = 0;
  float *parts_k = nullptr, *parts_v = nullptr;  // backward: [p][chunk][b][d] fp32
  float *red_k = nullptr, *red_v = nullptr;      // backward: [chunk][b][d] fp32
};

void rsa_carve(Carver& c, const RsaPlan& P, RsaWs* w) {
  const size_t ch = size_t(P.chunk);
  w->S = static_cast<float*>(c.take(ch * P.b * P.ls * 4));
  w->Pm = c.take(ch * P.b * P.ls * P.esz);
  w->kv[0] = c.take(ch * P.b * P.d * P.esz);
  w->kv[1] = c.take(ch * P.b * P.d * P.esz);
  w->acc = static_cast<float*>(c.take(ch * P.b * P.d * 4));
  const size_t fc = size_t(P.fchunk);
  w->facc = static_cast<float*>(c.take(fc * P.b * P.d * 4));
  w->fk[0] = c.take(fc * P.b * P.d * P.esz);
  w->fk[1] = c.take(fc * P.b * P.d * P.esz);
  w->vv[0] = c.take(fc * P.b * P.d * P.esz);
  w->vv[1] = c.take(fc * P.b * P.d * P.esz);
  w->ml = static_cast<float*>(c.take(fc * P.b * 2 * 4));
  w->gemm_ws_bytes = gemm_tc2_ws_bytes();
  w->gemm_ws = c.take(w->gemm_ws_bytes);
  // backward: per-destination-block dK / dV contributions and their reduce-scattered sums
  w->parts_k = static_cast<float*>(c.take(size_t(P.p) * ch * P.b * P.d * 4));
  w->parts_v = static_cast<float*>(c.take(size_t(P.p) * ch * P.b * P.d * 4));
  w->red_k = static_cast<float*>(c.take(ch * P.b * P.d * 4));
  w->red_v = static_cast<float*>(c.take(ch * P.b * P.d * 4));
}

GemmArgs rsa_gemm(int64_t M, int64_t N, int64_t K, const void* A, int64_t lda, const void* B,
                  int64_t ldb, bool tb, void* D, int64_t ldd, tp_dtype in, tp_dtype out, float alpha,
                  const float* C, const RsaWs& w, bool ta = false) {
  GemmArgs a;
  a.M = M;
  a.N = N;
  a.K = K;
  a.A = A;
  a.trans_a = ta;
  a.lda = lda;
  a.B = B;
  a.ldb = ldb;
  a.trans_b = tb;
  a.C = C;
  a.ldc = N;
  a.D = D;
  a.ldd = ldd;
  a.in_dtype = in;
  a.out_dtype = out;
  a.alpha = alpha;
  a.ws = w.gemm_ws;
  a.ws_bytes = w.gemm_ws_bytes;
  return a;
}

// Run `gs` (independent per-head GEMMs) four at a time as grouped launches.
tp_status run_heads(std::vector<GemmArgs>& gs, cudaStream_t s) {
  for (size_t i = 0; i < gs.size(); i += 4) {
    const int n = static_cast<int>(std::min<size_t>(4, gs.size() - i));
    if (n == 1) TP_TRY(gemm(gs[i], s));
    else TP_TRY(gemm_group(&gs[i], n, s));
  }
  return TP_OK;
}

}  // namespace

tp_status rsa_ws_bytes(const tp_grid* g, const tp_rsa_desc* d, size_t* bytes) {
  RsaPlan P;
  TP_TRY(rsa_plan(g, d, &P));
  Carver c;
  RsaWs w;
  rsa_carve(c, P, &w);
  *bytes = c.off + 256;
  return TP_OK;
}

tp_status rsa_fwd(tp_grid* g, const tp_rsa_desc* d, const void* q, const void* k, const void* v,
                  void* out, void* ws, size_t ws_bytes, cudaStream_t s, float* lse) {
  RsaPlan P;
  TP_TRY(rsa_plan(g, d, &P));
  size_t need = 0;
  TP_TRY(rsa_ws_bytes(g, d, &need));
  if (ws_bytes < need || !ws) return fail(TP_ERR_WORKSPACE, "rsa: workspace too small");
  if (!P.heads || !P.b || !P.d) return TP_OK;
  if (!q || !k || !v || !out) return fail(TP_ERR_ARG, "rsa: null q, k, v or out");
  Carver c;
  c.base = static_cast<char*>(ws);
  RsaWs w;
  rsa_carve(c, P, &w);
  Comm* ring = g->axis[0].get();  // nullptr when p == 1
  const tp_dtype dt = d->dtype;
  const float scale = d->scale != 0.f ? d->scale : 1.f / std::sqrt(static_cast<float>(P.d));
  const int64_t bd = P.b * P.d;
  std::vector<GemmArgs> gs;
  const int env_fused = knob("TP_RSA_FUSED");
  const bool fused = env_fused && P.fchunk > 0;
  const int64_t step_heads = fused ? P.fchunk : P.chunk;
  for (int64_t h0 = 0; h0 < P.heads; h0 += step_heads) {
    const int64_t nh = std::min<int64_t>(step_heads, P.heads - h0);
    const char* qc = static_cast<const char*>(q) + h0 * bd * P.esz;
    if (fused) {
      // ---- online-softmax ring: K and V blocks travel the ring together;
      // at every step one fused attention launch (flash.cu: scores in TMEM, never in HBM)
      // continues each row's softmax from the carried (O, max, sum) of the blocks seen so far
      const void* ck = static_cast<const char*>(k) + h0 * bd * P.esz;
      const void* cv = static_cast<const char*>(v) + h0 * bd * P.esz;
      char* oc = static_cast<char*>(out) + h0 * bd * P.esz;
      // block t+1 travels on the grid's comm stream while block t is attended on `s`
      // (double-buffered: the shift into buffer t % 2 waits for the launch that last read it)
      cudaStream_t cs = g->comm_stream ? g->comm_stream : s;
      cudaEvent_t ev_flash = nullptr, ev_shift = nullptr;
      if (P.p > 1 && cs != s) {
        cudaEvent_t e = g->ev();
        TP_CUDA(cudaEventRecord(e, s));  // inputs (and earlier users of the buffers) are done
        TP_CUDA(cudaStreamWaitEvent(cs, e, 0));
      }
      for (int t = 0; t < P.p; ++t) {
        const bool last = t + 1 == P.p;
        if (!last) {
          if (ev_flash && cs != s) TP_CUDA(cudaStreamWaitEvent(cs, ev_flash, 0));
          TP_TRY(ring->shift(ck, w.fk[t & 1], size_t(nh) * bd, dt, -1, cs));
          TP_TRY(ring->shift(cv, w.vv[t & 1], size_t(nh) * bd, dt, -1, cs));
        }
        TP_TRY(flash_attn_fwd_carry(nh, P.b, P.d, qc, ck, cv, oc, w.facc, w.ml, t > 0, last, scale, s,
                                    lse ? lse + h0 * P.b : nullptr));
        if (!last) {
          if (cs != s) {
            ev_flash = g->ev();
            TP_CUDA(cudaEventRecord(ev_flash, s));
            ev_shift = g->ev();
            TP_CUDA(cudaEventRecord(ev_shift, cs));
            TP_CUDA(cudaStreamWaitEvent(s, ev_shift, 0));  // block t+1 has arrived
          }
          ck = w.fk[t & 1];
          cv = w.vv[t & 1];
        }
      }
      continue;
    }
    // ---- pass 1: K ring -> scores
    TP_TRY(fill_pad(P, w.S, nh * P.b, s));
    const void* cur = static_cast<const char*>(k) + h0 * bd * P.esz;
    int nb = 0;
    for (int t = 0; t < P.p; ++t) {
      const int j = ((P.r - t) % P.p + P.p) % P.p;
      gs.clear();
      for (int64_t h = 0; h < nh; ++h)
        gs.push_back(rsa_gemm(P.b, P.b, P.d, qc + h * bd * P.esz, P.d,
                              static_cast<const char*>(cur) + h * bd * P.esz, P.d, true,
                              w.S + h * P.b * P.ls + j * P.bp, P.ls, dt, TP_FP32, scale, nullptr, w));
      TP_TRY(run_heads(gs, s));
      if (t + 1 < P.p) {
        TP_TRY(ring->shift(cur, w.kv[nb], size_t(nh) * bd, dt, -1, s));
        cur = w.kv[nb];
        nb ^= 1;
      }
    }
    // ---- softmax of the assembled rows
    TP_TRY(launch_softmax(w.S, nh * P.b, P.ls, dt, w.Pm, s));
    // ---- pass 2: V ring -> output
    cur = static_cast<const char*>(v) + h0 * bd * P.esz;
    nb = 0;
    char* oc = static_cast<char*>(out) + h0 * bd * P.esz;
    for (int t = 0; t < P.p; ++t) {
      const int j = ((P.r - t) % P.p + P.p) % P.p;
      const bool last = t + 1 == P.p;
      gs.clear();
      for (int64_t h = 0; h < nh; ++h) {
        const void* A = static_cast<const char*>(w.Pm) + (h * P.b * P.ls + j * P.bp) * P.esz;
        const void* B = static_cast<const char*>(cur) + h * bd * P.esz;
        void* D = last ? static_cast<void*>(oc + h * bd * P.esz) : static_cast<void*>(w.acc + h * bd);
        gs.push_back(rsa_gemm(P.b, P.d, P.b, A, P.ls, B, P.d, false, D, P.d, dt, last ? dt : TP_FP32,
                              1.f, t > 0 ? w.acc + h * bd : nullptr, w));
      }
      TP_TRY(run_heads(gs, s));
      if (!last) {
        TP_TRY(ring->shift(cur, w.kv[nb], size_t(nh) * bd, dt, -1, s));
        cur = w.kv[nb];
        nb ^= 1;
      }
    }
  }
  return TP_OK;
}


// Backward (reading N4; oracle/ring_attention.py ring_attention_bwd): per head chunk,
//   K ring -> scores (recomputed) -> softmax P;  dV parts P_r[:, j]^T dO_r for every block j;
//   V ring -> dP = dO V_j^T;  dS = scale P (dP - rowsum(P dP)) (over P);
//   K ring -> dQ = sum_j dS[:, j] K_j;  dK parts dS[:, j]^T Q_r;
//   reduce-scatter of the dK / dV parts over the ring -> this rank's blocks.
// Fused ring backward (reading N4 with the online-softmax forward's lse): K and V travel the
// ring together (double-buffered on the comm stream, block t+1 moving under launch t); each step
// one flash_bwd_step adds this rank's queries' dQ (fp32 accumulator) and writes the visiting
// block's dK / dV contribution (fp32) into its slot of the reduce-scatter buffers; at the end
// the contributions are reduce-scattered to the blocks' owners and everything cast to dtype.
tp_status rsa_bwd_fused(tp_grid* g, const RsaPlan& P, const RsaWs& w, const void* q, const void* k,
                        const void* v, const void* out, const float* lse, const void* dout, void* dq,
                        void* dk, void* dv, float scale, cudaStream_t s) {
  Comm* ring = g->axis[0].get();
  const tp_dtype dt = TP_BF16;
  const int64_t bd = P.b * P.d;
  cudaStream_t cs = g->comm_stream ? g->comm_stream : s;
  for (int64_t h0 = 0; h0 < P.heads; h0 += P.chunk) {
    const int64_t nh = std::min<int64_t>(P.chunk, P.heads - h0);
    const int64_t n = nh * bd;
    const char* qc = static_cast<const char*>(q) + h0 * bd * P.esz;
    const char* oc = static_cast<const char*>(out) + h0 * bd * P.esz;
    const char* doc = static_cast<const char*>(dout) + h0 * bd * P.esz;
    const float* lc = lse + h0 * P.b;
    float* delta = w.ml;        // [nh b] (the forward's carry buffer, free here)
    float* dq_acc = w.acc;      // [nh b d] fp32
    TP_TRY(flash_bwd_delta_launch(nh * P.b, P.d, oc, doc, delta, s));
    TP_CUDA(cudaMemsetAsync(dq_acc, 0, size_t(n) * 4, s));
    const void* ck = static_cast<const char*>(k) + h0 * bd * P.esz;
    const void* cv = static_cast<const char*>(v) + h0 * bd * P.esz;
    cudaEvent_t ev_used = nullptr;
    if (P.p > 1 && cs != s) {
      cudaEvent_t e = g->ev();
      TP_CUDA(cudaEventRecord(e, s));
      TP_CUDA(cudaStreamWaitEvent(cs, e, 0));
    }
    for (int t = 0; t < P.p; ++t) {
      const bool last = t + 1 == P.p;
      const int j = ((P.r - t) % P.p + P.p) % P.p;  // the visiting block's owner
      if (!last) {  // block t+1 moves while block t is processed
        if (ev_used && cs != s) TP_CUDA(cudaStreamWaitEvent(cs, ev_used, 0));
        TP_TRY(ring->shift(ck, w.fk[t & 1], size_t(n), dt, -1, cs));
        TP_TRY(ring->shift(cv, w.vv[t & 1], size_t(n), dt, -1, cs));
      }
      TP_TRY(flash_bwd_step(nh, P.b, P.d, qc, ck, cv, doc, lc, delta, dq_acc,
                            w.parts_k + int64_t(j) * n, w.parts_v + int64_t(j) * n, scale, s));
      if (!last) {
        if (cs != s) {
          ev_used = g->ev();
          TP_CUDA(cudaEventRecord(ev_used, s));
          cudaEvent_t arrived = g->ev();
          TP_CUDA(cudaEventRecord(arrived, cs));
          TP_CUDA(cudaStreamWaitEvent(s, arrived, 0));
        }
        ck = w.fk[t & 1];
        cv = w.vv[t & 1];
      }
    }
    const float* rk = w.parts_k;
    const float* rv = w.parts_v;
    if (ring) {
      TP_TRY(ring->reducescatter(w.parts_k, w.red_k, n, TP_FP32, s));
      TP_TRY(ring->reducescatter(w.parts_v, w.red_v, n, TP_FP32, s));
      rk = w.red_k;
      rv = w.red_v;
    }
    TP_TRY(flash_bwd_cast_launch(dq_acc, n, static_cast<char*>(dq) + h0 * bd * P.esz, s));
    TP_TRY(flash_bwd_cast_launch(rk, n, static_cast<char*>(dk) + h0 * bd * P.esz, s));
    TP_TRY(flash_bwd_cast_launch(rv, n, static_cast<char*>(dv) + h0 * bd * P.esz, s));
  }
  return TP_OK;
}

tp_status rsa_bwd(tp_grid* g, const tp_rsa_desc* d, const void* q, const void* k, const void* v,
                  const void* dout, void* dq, void* dk, void* dv, void* ws, size_t ws_bytes,
                  cudaStream_t s, const void* out, const float* lse) {
  RsaPlan P;
  TP_TRY(rsa_plan(g, d, &P));
  size_t need = 0;
  TP_TRY(rsa_ws_bytes(g, d, &need));
  if (ws_bytes < need || !ws) return fail(TP_ERR_WORKSPACE, "rsa: workspace too small");
  if (!P.heads || !P.b || !P.d) return TP_OK;
  if (!q || !k || !v || !dout || !dq || !dk || !dv) return fail(TP_ERR_ARG, "rsa_bwd: null pointer");
  Carver c;
  c.base = static_cast<char*>(ws);
  RsaWs w;
  rsa_carve(c, P, &w);
  Comm* ring = g->axis[0].get();
  const tp_dtype dt = d->dtype;
  const float scale = d->scale != 0.f ? d->scale : 1.f / std::sqrt(static_cast<float>(P.d));
  const int64_t bd = P.b * P.d;
  if (out && lse && P.fchunk > 0 && knob("TP_RSA_FUSED"))
    return rsa_bwd_fused(g, P, w, q, k, v, out, lse, dout, dq, dk, dv, scale, s);
  std::vector<GemmArgs> gs;
  for (int64_t h0 = 0; h0 < P.heads; h0 += P.chunk) {
    const int64_t nh = std::min<int64_t>(P.chunk, P.heads - h0);
    const char* qc = static_cast<const char*>(q) + h0 * bd * P.esz;
    const char* doc = static_cast<const char*>(dout) + h0 * bd * P.esz;
    // ---- K ring: recompute the score rows, softmax
    TP_TRY(fill_pad(P, w.S, nh * P.b, s));
    const void* cur = static_cast<const char*>(k) + h0 * bd * P.esz;
    int nb = 0;
    for (int t = 0; t < P.p; ++t) {
      const int j = ((P.r - t) % P.p + P.p) % P.p;
      gs.clear();
      for (int64_t h = 0; h < nh; ++h)
        gs.push_back(rsa_gemm(P.b, P.b, P.d, qc + h * bd * P.esz, P.d,
                              static_cast<const char*>(cur) + h * bd * P.esz, P.d, true,
                              w.S + h * P.b * P.ls + j * P.bp, P.ls, dt, TP_FP32, scale, nullptr, w));
      TP_TRY(run_heads(gs, s));
      if (t + 1 < P.p) {
        TP_TRY(ring->shift(cur, w.kv[nb], size_t(nh) * bd, dt, -1, s));
        cur = w.kv[nb];
        nb ^= 1;
      }
    }
    TP_TRY(launch_softmax(w.S, nh * P.b, P.ls, dt, w.Pm, s));
    // ---- dV parts: block j <- P[:, j]^T dO (fp32, laid out [j][h][b][d] for the reduce-scatter)
    gs.clear();
    for (int j = 0; j < P.p; ++j)
      for (int64_t h = 0; h < nh; ++h)
        gs.push_back(rsa_gemm(P.b, P.d, P.b,
                              static_cast<const char*>(w.Pm) + (h * P.b * P.ls + j * P.bp) * P.esz, P.ls,
                              doc + h * bd * P.esz, P.d, false,
                              w.parts_v + (int64_t(j) * nh + h) * bd, P.d, dt, TP_FP32, 1.f, nullptr, w,
                              true));
    TP_TRY(run_heads(gs, s));
    // ---- V ring: dP = dO V_j^T (over the score buffer)
    cur = static_cast<const char*>(v) + h0 * bd * P.esz;
    nb = 0;
    for (int t = 0; t < P.p; ++t) {
      const int j = ((P.r - t) % P.p + P.p) % P.p;
      gs.clear();
      for (int64_t h = 0; h < nh; ++h)
        gs.push_back(rsa_gemm(P.b, P.b, P.d, doc + h * bd * P.esz, P.d,
                              static_cast<const char*>(cur) + h * bd * P.esz, P.d, true,
                              w.S + h * P.b * P.ls + j * P.bp, P.ls, dt, TP_FP32, 1.f, nullptr, w));
      TP_TRY(run_heads(gs, s));
      if (t + 1 < P.p) {
        TP_TRY(ring->shift(cur, w.kv[nb], size_t(nh) * bd, dt, -1, s));
        cur = w.kv[nb];
        nb ^= 1;
      }
    }
    // ---- dS = scale P (dP - rowsum(P dP)), in place over P
    {
      const int64_t rows = nh * P.b;
      const unsigned G = static_cast<unsigned>((rows * 32 + 255) / 256);
      if (dt == TP_BF16)
        rsa_dscore<__nv_bfloat16><<<G, 256, 0, s>>>(static_cast<__nv_bfloat16*>(w.Pm), w.S, rows, P.ls, scale);
      else
        rsa_dscore<float><<<G, 256, 0, s>>>(static_cast<float*>(w.Pm), w.S, rows, P.ls, scale);
      count_launch();
      TP_CUDA(cudaGetLastError());
    }
    // ---- dK parts: block j <- dS[:, j]^T Q
    gs.clear();
    for (int j = 0; j < P.p; ++j)
      for (int64_t h = 0; h < nh; ++h)
        gs.push_back(rsa_gemm(P.b, P.d, P.b,
                              static_cast<const char*>(w.Pm) + (h * P.b * P.ls + j * P.bp) * P.esz, P.ls,
                              qc + h * bd * P.esz, P.d, false,
                              w.parts_k + (int64_t(j) * nh + h) * bd, P.d, dt, TP_FP32, 1.f, nullptr, w,
                              true));
    TP_TRY(run_heads(gs, s));
    // ---- K ring: dQ = sum_j dS[:, j] K_j (fp32 accumulator through C)
    cur = static_cast<const char*>(k) + h0 * bd * P.esz;
    nb = 0;
    char* dqc = static_cast<char*>(dq) + h0 * bd * P.esz;
    for (int t = 0; t < P.p; ++t) {
      const int j = ((P.r - t) % P.p + P.p) % P.p;
      const bool last = t + 1 == P.p;
      gs.clear();
      for (int64_t h = 0; h < nh; ++h) {
        void* D = last ? static_cast<void*>(dqc + h * bd * P.esz) : static_cast<void*>(w.acc + h * bd);
        gs.push_back(rsa_gemm(P.b, P.d, P.b,
                              static_cast<const char*>(w.Pm) + (h * P.b * P.ls + j * P.bp) * P.esz, P.ls,
                              static_cast<const char*>(cur) + h * bd * P.esz, P.d, false, D, P.d, dt,
                              last ? dt : TP_FP32, 1.f, t > 0 ? w.acc + h * bd : nullptr, w));
      }
      TP_TRY(run_heads(gs, s));
      if (!last) {
        TP_TRY(ring->shift(cur, w.kv[nb], size_t(nh) * bd, dt, -1, s));
        cur = w.kv[nb];
        nb ^= 1;
      }
    }
    // ---- dK, dV: sum every rank's contribution at the block's owner
    const int64_t n = nh * bd;
    const float* rk = w.parts_k;
    const float* rv = w.parts_v;
    if (ring) {
      TP_TRY(ring->reducescatter(w.parts_k, w.red_k, n, TP_FP32, s));
      TP_TRY(ring->reducescatter(w.parts_v, w.red_v, n, TP_FP32, s));
      rk = w.red_k;
      rv = w.red_v;
    }
    const unsigned G = static_cast<unsigned>((n + 255) / 256);
    char* dkc = static_cast<char*>(dk) + h0 * bd * P.esz;
    char* dvc = static_cast<char*>(dv) + h0 * bd * P.esz;
    if (dt == TP_BF16) {
      rsa_cast<__nv_bfloat16><<<G, 256, 0, s>>>(rk, n, reinterpret_cast<__nv_bfloat16*>(dkc));
      rsa_cast<__nv_bfloat16><<<G, 256, 0, s>>>(rv, n, reinterpret_cast<__nv_bfloat16*>(dvc));
    } else {
      rsa_cast<float><<<G, 256, 0, s>>>(rk, n, reinterpret_cast<float*>(dkc));
      rsa_cast<float><<<G, 256, 0, s>>>(rv, n, reinterpret_cast<float*>(dvc));
    }
    count_launch(2);
    TP_CUDA(cudaGetLastError());
  }
  return TP_OK;
}

}  // namespace tp
