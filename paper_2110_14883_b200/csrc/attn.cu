// Multi-head self-attention core in the tensor-parallel layouts (SURVEY 8(f) NEXT-2:
// "attention core with heads split across columns", formula P:L604).
//
// The QKV linear (h -> 3h) writes head g to columns [3 d g, 3 d (g+1)) as [q | k | v]
// (reading N5), so this rank's block of the QKV output (tp_shard_extent(desc, Y)) holds whole
// heads; when its row extent is a multiple of `seq` it also holds whole sequences, and the
// attention of every (sequence, head) it holds is local -- no communication in 1D, 2D, 2.5D or
// 3D. The output [rows, heads_local d] is the X block of the output projection (1D row split,
// the same 2D / 2.5D block, 3D parity + 1).
//
// Kernels: a gather of the interleaved q / k / v columns into [sequences x heads, seq, d]
// problems (16-byte vectors), the Ring Self-Attention path at p = 1 (rsa.cu: score GEMMs on the
// tensor cores, row softmax, PV GEMMs; backward by recomputation), and the scatter back.
#include <cuda_bf16.h>

#include <cmath>
#include <cstdlib>

#include "sched.h"
#include "tp_internal.h"

namespace tp {
namespace {

struct AttnPlan {
  Ext e;
  int64_t seq = 0, heads_local = 0, d = 0, batch_local = 0, problems = 0;
  size_t esz = 2;
  tp_rsa_desc rd{};
};

tp_status attn_plan(const tp_grid* g, const tp_linear_desc* qd, int64_t seq, int64_t heads,
                    float scale, AttnPlan* P) {
  if (!g || !qd) return fail(TP_ERR_ARG, "attention: null grid or desc");
  if (qd->dtype != TP_BF16 && qd->dtype != TP_FP32) return fail(TP_ERR_ARG, "attention: dtype");
  if (seq <= 0 || heads <= 0) return fail(TP_ERR_ARG, "attention: seq and heads must be > 0");
  if (qd->N % (3 * heads)) return fail(TP_ERR_SHAPE, "attention: N is not 3 x heads x d_head");
  TP_TRY(check_divisible(g, qd));
  TP_TRY(extent(g, qd, TP_TENSOR_Y, &P->e));
  P->d = qd->N / (3 * heads);
  if (P->e.cols % (3 * P->d) || P->e.c0 % (3 * P->d))
    return fail(TP_ERR_SHAPE, "attention: this rank's QKV column block splits a head");
  if (P->e.rows % seq || P->e.r0 % seq)
    return fail(TP_ERR_SHAPE, "attention: this rank's row block splits a sequence");
  if (P->d % 8) return fail(TP_ERR_SHAPE, "attention: d_head must be a multiple of 8");
  P->seq = seq;
  P->heads_local = P->e.cols / (3 * P->d);
  P->batch_local = P->e.rows / seq;
  P->problems = P->batch_local * P->heads_local;
  P->esz = dtype_size(qd->dtype);
  P->rd = tp_rsa_desc{seq, P->d, P->problems, qd->dtype, scale};
  return TP_OK;
}

// The p = 1 "ring" for the local attention problems.
tp_grid* local_grid() {
  static thread_local tp_grid g;
  g.mode = TP_1D;
  g.world = 1;
  g.rank = 0;
  g.q = 1;
  g.d = 1;
  g.ndims = 1;
  return &g;
}

// qkv [rows, 3 H d] (head g: [q | k | v] blocks of d) <-> problems [(b H + g), seq, d].
// dir 0: gather component `c` into dst; dir 1: scatter src into component `c` of qkv.
template <typename T>
__global__ void attn_pack(const T* __restrict__ src, T* __restrict__ dst, int64_t rows, int64_t seq,
                          int64_t H, int64_t d, int64_t ld, int64_t col_off, int64_t stride_g, int dir) {
  constexpr int V = 16 / sizeof(T);
  const int64_t dv = d / V;
  const int64_t n = rows * H * dv;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t e = i % dv, g = (i / dv) % H, t = i / (dv * H);
    const int64_t b = t / seq, pos = t % seq;
    const int64_t packed = ((b * H + g) * seq + pos) * d + e * V;
    const int64_t strided = t * ld + g * stride_g + col_off + e * V;
    if (dir == 0)
      *reinterpret_cast<uint4*>(dst + packed) = *reinterpret_cast<const uint4*>(src + strided);
    else
      *reinterpret_cast<uint4*>(dst + strided) = *reinterpret_cast<const uint4*>(src + packed);
  }
}

tp_status pack(const AttnPlan& P, const void* src, void* dst, int64_t ld, int64_t col_off,
               int64_t stride_g, int dir, cudaStream_t s) {
  const int64_t n = P.e.rows * P.heads_local * (P.d / (16 / int64_t(P.esz)));
  if (!n) return TP_OK;
  const unsigned G = static_cast<unsigned>(std::min<int64_t>((n + 255) / 256, 148 * 16));
  if (P.esz == 2)
    attn_pack<__nv_bfloat16><<<G, 256, 0, s>>>(static_cast<const __nv_bfloat16*>(src),
                                               static_cast<__nv_bfloat16*>(dst), P.e.rows, P.seq,
                                               P.heads_local, P.d, ld, col_off, stride_g, dir);
  else
    attn_pack<float><<<G, 256, 0, s>>>(static_cast<const float*>(src), static_cast<float*>(dst),
                                       P.e.rows, P.seq, P.heads_local, P.d, ld, col_off, stride_g, dir);
  count_launch();
  TP_CUDA(cudaGetLastError());
  return TP_OK;
}

struct AttnWs {
  void* buf[8] = {};  // q, k, v, o / do, dq, dk, dv, o (fused backward): [problems, seq, d]
  void* rsa = nullptr;
  size_t rsa_bytes = 0;
  void* fb = nullptr;  // fused backward: fp32 dQ accumulator + row deltas
};

tp_status attn_carve(const AttnPlan& P, Carver& c, AttnWs* w) {
  const size_t one = size_t(P.problems) * P.seq * P.d * P.esz;
  for (auto& b : w->buf) b = c.take(one);
  TP_TRY(rsa_ws_bytes(local_grid(), &P.rd, &w->rsa_bytes));
  w->rsa = c.take(w->rsa_bytes);
  if (flash_supported(P.d, P.rd.dtype)) w->fb = c.take(flash_bwd_ws_bytes(P.problems, P.seq, P.d));
  return TP_OK;
}

}  // namespace

tp_status attention_ws_bytes(const tp_grid* g, const tp_linear_desc* qd, int64_t seq, int64_t heads,
                             size_t* bytes) {
  AttnPlan P;
  TP_TRY(attn_plan(g, qd, seq, heads, 0.f, &P));
  Carver c;
  AttnWs w;
  TP_TRY(attn_carve(P, c, &w));
  *bytes = c.off + 256;
  return TP_OK;
}

tp_status attention_fwd(tp_grid* g, const tp_linear_desc* qd, int64_t seq, int64_t heads, float scale,
                        const void* qkv, void* out, float* lse, void* ws, size_t ws_bytes,
                        cudaStream_t s) {
  AttnPlan P;
  TP_TRY(attn_plan(g, qd, seq, heads, scale, &P));
  size_t need = 0;
  TP_TRY(attention_ws_bytes(g, qd, seq, heads, &need));
  if (ws_bytes < need || !ws) return fail(TP_ERR_WORKSPACE, "attention: workspace too small");
  if (!P.problems) return TP_OK;
  if (!qkv || !out) return fail(TP_ERR_ARG, "attention: null qkv or out");
  if ((reinterpret_cast<uintptr_t>(qkv) | reinterpret_cast<uintptr_t>(out)) % 16)
    return fail(TP_ERR_SHAPE, "attention: 16-byte aligned buffers required");
  Carver c;
  c.base = static_cast<char*>(ws);
  AttnWs w;
  TP_TRY(attn_carve(P, c, &w));
  const int64_t ld = P.e.cols, d = P.d;
  for (int comp = 0; comp < 3; ++comp) TP_TRY(pack(P, qkv, w.buf[comp], ld, comp * d, 3 * d, 0, s));
  const int use_flash = knob("TP_FLASH");
  if (use_flash && flash_supported(d, qd->dtype) && P.problems <= 65535) {
    // fused forward: the scores stay on chip (flash.cu)
    const float sc = scale != 0.f ? scale : 1.f / std::sqrt(static_cast<float>(d));
    TP_TRY(flash_attn_fwd(P.problems, P.seq, d, w.buf[0], w.buf[1], w.buf[2], w.buf[3], sc, s, lse));
  } else {
    TP_TRY(rsa_fwd(local_grid(), &P.rd, w.buf[0], w.buf[1], w.buf[2], w.buf[3], w.rsa, w.rsa_bytes, s));
  }
  return pack(P, w.buf[3], out, P.heads_local * d, 0, d, 1, s);
}

tp_status attention_bwd(tp_grid* g, const tp_linear_desc* qd, int64_t seq, int64_t heads, float scale,
                        const void* qkv, const void* out, const float* lse, const void* dout,
                        void* dqkv, void* ws, size_t ws_bytes, cudaStream_t s) {
  AttnPlan P;
  TP_TRY(attn_plan(g, qd, seq, heads, scale, &P));
  size_t need = 0;
  TP_TRY(attention_ws_bytes(g, qd, seq, heads, &need));
  if (ws_bytes < need || !ws) return fail(TP_ERR_WORKSPACE, "attention: workspace too small");
  if (!P.problems) return TP_OK;
  if (!qkv || !dout || !dqkv) return fail(TP_ERR_ARG, "attention: null qkv, dout or dqkv");
  Carver c;
  c.base = static_cast<char*>(ws);
  AttnWs w;
  TP_TRY(attn_carve(P, c, &w));
  const int64_t ld = P.e.cols, d = P.d;
  for (int comp = 0; comp < 3; ++comp) TP_TRY(pack(P, qkv, w.buf[comp], ld, comp * d, 3 * d, 0, s));
  TP_TRY(pack(P, dout, w.buf[3], P.heads_local * d, 0, d, 0, s));
  const int use_flash = knob("TP_FLASH");
  if (use_flash && out && lse && w.fb && P.problems <= 65535) {
    // fused backward: P recomputed on chip from the forward's lse (scores never in HBM)
    TP_TRY(pack(P, out, w.buf[7], P.heads_local * d, 0, d, 0, s));
    const float sc = scale != 0.f ? scale : 1.f / std::sqrt(static_cast<float>(d));
    TP_TRY(flash_attn_bwd(P.problems, P.seq, d, w.buf[0], w.buf[1], w.buf[2], w.buf[7], w.buf[3], lse,
                          w.buf[4], w.buf[5], w.buf[6], sc, w.fb, s));
  } else {
    TP_TRY(rsa_bwd(local_grid(), &P.rd, w.buf[0], w.buf[1], w.buf[2], w.buf[3], w.buf[4], w.buf[5],
                   w.buf[6], w.rsa, w.rsa_bytes, s));
  }
  for (int comp = 0; comp < 3; ++comp) TP_TRY(pack(P, w.buf[4 + comp], dqkv, ld, comp * d, 3 * d, 1, s));
  return TP_OK;
}

}  // namespace tp
