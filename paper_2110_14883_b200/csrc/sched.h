// Per-mode forward/backward schedules (SURVEY 8(a) rows a-3 .. a-10, a-13).
#pragma once

#include "tp_internal.h"

namespace tp {

struct Ext {
  int64_t r0 = 0, rows = 0, c0 = 0, cols = 0;
};

// Divisibility (hard error, no padding) and the per-rank extents of SURVEY 8(a).
tp_status check_divisible(const tp_grid* g, const tp_linear_desc* d);
tp_status extent(const tp_grid* g, const tp_linear_desc* d, int tensor, Ext* e);

// Bump allocator over the caller's workspace; with base == nullptr it only measures.
struct Carver {
  char* base = nullptr;
  size_t off = 0;
  void* take(size_t bytes) {
    off = (off + 255) & ~size_t(255);
    void* p = base ? base + off : nullptr;
    off += bytes;
    return p;
  }
};

struct Run {
  tp_grid* g = nullptr;
  const tp_linear_desc* d = nullptr;
  cudaStream_t s = nullptr;   // caller's stream: compute
  cudaStream_t cs = nullptr;  // communication stream (== s when serial)
  bool plan = false;          // carve only: nothing is enqueued
  Carver ws, saved;
};

// LayerNorm over the columns of a TP activation shard (norm.cu; tensor = TP_TENSOR_X / _Y).
tp_status layernorm_ws_bytes(const tp_grid* g, const tp_linear_desc* d, int tensor, size_t* bytes);
tp_status layernorm_fwd(tp_grid* g, const tp_linear_desc* d, int tensor, float eps, const void* x,
                        const void* gamma, const void* beta, void* y, float* stats, void* ws,
                        size_t ws_bytes, cudaStream_t s);
tp_status layernorm_bwd(tp_grid* g, const tp_linear_desc* d, int tensor, const void* dy,
                        const void* x, const void* gamma, const float* stats, void* dx,
                        void* dgamma, void* dbeta, void* ws, size_t ws_bytes, cudaStream_t s);

// Ring Self-Attention forward (rsa.cu).
tp_status rsa_ws_bytes(const tp_grid* g, const tp_rsa_desc* d, size_t* bytes);
tp_status rsa_fwd(tp_grid* g, const tp_rsa_desc* d, const void* q, const void* k, const void* v,
                  void* out, void* ws, size_t ws_bytes, cudaStream_t s, float* lse = nullptr);
tp_status rsa_bwd(tp_grid* g, const tp_rsa_desc* d, const void* q, const void* k, const void* v,
                  const void* dout, void* dq, void* dk, void* dv, void* ws, size_t ws_bytes,
                  cudaStream_t s, const void* out = nullptr, const float* lse = nullptr);

// Fused attention forward (flash.cu): [problems, s, d] bf16, d in {64, 128}.
bool flash_supported(int64_t d, tp_dtype dt);
// lse (optional, [problems*s] fp32): per-row log-sum-exp in scaled log2 units (for flash_attn_bwd)
tp_status flash_attn_fwd(int64_t problems, int64_t s, int64_t d, const void* q, const void* k,
                         const void* v, void* out, float scale, cudaStream_t st,
                         float* lse = nullptr);
// Fused attention backward (flash_bwd.cu): q, k, v, o, dout [problems, s, d] bf16, lse
// [problems*s] fp32 from flash_attn_fwd; writes dq, dk, dv [problems, s, d] bf16. ws: fp32
// scratch of flash_bwd_ws_bytes (dQ accumulator, row deltas).
size_t flash_bwd_ws_bytes(int64_t problems, int64_t s, int64_t d);
// building blocks of the ring (sequence-parallel) backward: row deltas, one ring step, cast
tp_status flash_bwd_delta_launch(int64_t rows, int64_t d, const void* o, const void* dout,
                                 float* delta, cudaStream_t st);
tp_status flash_bwd_step(int64_t problems, int64_t s, int64_t d, const void* q, const void* k,
                         const void* v, const void* dout, const float* lse, const float* delta,
                         float* dq_acc, float* dk32, float* dv32, float scale, cudaStream_t st);
tp_status flash_bwd_cast_launch(const float* src, int64_t n, void* dst, cudaStream_t st);
tp_status flash_attn_bwd(int64_t problems, int64_t s, int64_t d, const void* q, const void* k,
                         const void* v, const void* o, const void* dout, const float* lse,
                         void* dq, void* dk, void* dv, float scale, void* ws, cudaStream_t st);
// lse (optional): written at the last ring block (F.last), as flash_attn_fwd's
tp_status flash_attn_fwd_carry(int64_t problems, int64_t s, int64_t d, const void* q, const void* k,
                               const void* v, void* out, float* acc, float* ml, bool carry_in,
                               bool last, float scale, cudaStream_t st, float* lse = nullptr);

// Multi-head attention core in the TP layouts (attn.cu).
tp_status attention_ws_bytes(const tp_grid* g, const tp_linear_desc* qd, int64_t seq, int64_t heads,
                             size_t* bytes);
tp_status attention_fwd(tp_grid* g, const tp_linear_desc* qd, int64_t seq, int64_t heads, float scale,
                        const void* qkv, void* out, float* lse, void* ws, size_t ws_bytes,
                        cudaStream_t s);
tp_status attention_bwd(tp_grid* g, const tp_linear_desc* qd, int64_t seq, int64_t heads, float scale,
                        const void* qkv, const void* out, const float* lse, const void* dout,
                        void* dqkv, void* ws, size_t ws_bytes, cudaStream_t s);

tp_status sched_fwd(Run& R, const void* x, const void* w, const void* bias, void* y);
tp_status sched_bwd(Run& R, const void* dy, const void* x, const void* w, void* dx, void* dw,
                    void* dbias);

}  // namespace tp
