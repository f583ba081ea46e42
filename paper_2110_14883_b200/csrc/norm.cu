// LayerNorm over the hidden (column) dimension of a tensor-parallel activation shard
// ("LayerNorm (row statistics across the column axis)").
//
// A rank holds a dense block [rows, cols] of X in the layout of tensor X or Y of a layer desc
// (SURVEY 8(a) extent table). Row statistics need all H columns of a row, which are spread
// over the ranks of ONE grid axis (the axis along which the column block changes while the
// rows stay); gamma / beta are column blocks, and their gradients sum over the axes along
// which the row block changes while the columns stay:
//
//   layout            row-stat axis     dgamma/dbeta axes
//   1D  X col split   -                 -          (X replicated)
//   1D  X row split   0                 -
//   1D  Y col split   0                 -
//   1D  Y row split   -                 -          (Y replicated)
//   2D  X, Y          1 (j)             0 (i)
//   2.5D X, Y         2 (j)             0, 1 (depth, i)
//   3D  parity 0  X   1 (b)             0, 2       Y  2 (c)  0, 1
//   3D  parity 1  X   2 (c)             0, 1       Y  1 (b)  0, 2
//
// Forward, per row (two passes, reading N1): s = sum_c x (all-reduce) -> mu = s / H;
// q = sum_c (x - mu)^2 (all-reduce) -> rstd = 1/sqrt(q / H + eps); y = (x - mu) rstd g + b.
// Backward: a = sum_c dy g, b = sum_c dy g xhat (all-reduce) -> dx = rstd (dy g - a/H - xhat
// b/H); dgamma = sum_r dy xhat, dbeta = sum_r dy (deterministic slabs, all-reduce over the row
// axes). Statistics and partial sums are fp32; reductions run over fp32 buffers.
//
// Kernels are HBM-bound streaming passes: one warp per row, 16-byte vector loads when the row
// is 16-byte aligned; the column sums use fixed row slabs summed in slab order (bit-identical
// on every replica).
#include <cuda_bf16.h>

#include "sched.h"
#include "tp_internal.h"

namespace tp {
namespace {

template <typename T>
__device__ __forceinline__ float ld_f(const T* p) {
  if constexpr (sizeof(T) == 2) return __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(p));
  else return *p;
}
template <typename T>
__device__ __forceinline__ void st_f(T* p, float v) {
  if constexpr (sizeof(T) == 2) *reinterpret_cast<__nv_bfloat16*>(p) = __float2bfloat16_rn(v);
  else *p = v;
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Visit the row's columns: f(col, value) for each element this lane owns (vectorised when
// the row start is 16-byte aligned and cols is a multiple of the vector width).
template <typename T, typename F>
__device__ __forceinline__ void row_visit(const T* row, int64_t cols, bool vec, int lane, F&& f) {
  constexpr int V = 16 / sizeof(T);
  if (vec) {
    for (int64_t c = int64_t(lane) * V; c < cols; c += 32 * V) {
      const uint4 u = *reinterpret_cast<const uint4*>(row + c);
      const T* e = reinterpret_cast<const T*>(&u);
#pragma unroll
      for (int i = 0; i < V; ++i) f(c + i, ld_f(e + i));
    }
  } else {
    for (int64_t c = lane; c < cols; c += 32) f(c, ld_f(row + c));
  }
}

// out[r] = sum_c x            (sum == nullptr)
// out[r] = sum_c (x - mu)^2   with mu = sum[r] * inv_h
template <typename T>
__global__ void ln_row_partial(const T* __restrict__ x, int64_t rows, int64_t cols, int64_t ld,
                               const float* __restrict__ sum, float inv_h, float* __restrict__ out,
                               bool vec) {
  const int64_t r = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const T* row = x + r * ld;
  float acc = 0.f;
  if (!sum) {
    row_visit(row, cols, vec, lane, [&](int64_t, float v) { acc += v; });
  } else {
    const float mu = sum[r] * inv_h;
    row_visit(row, cols, vec, lane, [&](int64_t, float v) {
      const float d = v - mu;
      acc += d * d;
    });
  }
  acc = warp_sum(acc);
  if (lane == 0) out[r] = acc;
}

template <typename T>
__global__ void ln_apply(const T* __restrict__ x, int64_t rows, int64_t cols, int64_t ld,
                         const float* __restrict__ sum, const float* __restrict__ sq, float inv_h,
                         float eps, const T* __restrict__ gamma, const T* __restrict__ beta,
                         T* __restrict__ y, float* __restrict__ stats, bool vec) {
  const int64_t r = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const float mu = sum[r] * inv_h;
  const float rstd = rsqrtf(sq[r] * inv_h + eps);
  const T* row = x + r * ld;
  T* yrow = y + r * ld;
  row_visit(row, cols, vec, lane, [&](int64_t c, float v) {
    const float g = gamma ? ld_f(gamma + c) : 1.f;
    const float b = beta ? ld_f(beta + c) : 0.f;
    st_f(yrow + c, (v - mu) * rstd * g + b);
  });
  if (lane == 0 && stats) {
    stats[2 * r] = mu;
    stats[2 * r + 1] = rstd;
  }
}

// ab[2r] = sum_c dy g, ab[2r+1] = sum_c dy g xhat
template <typename T>
__global__ void ln_bwd_row_partial(const T* __restrict__ dy, const T* __restrict__ x, int64_t rows,
                                   int64_t cols, int64_t ld, const T* __restrict__ gamma,
                                   const float* __restrict__ stats, float* __restrict__ ab, bool vec) {
  const int64_t r = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const float mu = stats[2 * r], rstd = stats[2 * r + 1];
  const T* xr = x + r * ld;
  const T* dr = dy + r * ld;
  float a = 0.f, b = 0.f;
  // dy drives the visit; x is read at the same columns
  row_visit(dr, cols, vec, lane, [&](int64_t c, float d) {
    const float g = gamma ? ld_f(gamma + c) : 1.f;
    const float xh = (ld_f(xr + c) - mu) * rstd;
    a += d * g;
    b += d * g * xh;
  });
  a = warp_sum(a);
  b = warp_sum(b);
  if (lane == 0) {
    ab[2 * r] = a;
    ab[2 * r + 1] = b;
  }
}

template <typename T>
__global__ void ln_bwd_apply(const T* __restrict__ dy, const T* __restrict__ x, int64_t rows,
                             int64_t cols, int64_t ld, const T* __restrict__ gamma,
                             const float* __restrict__ stats, const float* __restrict__ ab,
                             float inv_h, T* __restrict__ dx, bool vec) {
  const int64_t r = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const float mu = stats[2 * r], rstd = stats[2 * r + 1];
  const float ma = ab[2 * r] * inv_h, mb = ab[2 * r + 1] * inv_h;
  const T* xr = x + r * ld;
  const T* dr = dy + r * ld;
  T* out = dx + r * ld;
  row_visit(dr, cols, vec, lane, [&](int64_t c, float d) {
    const float g = gamma ? ld_f(gamma + c) : 1.f;
    const float xh = (ld_f(xr + c) - mu) * rstd;
    st_f(out + c, rstd * (d * g - ma - xh * mb));
  });
}

// part[slab][0][c] = sum_{r in slab} dy xhat, part[slab][1][c] = sum_{r in slab} dy
template <typename T>
__global__ void ln_col_partial(const T* __restrict__ dy, const T* __restrict__ x, int64_t rows,
                               int64_t cols, int64_t ld, const float* __restrict__ stats,
                               int64_t per, float* __restrict__ part) {
  const int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int slab = blockIdx.y;
  if (c >= cols) return;
  const int64_t r0 = slab * per, r1 = r0 + per < rows ? r0 + per : rows;
  float g = 0.f, b = 0.f;
  for (int64_t r = r0; r < r1; ++r) {
    const float d = ld_f(dy + r * ld + c);
    g += d * (ld_f(x + r * ld + c) - stats[2 * r]) * stats[2 * r + 1];
    b += d;
  }
  part[(int64_t(slab) * 2) * cols + c] = g;
  part[(int64_t(slab) * 2 + 1) * cols + c] = b;
}

__global__ void ln_col_final(const float* __restrict__ part, int slabs, int64_t cols,
                             float* __restrict__ out) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= 2 * cols) return;
  const int64_t which = i / cols, c = i % cols;
  float s = 0.f;
  for (int k = 0; k < slabs; ++k) s += part[(int64_t(k) * 2 + which) * cols + c];
  out[i] = s;
}

template <typename T>
__global__ void cast_out(const float* __restrict__ src, int64_t n, T* __restrict__ dst) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) st_f(dst + i, src[i]);
}

unsigned rows_grid(int64_t rows) { return static_cast<unsigned>((rows * 32 + 255) / 256); }

// Row-stat axis and gradient axes of a layout (table in the header comment); -1 = none.
struct LnAxes {
  int row = -1;
  int col[2] = {-1, -1};
};

tp_status ln_axes(const tp_grid* g, const tp_linear_desc* d, int tensor, LnAxes* a) {
  if (tensor != TP_TENSOR_X && tensor != TP_TENSOR_Y)
    return fail(TP_ERR_ARG, "layernorm: tensor must be TP_TENSOR_X or TP_TENSOR_Y");
  const bool X = tensor == TP_TENSOR_X;
  switch (g->mode) {
    case TP_1D:
      if (X ? d->split_1d == 1 : d->split_1d == 0) a->row = 0;  // the column-split one
      break;
    case TP_2D:
      a->row = 1;
      a->col[0] = 0;
      break;
    case TP_2P5D:
      a->row = 2;
      a->col[0] = 0;
      a->col[1] = 1;
      break;
    case TP_3D: {
      const bool p0 = d->parity_3d == 0;
      const bool b_is_cols = X ? p0 : !p0;  // X p0 / Y p1: column block along b (axis 1)
      a->row = b_is_cols ? 1 : 2;
      a->col[0] = 0;
      a->col[1] = b_is_cols ? 2 : 1;
      break;
    }
  }
  return TP_OK;
}

struct LnWs {
  float *s0, *s1, *q0, *q1;        // fwd: partial / reduced row sums and centred squares
  float *ab0, *ab1, *part, *cg0, *cg1;  // bwd
  int slabs;
  int64_t per;
};

void ln_carve(Carver& c, int64_t rows, int64_t cols, bool bwd, LnWs* w) {
  *w = LnWs{};
  if (!bwd) {
    w->s0 = static_cast<float*>(c.take(rows * 4));
    w->s1 = static_cast<float*>(c.take(rows * 4));
    w->q0 = static_cast<float*>(c.take(rows * 4));
    w->q1 = static_cast<float*>(c.take(rows * 4));
    return;
  }
  w->ab0 = static_cast<float*>(c.take(rows * 8));
  w->ab1 = static_cast<float*>(c.take(rows * 8));
  int64_t slabs = rows < kColsumSlabs ? rows : kColsumSlabs;
  if (slabs < 1) slabs = 1;
  w->per = (rows + slabs - 1) / slabs;
  if (w->per < 1) w->per = 1;
  w->slabs = static_cast<int>((rows + w->per - 1) / w->per);
  if (w->slabs < 1) w->slabs = 1;
  w->part = static_cast<float*>(c.take(size_t(w->slabs) * 2 * cols * 4));
  w->cg0 = static_cast<float*>(c.take(2 * cols * 4));
  w->cg1 = static_cast<float*>(c.take(2 * cols * 4));
}

tp_status ln_shape(const tp_grid* g, const tp_linear_desc* d, int tensor, Ext* e, int64_t* H) {
  TP_TRY(check_divisible(g, d));
  TP_TRY(extent(g, d, tensor, e));
  *H = tensor == TP_TENSOR_X ? d->K : d->N;
  return TP_OK;
}

// all-reduce n fp32 over grid axis `ax` (src -> dst); a size-1 / absent axis copies
tp_status ar_axis(tp_grid* g, int ax, const float* src, float* dst, int64_t n, cudaStream_t s) {
  if (ax >= 0 && g->axis[ax]) return g->axis[ax]->allreduce(src, dst, n, TP_FP32, s);
  if (src != dst) TP_CUDA(cudaMemcpyAsync(dst, src, n * 4, cudaMemcpyDeviceToDevice, s));
  return TP_OK;
}

}  // namespace

tp_status layernorm_ws_bytes(const tp_grid* g, const tp_linear_desc* d, int tensor, size_t* bytes) {
  Ext e;
  int64_t H;
  TP_TRY(ln_shape(g, d, tensor, &e, &H));
  LnAxes ax;
  TP_TRY(ln_axes(g, d, tensor, &ax));
  Carver f, b;
  LnWs w;
  ln_carve(f, e.rows, e.cols, false, &w);
  ln_carve(b, e.rows, e.cols, true, &w);
  *bytes = (f.off > b.off ? f.off : b.off) + 256;
  return TP_OK;
}

tp_status layernorm_fwd(tp_grid* g, const tp_linear_desc* d, int tensor, float eps, const void* x,
                        const void* gamma, const void* beta, void* y, float* stats, void* ws,
                        size_t ws_bytes, cudaStream_t s) {
  Ext e;
  int64_t H;
  TP_TRY(ln_shape(g, d, tensor, &e, &H));
  LnAxes ax;
  TP_TRY(ln_axes(g, d, tensor, &ax));
  size_t need = 0;
  TP_TRY(layernorm_ws_bytes(g, d, tensor, &need));
  if (ws_bytes < need || (!ws && need)) return fail(TP_ERR_WORKSPACE, "layernorm: workspace too small");
  if (e.rows == 0 || e.cols == 0) return TP_OK;
  if (!x || !y || !stats) return fail(TP_ERR_ARG, "layernorm: null x, y or stats");
  Carver c;
  c.base = static_cast<char*>(ws);
  LnWs w;
  ln_carve(c, e.rows, e.cols, false, &w);
  const float inv_h = 1.f / static_cast<float>(H);
  const bool bf = d->dtype == TP_BF16;
  const size_t esz = bf ? 2 : 4;
  const bool vec = (reinterpret_cast<uintptr_t>(x) % 16 == 0) && ((e.cols * esz) % 16 == 0) &&
                   (reinterpret_cast<uintptr_t>(y) % 16 == 0);
  const unsigned G = rows_grid(e.rows);
#define LN_T(T)                                                                                  \
  do {                                                                                           \
    ln_row_partial<T><<<G, 256, 0, s>>>(static_cast<const T*>(x), e.rows, e.cols, e.cols, nullptr, \
                                        inv_h, w.s0, vec);                                       \
    count_launch();                                                                              \
    TP_TRY(ar_axis(g, ax.row, w.s0, w.s1, e.rows, s));                                           \
    ln_row_partial<T><<<G, 256, 0, s>>>(static_cast<const T*>(x), e.rows, e.cols, e.cols, w.s1,   \
                                        inv_h, w.q0, vec);                                       \
    count_launch();                                                                              \
    TP_TRY(ar_axis(g, ax.row, w.q0, w.q1, e.rows, s));                                           \
    ln_apply<T><<<G, 256, 0, s>>>(static_cast<const T*>(x), e.rows, e.cols, e.cols, w.s1, w.q1,  \
                                  inv_h, eps, static_cast<const T*>(gamma),                      \
                                  static_cast<const T*>(beta), static_cast<T*>(y), stats, vec);  \
    count_launch();                                                                              \
  } while (0)
  if (bf) LN_T(__nv_bfloat16);
  else LN_T(float);
#undef LN_T
  TP_CUDA(cudaGetLastError());
  return TP_OK;
}

tp_status layernorm_bwd(tp_grid* g, const tp_linear_desc* d, int tensor, const void* dy,
                        const void* x, const void* gamma, const float* stats, void* dx,
                        void* dgamma, void* dbeta, void* ws, size_t ws_bytes, cudaStream_t s) {
  Ext e;
  int64_t H;
  TP_TRY(ln_shape(g, d, tensor, &e, &H));
  LnAxes ax;
  TP_TRY(ln_axes(g, d, tensor, &ax));
  size_t need = 0;
  TP_TRY(layernorm_ws_bytes(g, d, tensor, &need));
  if (ws_bytes < need || (!ws && need)) return fail(TP_ERR_WORKSPACE, "layernorm: workspace too small");
  if (e.cols == 0) return TP_OK;
  if (e.rows && (!dy || !x || !stats)) return fail(TP_ERR_ARG, "layernorm: null dy, x or stats");
  Carver c;
  c.base = static_cast<char*>(ws);
  LnWs w;
  ln_carve(c, e.rows, e.cols, true, &w);
  const float inv_h = 1.f / static_cast<float>(H);
  const bool bf = d->dtype == TP_BF16;
  const size_t esz = bf ? 2 : 4;
  const bool vec = (reinterpret_cast<uintptr_t>(dy) % 16 == 0) && ((e.cols * esz) % 16 == 0) &&
                   (!dx || reinterpret_cast<uintptr_t>(dx) % 16 == 0);
  const unsigned G = rows_grid(e.rows);
  const unsigned CB = static_cast<unsigned>((e.cols + 127) / 128);
#define LNB_T(T)                                                                                 \
  do {                                                                                           \
    if (dx && e.rows) {                                                                          \
      ln_bwd_row_partial<T><<<G, 256, 0, s>>>(static_cast<const T*>(dy), static_cast<const T*>(x), \
                                              e.rows, e.cols, e.cols, static_cast<const T*>(gamma), \
                                              stats, w.ab0, vec);                                \
      count_launch();                                                                            \
      TP_TRY(ar_axis(g, ax.row, w.ab0, w.ab1, 2 * e.rows, s));                                   \
      ln_bwd_apply<T><<<G, 256, 0, s>>>(static_cast<const T*>(dy), static_cast<const T*>(x),     \
                                        e.rows, e.cols, e.cols, static_cast<const T*>(gamma), stats, \
                                        w.ab1, inv_h, static_cast<T*>(dx), vec);                 \
      count_launch();                                                                            \
    }                                                                                            \
    if (dgamma || dbeta) {                                                                       \
      if (e.rows) {                                                                              \
        ln_col_partial<T><<<dim3(CB, w.slabs), 128, 0, s>>>(static_cast<const T*>(dy),           \
                                                            static_cast<const T*>(x), e.rows,    \
                                                            e.cols, e.cols, stats, w.per, w.part); \
        count_launch();                                                                          \
        ln_col_final<<<static_cast<unsigned>((2 * e.cols + 255) / 256), 256, 0, s>>>(            \
            w.part, w.slabs, e.cols, w.cg0);                                                     \
        count_launch();                                                                          \
      } else {                                                                                   \
        TP_CUDA(cudaMemsetAsync(w.cg0, 0, 2 * e.cols * 4, s));                                   \
      }                                                                                          \
      float* cur = w.cg0;                                                                        \
      float* nxt = w.cg1;                                                                        \
      for (int k = 0; k < 2; ++k)                                                                \
        if (ax.col[k] >= 0 && g->axis[ax.col[k]]) {                                              \
          TP_TRY(ar_axis(g, ax.col[k], cur, nxt, 2 * e.cols, s));                                \
          float* t = cur;                                                                        \
          cur = nxt;                                                                             \
          nxt = t;                                                                               \
        }                                                                                        \
      const unsigned CG = static_cast<unsigned>((e.cols + 255) / 256);                           \
      if (dgamma) {                                                                              \
        cast_out<T><<<CG, 256, 0, s>>>(cur, e.cols, static_cast<T*>(dgamma));                    \
        count_launch();                                                                          \
      }                                                                                          \
      if (dbeta) {                                                                               \
        cast_out<T><<<CG, 256, 0, s>>>(cur + e.cols, e.cols, static_cast<T*>(dbeta));           \
        count_launch();                                                                          \
      }                                                                                          \
    }                                                                                            \
  } while (0)
  if (bf) LNB_T(__nv_bfloat16);
  else LNB_T(float);
#undef LNB_T
  TP_CUDA(cudaGetLastError());
  return TP_OK;
}

}  // namespace tp
