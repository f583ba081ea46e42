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
// Kernels are HBM-bound streaming passes. Fast path (16-byte aligned rows, <= 4096 vectors
// per row): a CTA holds a whole row in registers, so the forward reads x once (no reduction)
// or twice (the row group exchanges per-row (count, mean, M2) partials by all-gather and
// combines them in member order, Chan et al.), and the backward reads (dy, x) once (or twice)
// and accumulates dgamma / dbeta per CTA in shared memory. Fallback: one warp per row, three
// passes. Every sum has a fixed order: replicas are bit-identical.
#include <cuda_bf16.h>

#include <utility>

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

// Stage 1 of the slab sum when there are many slabs: mid[grp][i] = sum of 32 consecutive slabs.
__global__ void ln_col_mid(const float* __restrict__ part, int slabs, int64_t cols,
                           float* __restrict__ mid) {
  const int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= 2 * cols) return;
  const int grp = blockIdx.y;
  const int k0 = grp * 32, k1 = k0 + 32 < slabs ? k0 + 32 : slabs;
  float s = 0.f;
  for (int k = k0; k < k1; ++k) s += part[int64_t(k) * 2 * cols + i];
  mid[int64_t(grp) * 2 * cols + i] = s;
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

// ---------------------------------------------------------------- row-resident fast path
// TPR threads hold one row in registers (VPT 16-byte vectors each); a 256-thread CTA holds
// 256/TPR rows. A pass reads each element once; statistics are group sums in a fixed order.
constexpr int kRT = 256;

// Sum (a, b) over the TPR threads of this thread's row group (fixed order, deterministic).
template <int TPR>
__device__ __forceinline__ void group_sum2(float& a, float& b, float (*sh)[2]) {
  a = warp_sum(a);
  b = warp_sum(b);
  if constexpr (TPR > 32) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int W = TPR / 32;
    if (lane == 0) {
      sh[warp][0] = a;
      sh[warp][1] = b;
    }
    __syncthreads();
    const int w0 = (warp / W) * W;
    float ta = 0.f, tb = 0.f;
#pragma unroll
    for (int w = 0; w < W; ++w) {
      ta += sh[w0 + w][0];
      tb += sh[w0 + w][1];
    }
    __syncthreads();
    a = ta;
    b = tb;
  }
}

template <typename T, int TPR, int VPT>
struct RowV {
  static constexpr int V = 16 / sizeof(T);
  float v[VPT][V];
  __device__ __forceinline__ void load(const T* row, int64_t nvec, int t, bool ok) {
#pragma unroll
    for (int i = 0; i < VPT; ++i) {
      const int64_t k = t + int64_t(i) * TPR;
      if (ok && k < nvec) {
        const uint4 u = __ldg(reinterpret_cast<const uint4*>(row) + k);
        const T* e = reinterpret_cast<const T*>(&u);
#pragma unroll
        for (int j = 0; j < V; ++j) v[i][j] = ld_f(e + j);
      } else {
#pragma unroll
        for (int j = 0; j < V; ++j) v[i][j] = 0.f;
      }
    }
  }
};

template <typename T, int V>
__device__ __forceinline__ void store_vec(T* dst, const float (&f)[V]) {
  uint4 u;
  T* e = reinterpret_cast<T*>(&u);
#pragma unroll
  for (int j = 0; j < V; ++j) st_f(e + j, f[j]);
  *reinterpret_cast<uint4*>(dst) = u;
}

template <typename T, int V>
__device__ __forceinline__ void load_vec(const T* p, float (&f)[V]) {
  if (!p) {
#pragma unroll
    for (int j = 0; j < V; ++j) f[j] = 0.f;
    return;
  }
  const uint4 u = __ldg(reinterpret_cast<const uint4*>(p));
  const T* e = reinterpret_cast<const T*>(&u);
#pragma unroll
  for (int j = 0; j < V; ++j) f[j] = ld_f(e + j);
}

// mode 0: complete statistics locally, write y and stats.
// mode 1: write this rank's partial (count, mean, M2) of each row to part[3r..].
// mode 2: apply with the given stats (y only).
template <typename T, int TPR, int VPT>
__global__ void __launch_bounds__(kRT) ln_fwd_rows(const T* __restrict__ x, int64_t rows, int64_t cols,
                                                    float eps, const T* __restrict__ gamma,
                                                    const T* __restrict__ beta, T* __restrict__ y,
                                                    float* __restrict__ stats, float* __restrict__ part,
                                                    int mode) {
  using R = RowV<T, TPR, VPT>;
  constexpr int V = R::V;
  __shared__ float sh[kRT / 32][2];
  const int64_t nvec = cols / V;
  const int t = threadIdx.x % TPR;
  const int64_t r = int64_t(blockIdx.x) * (kRT / TPR) + threadIdx.x / TPR;
  const bool ok = r < rows;
  R row;
  row.load(x + (ok ? r : 0) * cols, nvec, t, ok);
  float mu, rstd;
  if (mode == 2) {
    mu = ok ? stats[2 * r] : 0.f;
    rstd = ok ? stats[2 * r + 1] : 0.f;
  } else {
    float sum = 0.f, z = 0.f;
#pragma unroll
    for (int i = 0; i < VPT; ++i)
#pragma unroll
      for (int j = 0; j < V; ++j) sum += row.v[i][j];
    group_sum2<TPR>(sum, z, sh);
    mu = sum / static_cast<float>(cols);
    float m2 = 0.f;
    z = 0.f;
#pragma unroll
    for (int i = 0; i < VPT; ++i) {
      if (t + int64_t(i) * TPR >= nvec) continue;
#pragma unroll
      for (int j = 0; j < V; ++j) {
        const float dd = row.v[i][j] - mu;
        m2 += dd * dd;
      }
    }
    group_sum2<TPR>(m2, z, sh);
    if (mode == 1) {
      if (ok && t == 0) {
        part[3 * r] = static_cast<float>(cols);
        part[3 * r + 1] = mu;
        part[3 * r + 2] = m2;
      }
      return;
    }
    rstd = rsqrtf(m2 / static_cast<float>(cols) + eps);
    if (ok && t == 0) {
      stats[2 * r] = mu;
      stats[2 * r + 1] = rstd;
    }
  }
  if (!ok) return;
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const int64_t k = t + int64_t(i) * TPR;
    if (k >= nvec) continue;
    float gv[V], bv[V], o[V];
    load_vec<T, V>(gamma ? gamma + k * V : nullptr, gv);
    load_vec<T, V>(beta ? beta + k * V : nullptr, bv);
#pragma unroll
    for (int j = 0; j < V; ++j) o[j] = (row.v[i][j] - mu) * rstd * (gamma ? gv[j] : 1.f) + bv[j];
    store_vec<T, V>(y + r * cols + k * V, o);
  }
}

// Combine the row-group members' (count, mean, M2) in member order (Chan et al.): stats.
__global__ void ln_combine(const float* __restrict__ parts, int members, int64_t rows, float eps,
                           float* __restrict__ stats) {
  const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  float n = parts[3 * r], mu = parts[3 * r + 1], m2 = parts[3 * r + 2];
  for (int k = 1; k < members; ++k) {
    const float* q = parts + (int64_t(k) * rows + r) * 3;
    const float nb = q[0], d = q[1] - mu, nn = n + nb;
    mu += d * nb / nn;
    m2 += q[2] + d * d * n * nb / nn;
    n = nn;
  }
  stats[2 * r] = mu;
  stats[2 * r + 1] = rsqrtf(m2 / n + eps);
}

// Backward rows. mode 0: local row sums -> dx. mode 1: write ab[2r..] = (a, b) only.
// mode 2: dx from the reduced ab.
template <typename T, int TPR, int VPT>
__global__ void __launch_bounds__(kRT) ln_bwd_rows(const T* __restrict__ dy, const T* __restrict__ x,
                                                    int64_t rows, int64_t cols,
                                                    const T* __restrict__ gamma,
                                                    const float* __restrict__ stats,
                                                    float* __restrict__ ab, float inv_h,
                                                    T* __restrict__ dx, int mode) {
  using R = RowV<T, TPR, VPT>;
  constexpr int V = R::V;
  __shared__ float sh[kRT / 32][2];
  const int64_t nvec = cols / V;
  const int t = threadIdx.x % TPR;
  const int64_t r = int64_t(blockIdx.x) * (kRT / TPR) + threadIdx.x / TPR;
  const bool ok = r < rows;
  R xr, dr;
  xr.load(x + (ok ? r : 0) * cols, nvec, t, ok);
  dr.load(dy + (ok ? r : 0) * cols, nvec, t, ok);
  const float mu = ok ? stats[2 * r] : 0.f, rstd = ok ? stats[2 * r + 1] : 0.f;
  float ma, mb;
  if (mode == 2) {
    ma = ok ? ab[2 * r] * inv_h : 0.f;
    mb = ok ? ab[2 * r + 1] * inv_h : 0.f;
  } else {
    float a = 0.f, b = 0.f;
#pragma unroll
    for (int i = 0; i < VPT; ++i) {
      const int64_t k = t + int64_t(i) * TPR;
      if (k >= nvec) continue;
      float gv[V];
      load_vec<T, V>(gamma ? gamma + k * V : nullptr, gv);
#pragma unroll
      for (int j = 0; j < V; ++j) {
        const float g = gamma ? gv[j] : 1.f;
        const float xh = (xr.v[i][j] - mu) * rstd;
        a += dr.v[i][j] * g;
        b += dr.v[i][j] * g * xh;
      }
    }
    group_sum2<TPR>(a, b, sh);
    if (mode == 1) {
      if (ok && t == 0) {
        ab[2 * r] = a;
        ab[2 * r + 1] = b;
      }
      return;
    }
    ma = a * inv_h;
    mb = b * inv_h;
  }
  if (!ok) return;
#pragma unroll
  for (int i = 0; i < VPT; ++i) {
    const int64_t k = t + int64_t(i) * TPR;
    if (k >= nvec) continue;
    float gv[V], o[V];
    load_vec<T, V>(gamma ? gamma + k * V : nullptr, gv);
#pragma unroll
    for (int j = 0; j < V; ++j) {
      const float xh = (xr.v[i][j] - mu) * rstd;
      o[j] = rstd * (dr.v[i][j] * (gamma ? gv[j] : 1.f) - ma - xh * mb);
    }
    store_vec<T, V>(dx + r * cols + k * V, o);
  }
}

// dgamma / dbeta partials over fixed row slabs, one 16-byte column vector per thread:
// part[slab][0][c] = sum_{r in slab} dy xhat, part[slab][1][c] = sum_{r in slab} dy.
template <typename T>
__global__ void ln_col_partial_v(const T* __restrict__ dy, const T* __restrict__ x, int64_t rows,
                                 int64_t cols, const float* __restrict__ stats, int64_t per,
                                 float* __restrict__ part) {
  constexpr int V = 16 / sizeof(T);
  const int64_t k = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  const int64_t nvec = cols / V;
  if (k >= nvec) return;
  const int64_t slab = blockIdx.y;
  const int64_t r0 = slab * per, r1 = r0 + per < rows ? r0 + per : rows;
  float g[V], b[V];
#pragma unroll
  for (int j = 0; j < V; ++j) g[j] = b[j] = 0.f;
  int64_t r = r0;
  for (; r + 4 <= r1; r += 4) {  // 8 independent 16-byte loads in flight per thread
    float dv[4][V], xv[4][V];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      load_vec<T, V>(dy + (r + u) * cols + k * V, dv[u]);
      load_vec<T, V>(x + (r + u) * cols + k * V, xv[u]);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const float mu = stats[2 * (r + u)], rstd = stats[2 * (r + u) + 1];
#pragma unroll
      for (int j = 0; j < V; ++j) {
        g[j] += dv[u][j] * (xv[u][j] - mu) * rstd;
        b[j] += dv[u][j];
      }
    }
  }
  for (; r < r1; ++r) {
    float dv[V], xv[V];
    load_vec<T, V>(dy + r * cols + k * V, dv);
    load_vec<T, V>(x + r * cols + k * V, xv);
    const float mu = stats[2 * r], rstd = stats[2 * r + 1];
#pragma unroll
    for (int j = 0; j < V; ++j) {
      g[j] += dv[j] * (xv[j] - mu) * rstd;
      b[j] += dv[j];
    }
  }
  float* pg = part + (slab * 2) * cols + k * V;
  float* pb = part + (slab * 2 + 1) * cols + k * V;
#pragma unroll
  for (int j = 0; j < V; ++j) {
    pg[j] = g[j];
    pb[j] = b[j];
  }
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
  float *wp, *wall;                // fast fwd: (count, mean, M2) partials, gathered over the row group
  float* colpart;                  // fast bwd: per-slab dgamma / dbeta partials
  float* colmid;                   // fast bwd: sums of 32 slabs
  int slabs;
  int64_t per;
};

constexpr int kLnCtasPerSm = 2;  // fast-path persistent grid (CTAs per SM)
constexpr int kLnColSlabs = 1024;  // fast-path dgamma / dbeta row slabs (max)

int ln_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

int64_t ln_grid(int64_t rows) {
  const int64_t g = int64_t(ln_sms()) * kLnCtasPerSm;
  return rows < g ? (rows > 0 ? rows : 1) : g;
}

void ln_carve(Carver& c, int64_t rows, int64_t cols, bool bwd, LnWs* w, int members = 1) {
  *w = LnWs{};
  if (!bwd) {
    w->s0 = static_cast<float*>(c.take(rows * 4));
    w->s1 = static_cast<float*>(c.take(rows * 4));
    w->q0 = static_cast<float*>(c.take(rows * 4));
    w->q1 = static_cast<float*>(c.take(rows * 4));
    w->wp = static_cast<float*>(c.take(rows * 12));
    w->wall = static_cast<float*>(c.take(size_t(members) * rows * 12));
    return;
  }
  w->colpart = static_cast<float*>(c.take(size_t(kLnColSlabs) * 2 * cols * 4));
  w->colmid = static_cast<float*>(c.take(size_t(kLnColSlabs / 32) * 2 * cols * 4));
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


// TPR (threads per row) and VPT (16-byte vectors per thread) for a row of nvec vectors:
// about 4 vectors per thread, 32..256 threads per row; 0 when the row is too long.
void ln_shape_choice(int64_t nvec, int* tpr, int* vpt) {
  int t = 32;
  while (t < kRT && int64_t(t) * 4 < nvec) t *= 2;
  int v = 1;
  while (v < 8 && int64_t(t) * v < nvec) v *= 2;
  if (int64_t(t) * v < nvec) {
    *tpr = *vpt = 0;
    return;
  }
  *tpr = t;
  *vpt = v;
}

template <typename T, int TPR>
tp_status ln_fwd_launch_t(int vpt, unsigned grid, cudaStream_t s, const void* x, int64_t rows,
                          int64_t cols, float eps, const void* gamma, const void* beta, void* y,
                          float* stats, float* part, int mode) {
#define LF(VP)                                                                                   \
  ln_fwd_rows<T, TPR, VP><<<grid, kRT, 0, s>>>(static_cast<const T*>(x), rows, cols, eps,         \
                                                static_cast<const T*>(gamma),                      \
                                                static_cast<const T*>(beta), static_cast<T*>(y),   \
                                                stats, part, mode)
  switch (vpt) {
    case 1: LF(1); break;
    case 2: LF(2); break;
    case 4: LF(4); break;
    default: LF(8); break;
  }
#undef LF
  count_launch();
  return TP_OK;
}

template <typename T>
tp_status ln_fwd_launch(int tpr, int vpt, unsigned grid, cudaStream_t s, const void* x, int64_t rows,
                        int64_t cols, float eps, const void* gamma, const void* beta, void* y,
                        float* stats, float* part, int mode) {
  switch (tpr) {
    case 32: return ln_fwd_launch_t<T, 32>(vpt, grid, s, x, rows, cols, eps, gamma, beta, y, stats, part, mode);
    case 64: return ln_fwd_launch_t<T, 64>(vpt, grid, s, x, rows, cols, eps, gamma, beta, y, stats, part, mode);
    case 128: return ln_fwd_launch_t<T, 128>(vpt, grid, s, x, rows, cols, eps, gamma, beta, y, stats, part, mode);
    default: return ln_fwd_launch_t<T, 256>(vpt, grid, s, x, rows, cols, eps, gamma, beta, y, stats, part, mode);
  }
}

template <typename T, int TPR>
tp_status ln_bwd_launch_t(int vpt, unsigned grid, cudaStream_t s, const void* dy, const void* x,
                          int64_t rows, int64_t cols, const void* gamma, const float* stats,
                          float* ab, float inv_h, void* dx, int mode) {
#define LB(VP)                                                                                   \
  ln_bwd_rows<T, TPR, VP><<<grid, kRT, 0, s>>>(static_cast<const T*>(dy), static_cast<const T*>(x), \
                                                rows, cols, static_cast<const T*>(gamma), stats,   \
                                                ab, inv_h, static_cast<T*>(dx), mode)
  switch (vpt) {
    case 1: LB(1); break;
    case 2: LB(2); break;
    case 4: LB(4); break;
    default: LB(8); break;
  }
#undef LB
  count_launch();
  return TP_OK;
}

template <typename T>
tp_status ln_bwd_launch(int tpr, int vpt, unsigned grid, cudaStream_t s, const void* dy,
                        const void* x, int64_t rows, int64_t cols, const void* gamma,
                        const float* stats, float* ab, float inv_h, void* dx, int mode) {
  switch (tpr) {
    case 32: return ln_bwd_launch_t<T, 32>(vpt, grid, s, dy, x, rows, cols, gamma, stats, ab, inv_h, dx, mode);
    case 64: return ln_bwd_launch_t<T, 64>(vpt, grid, s, dy, x, rows, cols, gamma, stats, ab, inv_h, dx, mode);
    case 128: return ln_bwd_launch_t<T, 128>(vpt, grid, s, dy, x, rows, cols, gamma, stats, ab, inv_h, dx, mode);
    default: return ln_bwd_launch_t<T, 256>(vpt, grid, s, dy, x, rows, cols, gamma, stats, ab, inv_h, dx, mode);
  }
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
  const int members = (ax.row >= 0 && g->axis[ax.row]) ? g->dims[ax.row] : 1;
  ln_carve(f, e.rows, e.cols, false, &w, members);
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
  const bool reduce = ax.row >= 0 && g->axis[ax.row];
  const int members = reduce ? g->dims[ax.row] : 1;
  ln_carve(c, e.rows, e.cols, false, &w, members);
  const float inv_h = 1.f / static_cast<float>(H);
  const bool bf = d->dtype == TP_BF16;
  const size_t esz = bf ? 2 : 4;
  const bool vec = (reinterpret_cast<uintptr_t>(x) % 16 == 0) && ((e.cols * esz) % 16 == 0) &&
                   (reinterpret_cast<uintptr_t>(y) % 16 == 0) &&
                   (reinterpret_cast<uintptr_t>(gamma) % 16 == 0) &&
                   (reinterpret_cast<uintptr_t>(beta) % 16 == 0);
  int tpr = 0, vpt = 0;
  if (vec) ln_shape_choice(e.cols / (16 / int64_t(esz)), &tpr, &vpt);
  if (vpt) {  // row-resident fast path: x read once (no reduction) or twice
    const unsigned GR = static_cast<unsigned>((e.rows + (kRT / tpr) - 1) / (kRT / tpr));
    const int mode = reduce ? 1 : 0;
    if (bf)
      TP_TRY(ln_fwd_launch<__nv_bfloat16>(tpr, vpt, GR, s, x, e.rows, e.cols, eps, gamma, beta, y,
                                          stats, w.wp, mode));
    else
      TP_TRY(ln_fwd_launch<float>(tpr, vpt, GR, s, x, e.rows, e.cols, eps, gamma, beta, y, stats,
                                  w.wp, mode));
    if (reduce) {
      TP_TRY(g->axis[ax.row]->allgather(w.wp, w.wall, 3 * e.rows, TP_FP32, s));
      ln_combine<<<static_cast<unsigned>((e.rows + 255) / 256), 256, 0, s>>>(w.wall, members, e.rows,
                                                                           eps, stats);
      count_launch();
      if (bf)
        TP_TRY(ln_fwd_launch<__nv_bfloat16>(tpr, vpt, GR, s, x, e.rows, e.cols, eps, gamma, beta,
                                            y, stats, w.wp, 2));
      else
        TP_TRY(ln_fwd_launch<float>(tpr, vpt, GR, s, x, e.rows, e.cols, eps, gamma, beta, y, stats,
                                    w.wp, 2));
    }
    TP_CUDA(cudaGetLastError());
    return TP_OK;
  }
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
                   (!dx || reinterpret_cast<uintptr_t>(dx) % 16 == 0) &&
                   (reinterpret_cast<uintptr_t>(x) % 16 == 0) &&
                   (reinterpret_cast<uintptr_t>(gamma) % 16 == 0);
  int tpr = 0, vpt = 0;
  if (vec) ln_shape_choice(e.cols / (16 / int64_t(esz)), &tpr, &vpt);
  const bool want_cols = dgamma || dbeta;
  if (vpt && e.rows) {
    const bool reduce = ax.row >= 0 && g->axis[ax.row];
    const unsigned GR = static_cast<unsigned>((e.rows + (kRT / tpr) - 1) / (kRT / tpr));
    if (dx) {
      if (bf)
        TP_TRY(ln_bwd_launch<__nv_bfloat16>(tpr, vpt, GR, s, dy, x, e.rows, e.cols, gamma, stats,
                                            w.ab0, inv_h, dx, reduce ? 1 : 0));
      else
        TP_TRY(ln_bwd_launch<float>(tpr, vpt, GR, s, dy, x, e.rows, e.cols, gamma, stats, w.ab0,
                                    inv_h, dx, reduce ? 1 : 0));
      if (reduce) {
        TP_TRY(ar_axis(g, ax.row, w.ab0, w.ab1, 2 * e.rows, s));
        if (bf)
          TP_TRY(ln_bwd_launch<__nv_bfloat16>(tpr, vpt, GR, s, dy, x, e.rows, e.cols, gamma, stats,
                                              w.ab1, inv_h, dx, 2));
        else
          TP_TRY(ln_bwd_launch<float>(tpr, vpt, GR, s, dy, x, e.rows, e.cols, gamma, stats, w.ab1,
                                      inv_h, dx, 2));
      }
    }
    if (want_cols) {
      const int64_t nv = e.cols / (16 / int64_t(esz));
      // enough (slab x column-vector) threads to fill the machine, at most kLnColSlabs slabs
      int64_t slabs = (262144 + nv - 1) / nv;
      if (slabs < 256) slabs = 256;
      if (slabs > kLnColSlabs) slabs = kLnColSlabs;
      if (slabs > e.rows) slabs = e.rows;
      const int64_t per = (e.rows + slabs - 1) / slabs;
      slabs = (e.rows + per - 1) / per;
      const dim3 grid(static_cast<unsigned>((nv + 127) / 128), static_cast<unsigned>(slabs));
      if (bf)
        ln_col_partial_v<__nv_bfloat16><<<grid, 128, 0, s>>>(static_cast<const __nv_bfloat16*>(dy),
                                                            static_cast<const __nv_bfloat16*>(x),
                                                            e.rows, e.cols, stats, per, w.colpart);
      else
        ln_col_partial_v<float><<<grid, 128, 0, s>>>(static_cast<const float*>(dy),
                                                    static_cast<const float*>(x), e.rows, e.cols,
                                                    stats, per, w.colpart);
      count_launch();
      if (slabs > 32) {
        const int grps = static_cast<int>((slabs + 31) / 32);
        ln_col_mid<<<dim3(static_cast<unsigned>((2 * e.cols + 255) / 256), grps), 256, 0, s>>>(
            w.colpart, static_cast<int>(slabs), e.cols, w.colmid);
        ln_col_final<<<static_cast<unsigned>((2 * e.cols + 255) / 256), 256, 0, s>>>(
            w.colmid, grps, e.cols, w.cg0);
        count_launch(2);
      } else {
        ln_col_final<<<static_cast<unsigned>((2 * e.cols + 255) / 256), 256, 0, s>>>(
            w.colpart, static_cast<int>(slabs), e.cols, w.cg0);
        count_launch();
      }
      float* cur = w.cg0;
      float* nxt = w.cg1;
      for (int k = 0; k < 2; ++k)
        if (ax.col[k] >= 0 && g->axis[ax.col[k]]) {
          TP_TRY(ar_axis(g, ax.col[k], cur, nxt, 2 * e.cols, s));
          std::swap(cur, nxt);
        }
      const unsigned CG = static_cast<unsigned>((e.cols + 255) / 256);
      if (bf) {
        if (dgamma) cast_out<__nv_bfloat16><<<CG, 256, 0, s>>>(cur, e.cols, static_cast<__nv_bfloat16*>(dgamma));
        if (dbeta) cast_out<__nv_bfloat16><<<CG, 256, 0, s>>>(cur + e.cols, e.cols, static_cast<__nv_bfloat16*>(dbeta));
      } else {
        if (dgamma) cast_out<float><<<CG, 256, 0, s>>>(cur, e.cols, static_cast<float*>(dgamma));
        if (dbeta) cast_out<float><<<CG, 256, 0, s>>>(cur + e.cols, e.cols, static_cast<float*>(dbeta));
      }
      count_launch((dgamma ? 1 : 0) + (dbeta ? 1 : 0));
    }
    TP_CUDA(cudaGetLastError());
    return TP_OK;
  }
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
