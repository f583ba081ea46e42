// HBM-bound helper kernels: shard pack/unpack, bias-gradient column sums
// (a-12), the seeded input generator, and the n-way sum used by the in-process transport.
// Plain coalesced CUDA with 16-byte vector accesses where alignment allows; grids are sized
// in multiples of the SM count (grid-stride loops).
#include <cuda_bf16.h>

#include "tp_internal.h"

namespace tp {
namespace {

int blocks_for(int64_t work, int per_block) {
  int64_t b = (work + per_block - 1) / per_block;
  const int64_t cap = 148 * 8;
  if (b > cap) b = cap;
  return b < 1 ? 1 : static_cast<int>(b);
}

// ---- 2-D strided copy ----------------------------------------------------------------------
__global__ void copy2d_vec16(const uint4* __restrict__ src, int64_t sld, uint4* __restrict__ dst,
                             int64_t dld, int64_t rows, int64_t cols16) {
  const int64_t total = rows * cols16;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = i / cols16, c = i % cols16;
    dst[r * dld + c] = src[r * sld + c];
  }
}

template <typename T>
__global__ void copy2d_scalar(const T* __restrict__ src, int64_t sld, T* __restrict__ dst,
                              int64_t dld, int64_t rows, int64_t cols) {
  const int64_t total = rows * cols;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = i / cols, c = i % cols;
    dst[r * dld + c] = src[r * sld + c];
  }
}

// ---- column sums: db = 1^T dY --------------------------------------------------------------
// Deterministic two-pass reduction (replicas of db on different ranks must be bit-equal):
// pass 1, block (x: 128 columns, y: row slab) sums its slab per column in fp32 into
// part[slab][col]; pass 2 sums the slabs in ascending order.
template <typename T>
__global__ void colsum_partial(const T* __restrict__ src, int64_t rows, int64_t cols, int64_t ld,
                               int64_t rows_per_slab, float* __restrict__ part) {
  const int64_t c = (blockIdx.x * int64_t(blockDim.x) + threadIdx.x);
  if (c >= cols) return;
  const int64_t r0 = blockIdx.y * rows_per_slab;
  const int64_t r1 = min(rows, r0 + rows_per_slab);
  float s = 0.f;
  for (int64_t r = r0; r < r1; ++r) {
    if constexpr (sizeof(T) == 2)
      s += __bfloat162float(src[r * ld + c]);
    else
      s += src[r * ld + c];
  }
  part[blockIdx.y * cols + c] = s;
}

template <typename T>
__global__ void colsum_final(const float* __restrict__ part, int slabs, T* __restrict__ dst,
                             int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    float s = 0.f;
    for (int k = 0; k < slabs; ++k) s += part[k * n + i];
    if constexpr (sizeof(T) == 2)
      dst[i] = __float2bfloat16_rn(s);
    else
      dst[i] = s;
  }
}

// ---- seeded generator (same counter-based SplitMix64 as synth/__init__.py) -----------------
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__global__ void fill_kernel(void* dst, int bf16, int64_t rows, int64_t cols, int64_t ld,
                            uint64_t sseed, int kind, float scale, int64_t r0, int64_t c0,
                            int64_t gcols) {
  const int64_t total = rows * cols;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = i / cols, c = i % cols;
    const uint64_t ctr = static_cast<uint64_t>(r0 + r) * static_cast<uint64_t>(gcols) +
                         static_cast<uint64_t>(c0 + c);
    const uint64_t z = mix64(sseed + (ctr + 1ull) * 0x9E3779B97F4A7C15ull);
    float v;
    if (kind == 0) {
      const int64_t n = static_cast<int64_t>(z >> 40) - (1ll << 23);
      v = __fmul_rn(static_cast<float>(n), 1.1920928955078125e-07f);  // 2^-23, exact
      v = __fmul_rn(v, scale);
    } else {
      v = static_cast<float>(static_cast<int>((z >> 32) % 3ull)) - 1.0f;
    }
    if (bf16)
      reinterpret_cast<__nv_bfloat16*>(dst)[r * ld + c] = __float2bfloat16_rn(v);
    else
      reinterpret_cast<float*>(dst)[r * ld + c] = v;
  }
}

// ---- n-way sum (in-process transport reductions) -------------------------------------------
struct Ptrs {
  const void* p[16];
};

__global__ void sum_n_bf16(Ptrs in, int n, __nv_bfloat16* __restrict__ out, size_t count) {
  const size_t pairs = count / 2;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < pairs;
       i += size_t(gridDim.x) * blockDim.x) {
    float2 s = make_float2(0.f, 0.f);
    for (int j = 0; j < n; ++j) {
      float2 f = __bfloat1622float2(reinterpret_cast<const __nv_bfloat162*>(in.p[j])[i]);
      s.x += f.x;
      s.y += f.y;
    }
    reinterpret_cast<__nv_bfloat162*>(out)[i] = __floats2bfloat162_rn(s.x, s.y);
  }
  if ((count & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    float s = 0.f;
    for (int j = 0; j < n; ++j)
      s += __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(in.p[j])[count - 1]);
    out[count - 1] = __float2bfloat16_rn(s);
  }
}

__global__ void sum_n_f32(Ptrs in, int n, float* __restrict__ out, size_t count) {
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < count;
       i += size_t(gridDim.x) * blockDim.x) {
    float s = 0.f;
    for (int j = 0; j < n; ++j) s += reinterpret_cast<const float*>(in.p[j])[i];
    out[i] = s;
  }
}

}  // namespace

tp_status launch_copy2d(const void* src, int64_t src_ld, void* dst, int64_t dst_ld, int64_t rows,
                        int64_t cols, size_t esz, cudaStream_t s) {
  if (rows <= 0 || cols <= 0) return TP_OK;
  const size_t rb = cols * esz;
  const bool vec = (reinterpret_cast<uintptr_t>(src) % 16 == 0) &&
                   (reinterpret_cast<uintptr_t>(dst) % 16 == 0) && (rb % 16 == 0) &&
                   ((src_ld * esz) % 16 == 0) && ((dst_ld * esz) % 16 == 0);
  if (vec) {
    const int64_t c16 = rb / 16;
    copy2d_vec16<<<blocks_for(rows * c16, 256), 256, 0, s>>>(
        static_cast<const uint4*>(src), src_ld * esz / 16, static_cast<uint4*>(dst),
        dst_ld * esz / 16, rows, c16);
  } else if (esz == 2) {
    copy2d_scalar<uint16_t><<<blocks_for(rows * cols, 256), 256, 0, s>>>(
        static_cast<const uint16_t*>(src), src_ld, static_cast<uint16_t*>(dst), dst_ld, rows, cols);
  } else {
    copy2d_scalar<uint32_t><<<blocks_for(rows * cols, 256), 256, 0, s>>>(
        static_cast<const uint32_t*>(src), src_ld, static_cast<uint32_t*>(dst), dst_ld, rows, cols);
  }
  count_launch();
  TP_CUDA(cudaGetLastError());
  return TP_OK;
}

tp_status launch_colsum(const void* src, int64_t rows, int64_t cols, int64_t ld, tp_dtype dt,
                        void* dst, float* scratch, cudaStream_t s) {
  if (cols <= 0) return TP_OK;
  int64_t slabs = 0;
  if (rows > 0) {
    const int64_t colblocks = (cols + 127) / 128;
    slabs = (148 * 4 + colblocks - 1) / colblocks;
    if (slabs > rows) slabs = rows;
    if (slabs < 1) slabs = 1;
    if (slabs > kColsumSlabs) slabs = kColsumSlabs;
    const int64_t per = (rows + slabs - 1) / slabs;
    slabs = (rows + per - 1) / per;
    dim3 grid(static_cast<unsigned>(colblocks), static_cast<unsigned>(slabs));
    if (dt == TP_BF16)
      colsum_partial<__nv_bfloat16><<<grid, 128, 0, s>>>(static_cast<const __nv_bfloat16*>(src),
                                                         rows, cols, ld, per, scratch);
    else
      colsum_partial<float><<<grid, 128, 0, s>>>(static_cast<const float*>(src), rows, cols, ld,
                                                 per, scratch);
    count_launch();
  }
  if (dt == TP_BF16)
    colsum_final<__nv_bfloat16><<<blocks_for(cols, 256), 256, 0, s>>>(
        scratch, static_cast<int>(slabs), static_cast<__nv_bfloat16*>(dst), cols);
  else
    colsum_final<float><<<blocks_for(cols, 256), 256, 0, s>>>(scratch, static_cast<int>(slabs),
                                                              static_cast<float*>(dst), cols);
  count_launch();
  TP_CUDA(cudaGetLastError());
  return TP_OK;
}

tp_status launch_fill(void* dst, tp_dtype dt, int64_t rows, int64_t cols, int64_t ld, uint64_t seed,
                      int tensor_id, int kind, float scale, int64_t r0, int64_t c0, int64_t gcols,
                      cudaStream_t s) {
  if (rows <= 0 || cols <= 0) return TP_OK;
  // stream seed s_t = mix(seed + (tensor_id + 1) * GOLDEN)   (synth.stream_seed)
  uint64_t z = seed + static_cast<uint64_t>(tensor_id + 1) * 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  const uint64_t sseed = z ^ (z >> 31);
  fill_kernel<<<blocks_for(rows * cols, 256), 256, 0, s>>>(dst, dt == TP_BF16, rows, cols, ld, sseed,
                                                           kind, scale, r0, c0, gcols);
  count_launch();
  TP_CUDA(cudaGetLastError());
  return TP_OK;
}

tp_status launch_sum_n(const void* const* in, int n, void* out, size_t count, tp_dtype dt,
                       cudaStream_t s) {
  if (count == 0) return TP_OK;
  if (n < 1 || n > 16) return fail(TP_ERR_UNSUPPORTED, "sum_n: 1..16 inputs");
  Ptrs p{};
  for (int i = 0; i < n; ++i) p.p[i] = in[i];
  if (dt == TP_BF16)
    sum_n_bf16<<<blocks_for(static_cast<int64_t>(count / 2 + 1), 256), 256, 0, s>>>(
        p, n, static_cast<__nv_bfloat16*>(out), count);
  else
    sum_n_f32<<<blocks_for(static_cast<int64_t>(count), 256), 256, 0, s>>>(p, n, static_cast<float*>(out),
                                                                           count);
  count_launch();
  TP_CUDA(cudaGetLastError());
  return TP_OK;
}

tp_status launch_memset(void* dst, size_t bytes, cudaStream_t s) {
  if (bytes) TP_CUDA(cudaMemsetAsync(dst, 0, bytes, s));
  return TP_OK;
}


// ------------------------------------------------------------------------------------ GeLU
// gelu(z) = z Phi(z) = 0.5 z (1 + erf(z / sqrt 2)), gelu'(z) = Phi(z) + z phi(z) (fp32 math,
// exact erf form; oracle/activation.py). Elementwise over the Y shard; 16-byte vectors.
namespace {
__device__ __forceinline__ float gelu_f(float z) { return 0.5f * z * (1.f + erff(z * 0.70710678118654752f)); }
__device__ __forceinline__ float gelu_grad_f(float z) {
  const float Phi = 0.5f * (1.f + erff(z * 0.70710678118654752f));
  return Phi + z * 0.39894228040143268f * __expf(-0.5f * z * z);
}
template <typename T>
__device__ __forceinline__ float to_f(T v) {
  if constexpr (sizeof(T) == 2) return __bfloat162float(v);
  else return v;
}
template <typename T>
__device__ __forceinline__ T from_f(float v) {
  if constexpr (sizeof(T) == 2) return __float2bfloat16_rn(v);
  else return v;
}

template <typename T>
__global__ void gelu_fwd_kernel(T* __restrict__ y, T* __restrict__ z, size_t n) {
  constexpr int V = 16 / sizeof(T);
  const size_t nv = n / V;
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nv; i += stride) {
    uint4 u = reinterpret_cast<const uint4*>(y)[i];
    reinterpret_cast<uint4*>(z)[i] = u;
    T* e = reinterpret_cast<T*>(&u);
#pragma unroll
    for (int j = 0; j < V; ++j) e[j] = from_f<T>(gelu_f(to_f(e[j])));
    reinterpret_cast<uint4*>(y)[i] = u;
  }
  for (size_t i = nv * V + size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) {
    const T v = y[i];
    z[i] = v;
    y[i] = from_f<T>(gelu_f(to_f(v)));
  }
}

template <typename T>
__global__ void gelu_bwd_kernel(const T* __restrict__ dy, const T* __restrict__ z, T* __restrict__ dz,
                                size_t n) {
  constexpr int V = 16 / sizeof(T);
  const size_t nv = n / V;
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nv; i += stride) {
    const uint4 a = reinterpret_cast<const uint4*>(dy)[i];
    const uint4 b = reinterpret_cast<const uint4*>(z)[i];
    uint4 o;
    const T* ea = reinterpret_cast<const T*>(&a);
    const T* eb = reinterpret_cast<const T*>(&b);
    T* eo = reinterpret_cast<T*>(&o);
#pragma unroll
    for (int j = 0; j < V; ++j) eo[j] = from_f<T>(to_f(ea[j]) * gelu_grad_f(to_f(eb[j])));
    reinterpret_cast<uint4*>(dz)[i] = o;
  }
  for (size_t i = nv * V + size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    dz[i] = from_f<T>(to_f(dy[i]) * gelu_grad_f(to_f(z[i])));
}

unsigned elem_grid(size_t n) {
  const size_t b = (n / 8 + 255) / 256;
  return static_cast<unsigned>(b < 148 * 16 ? (b > 0 ? b : 1) : 148 * 16);
}
}  // namespace

tp_status launch_gelu_fwd(void* y, void* z, size_t n, tp_dtype dt, cudaStream_t s) {
  if (!n) return TP_OK;
  if ((reinterpret_cast<uintptr_t>(y) | reinterpret_cast<uintptr_t>(z)) % 16)
    return fail(TP_ERR_SHAPE, "gelu: 16-byte aligned buffers required");
  if (dt == TP_BF16)
    gelu_fwd_kernel<__nv_bfloat16><<<elem_grid(n), 256, 0, s>>>(static_cast<__nv_bfloat16*>(y),
                                                               static_cast<__nv_bfloat16*>(z), n);
  else
    gelu_fwd_kernel<float><<<elem_grid(n), 256, 0, s>>>(static_cast<float*>(y), static_cast<float*>(z), n);
  count_launch();
  TP_CUDA(cudaGetLastError());
  return TP_OK;
}

tp_status launch_gelu_bwd(const void* dy, const void* z, void* dz, size_t n, tp_dtype dt,
                          cudaStream_t s) {
  if (!n) return TP_OK;
  if ((reinterpret_cast<uintptr_t>(dy) | reinterpret_cast<uintptr_t>(z) |
       reinterpret_cast<uintptr_t>(dz)) % 16)
    return fail(TP_ERR_SHAPE, "gelu: 16-byte aligned buffers required");
  if (dt == TP_BF16)
    gelu_bwd_kernel<__nv_bfloat16><<<elem_grid(n), 256, 0, s>>>(
        static_cast<const __nv_bfloat16*>(dy), static_cast<const __nv_bfloat16*>(z),
        static_cast<__nv_bfloat16*>(dz), n);
  else
    gelu_bwd_kernel<float><<<elem_grid(n), 256, 0, s>>>(static_cast<const float*>(dy),
                                                       static_cast<const float*>(z),
                                                       static_cast<float*>(dz), n);
  count_launch();
  TP_CUDA(cudaGetLastError());
  return TP_OK;
}


// ------------------------------------------------------------------------------ residual add
namespace {
template <typename T>
__global__ void add_kernel(const T* __restrict__ a, const T* __restrict__ b, T* __restrict__ out, size_t n) {
  constexpr int V = 16 / sizeof(T);
  const size_t nv = n / V;
  const size_t stride = size_t(gridDim.x) * blockDim.x;
  for (size_t i = size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < nv; i += stride) {
    const uint4 x = reinterpret_cast<const uint4*>(a)[i];
    const uint4 y = reinterpret_cast<const uint4*>(b)[i];
    uint4 o;
    const T* ex = reinterpret_cast<const T*>(&x);
    const T* ey = reinterpret_cast<const T*>(&y);
    T* eo = reinterpret_cast<T*>(&o);
#pragma unroll
    for (int j = 0; j < V; ++j) eo[j] = from_f<T>(to_f(ex[j]) + to_f(ey[j]));
    reinterpret_cast<uint4*>(out)[i] = o;
  }
  for (size_t i = nv * V + size_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = from_f<T>(to_f(a[i]) + to_f(b[i]));
}
}  // namespace

tp_status launch_add(const void* a, const void* b, void* out, size_t n, tp_dtype dt, cudaStream_t s) {
  if (!n) return TP_OK;
  if ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b) | reinterpret_cast<uintptr_t>(out)) % 16)
    return fail(TP_ERR_SHAPE, "add: 16-byte aligned buffers required");
  if (dt == TP_BF16)
    add_kernel<__nv_bfloat16><<<elem_grid(n), 256, 0, s>>>(static_cast<const __nv_bfloat16*>(a),
                                                          static_cast<const __nv_bfloat16*>(b),
                                                          static_cast<__nv_bfloat16*>(out), n);
  else
    add_kernel<float><<<elem_grid(n), 256, 0, s>>>(static_cast<const float*>(a), static_cast<const float*>(b),
                                                  static_cast<float*>(out), n);
  count_launch();
  TP_CUDA(cudaGetLastError());
  return TP_OK;
}

}  // namespace tp
