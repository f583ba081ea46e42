// fp32-mode local GEMM ("3xTF32 ... or SIMT FFMA"): the correctness mode of
// config C1 (BASELINE.json configs[0], batch 16 x hidden 64, fp32). Plain smem-tiled FFMA,
// fp32 accumulate; relative error ~1e-7, inside the north star's 1e-5 bar that plain TF32
// misses (reading A12). Also the GEMM dispatcher and the K == 0 epilogue.
#include <cuda_bf16.h>

#include <cstdlib>

#include "tp_internal.h"

namespace tp {
namespace {

constexpr int TM = 64, TN = 64, TK = 16;

template <bool TA, bool TB>
__global__ void __launch_bounds__(256) gemm_simt_kernel(int M, int N, int K, const float* __restrict__ A,
                                                        int64_t lda, const float* __restrict__ B,
                                                        int64_t ldb, const float* C, int64_t ldc,
                                                        void* D, int64_t ldd, int out_bf16,
                                                        float alpha, const float* __restrict__ bias) {
  __shared__ float As[TK][TM + 4];
  __shared__ float Bs[TK][TN + 4];
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  const int m0 = blockIdx.y * TM, n0 = blockIdx.x * TN;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += TK) {
    for (int idx = threadIdx.x; idx < TM * TK; idx += 256) {
      int mm, kk;
      if (TA) { mm = idx % TM; kk = idx / TM; } else { kk = idx % TK; mm = idx / TK; }
      const int gm = m0 + mm, gk = k0 + kk;
      float v = 0.f;
      if (gm < M && gk < K) v = TA ? A[int64_t(gk) * lda + gm] : A[int64_t(gm) * lda + gk];
      As[kk][mm] = v;
    }
    for (int idx = threadIdx.x; idx < TN * TK; idx += 256) {
      int nn, kk;
      if (TB) { kk = idx % TK; nn = idx / TK; } else { nn = idx % TN; kk = idx / TN; }
      const int gn = n0 + nn, gk = k0 + kk;
      float v = 0.f;
      if (gn < N && gk < K) v = TB ? B[int64_t(gn) * ldb + gk] : B[int64_t(gk) * ldb + gn];
      Bs[kk][nn] = v;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < TK; ++kk) {
      float a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gm = m0 + ty * 4 + i;
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gn = n0 + tx * 4 + j;
      if (gn >= N) continue;
      float x = acc[i][j];
      if (C) x += C[int64_t(gm) * ldc + gn];
      x *= alpha;
      if (bias) x += bias[gn];
      if (out_bf16)
        reinterpret_cast<__nv_bfloat16*>(D)[int64_t(gm) * ldd + gn] = __float2bfloat16_rn(x);
      else
        reinterpret_cast<float*>(D)[int64_t(gm) * ldd + gn] = x;
    }
  }
}

__global__ void gemm_k0_kernel(int64_t M, int64_t N, const float* C, int64_t ldc, void* D,
                               int64_t ldd, int out_bf16, float alpha, const void* bias,
                               int bias_bf16) {
  const int64_t total = M * N;
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = i / N, c = i % N;
    float x = C ? C[r * ldc + c] : 0.f;
    x *= alpha;
    if (bias)
      x += bias_bf16 ? __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(bias)[c])
                     : reinterpret_cast<const float*>(bias)[c];
    if (out_bf16)
      reinterpret_cast<__nv_bfloat16*>(D)[r * ldd + c] = __float2bfloat16_rn(x);
    else
      reinterpret_cast<float*>(D)[r * ldd + c] = x;
  }
}

}  // namespace

tp_status gemm_simt_f32(const GemmArgs& g, cudaStream_t s) {
  dim3 grid(static_cast<unsigned>((g.N + TN - 1) / TN), static_cast<unsigned>((g.M + TM - 1) / TM));
  if (grid.y > 65535) return fail(TP_ERR_UNSUPPORTED, "fp32 GEMM: M too large for SIMT grid");
  const float* A = static_cast<const float*>(g.A);
  const float* B = static_cast<const float*>(g.B);
  const float* bias = static_cast<const float*>(g.bias);
  const int ob = g.out_dtype == TP_BF16;
  const int M = int(g.M), N = int(g.N), K = int(g.K);
  const int tok = prof_begin(1, s, 2.0 * double(g.M) * double(g.N) * double(g.K));
  if (!g.trans_a && !g.trans_b)
    gemm_simt_kernel<false, false><<<grid, 256, 0, s>>>(M, N, K, A, g.lda, B, g.ldb, g.C, g.ldc, g.D, g.ldd, ob, g.alpha, bias);
  else if (!g.trans_a && g.trans_b)
    gemm_simt_kernel<false, true><<<grid, 256, 0, s>>>(M, N, K, A, g.lda, B, g.ldb, g.C, g.ldc, g.D, g.ldd, ob, g.alpha, bias);
  else if (g.trans_a && !g.trans_b)
    gemm_simt_kernel<true, false><<<grid, 256, 0, s>>>(M, N, K, A, g.lda, B, g.ldb, g.C, g.ldc, g.D, g.ldd, ob, g.alpha, bias);
  else
    gemm_simt_kernel<true, true><<<grid, 256, 0, s>>>(M, N, K, A, g.lda, B, g.ldb, g.C, g.ldc, g.D, g.ldd, ob, g.alpha, bias);
  count_launch();
  prof_end(tok, s);
  TP_CUDA(cudaGetLastError());
  return TP_OK;
}

tp_status gemm_k0(const GemmArgs& g, cudaStream_t s) {
  const int64_t total = g.M * g.N;
  if (total == 0) return TP_OK;
  const int blocks = static_cast<int>(std::min<int64_t>((total + 255) / 256, 4096));
  gemm_k0_kernel<<<blocks, 256, 0, s>>>(g.M, g.N, g.C, g.ldc, g.D, g.ldd, g.out_dtype == TP_BF16,
                                        g.alpha, g.bias, g.in_dtype == TP_BF16);
  count_launch();
  TP_CUDA(cudaGetLastError());
  return TP_OK;
}

tp_status gemm(const GemmArgs& g, cudaStream_t s) {
  if (g.M < 0 || g.N < 0 || g.K < 0) return fail(TP_ERR_SHAPE, "gemm: negative dim");
  if (g.M == 0 || g.N == 0) return TP_OK;
  if (!g.D) return fail(TP_ERR_ARG, "gemm: D is null");
  const int64_t need_ldd = g.N;
  if (g.ldd < need_ldd) return fail(TP_ERR_SHAPE, "gemm: ldd < N");
  if (g.C && g.ldc < g.N) return fail(TP_ERR_SHAPE, "gemm: ldc < N");
  if (g.K == 0) return gemm_k0(g, s);
  if (!g.A || !g.B) return fail(TP_ERR_ARG, "gemm: A or B is null");
  if (g.lda < (g.trans_a ? g.M : g.K)) return fail(TP_ERR_SHAPE, "gemm: lda too small");
  if (g.ldb < (g.trans_b ? g.K : g.N)) return fail(TP_ERR_SHAPE, "gemm: ldb too small");
  if (g.M > INT32_MAX || g.N > INT32_MAX || g.K > INT32_MAX)
    return fail(TP_ERR_UNSUPPORTED, "gemm: dims must fit int32");
  if (g.dpanels > 1) {  // fused 1D reduce-scatter: D row-panels, CTA-pair kernel only
    if (g.in_dtype != TP_BF16 || g.npanels > 1 || !gemm_tc2_supported(g))
      return fail(TP_ERR_UNSUPPORTED, "gemm: D row-panels need bf16, M > 128, d_rows % 32 == 0");
    if ((reinterpret_cast<uintptr_t>(g.A) % 16) || (reinterpret_cast<uintptr_t>(g.B) % 16) ||
        (g.lda % 8) || (g.ldb % 8))
      return fail(TP_ERR_SHAPE, "gemm: TMA needs 16-byte aligned operands");
    return gemm_tc2_bf16(g, s);
  }
  if (g.npanels > 1) {  // fused peer-panel product: CTA-pair kernel only
    if (g.in_dtype != TP_BF16 || g.npanels > 4 || !gemm_tc2_supported(g))
      return fail(TP_ERR_UNSUPPORTED, "gemm: K-panels need bf16, <= 4 panels and M > 128");
    for (int p = 0; p < g.npanels; ++p)
      if (!g.Ap[p] || !g.Bp[p] || (reinterpret_cast<uintptr_t>(g.Ap[p]) % 16) ||
          (reinterpret_cast<uintptr_t>(g.Bp[p]) % 16) || (g.lda % 8) || (g.ldb % 8))
        return fail(TP_ERR_SHAPE, "gemm: K-panel operands need 16-byte aligned bases / strides");
    return gemm_tc2_bf16(g, s);
  }
  if (g.in_dtype == TP_FP32) return gemm_simt_f32(g, s);
  // TMA: 16-byte aligned bases and row strides (bf16: multiples of 8 elements)
  if ((reinterpret_cast<uintptr_t>(g.A) % 16) || (reinterpret_cast<uintptr_t>(g.B) % 16) ||
      (g.lda % 8) || (g.ldb % 8))
    return fail(TP_ERR_SHAPE,
                "gemm(bf16): TMA needs 16-byte aligned A/B and row strides that are multiples "
                "of 8 elements (lda=" + std::to_string(g.lda) + ", ldb=" + std::to_string(g.ldb) + ")");
  // Kernel choice: the CTA-pair kernel unless the problem is a single 128-row strip or the
  // output cannot take TMA stores; TP_GEMM_KERNEL=1|2 forces one (A/B measurements).
  const int force = knob("TP_GEMM_KERNEL");
  // The pair kernel needs enough 256x256 pair tiles to occupy the SM pairs; below that, the
  // streaming-bound small-M shapes run faster as 1-CTA tiles (measured, see
  // profiles/r01_gemm_v2_summary.md).
  static int sms_cache[64] = {0};
  int dev = 0;
  cudaGetDevice(&dev);
  int& sms = sms_cache[dev & 63];
  if (!sms) {
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  const int64_t pair_tiles = ((g.M + 255) / 256) * ((g.N + 255) / 256);
  // Few output tiles and a long K (e.g. C4's dW 192 x 403456 x 576: ten 1-CTA tiles) starve
  // the 1-CTA kernel, which cannot split K: the pair kernel splits K across the idle SM pairs.
  const int64_t tiles1 = ((g.M + 127) / 128) * ((g.N + 127) / 128);
  const bool long_k = tiles1 < sms / 2 && (g.K + 63) / 64 >= 64 && g.ws && g.ws_bytes;
  const bool pair_ok = force == 2 || (force == 0 && (pair_tiles >= sms / 2 || long_k));
  if (force != 1 && pair_ok && gemm_tc2_supported(g)) return gemm_tc2_bf16(g, s);
  return gemm_tc_bf16(g, s);
}

}  // namespace tp

namespace tp {

// Two independent GEMMs (e.g. a layer's dX and dW). When both are bf16 tensor-core problems
// the CTA-pair kernel takes them in ONE persistent launch, so the tiles of a small-M product
// (few tiles, long K) and of a short-K product (many tiles) share the machine instead of
// each leaving SMs idle; otherwise (or with TP_GEMM_KERNEL=1 / TP_GEMM_GROUP=0) two launches.
namespace {
bool group_eligible(const GemmArgs& g) {
  if (g.in_dtype != TP_BF16 || g.M <= 0 || g.N <= 0 || g.K <= 0 || !g.A || !g.B || !g.D ||
      g.ldd < g.N || (g.C && g.ldc < g.N) || g.lda < (g.trans_a ? g.M : g.K) ||
      g.ldb < (g.trans_b ? g.K : g.N) || g.M > INT32_MAX || g.N > INT32_MAX || g.K > INT32_MAX ||
      (g.lda % 8) || (g.ldb % 8) || g.npanels > 4 || !gemm_tc2_supported(g))
    return false;
  const int np = g.npanels > 1 ? g.npanels : 1;
  for (int p = 0; p < np; ++p) {
    const void* A = g.npanels > 1 ? g.Ap[p] : g.A;
    const void* B = g.npanels > 1 ? g.Bp[p] : g.B;
    if (!A || !B || (reinterpret_cast<uintptr_t>(A) % 16) || (reinterpret_cast<uintptr_t>(B) % 16))
      return false;
  }
  return true;
}
}  // namespace

tp_status gemm_group(const GemmArgs* gs, int n, cudaStream_t s) {
  const int force = knob("TP_GEMM_KERNEL");
  const int group_env = knob("TP_GEMM_GROUP");
  bool all = n >= 1 && n <= 4 && force != 1 && group_env;
  for (int i = 0; all && i < n; ++i) all = group_eligible(gs[i]);
  // a member that the group would split (long K: e.g. C4's token-long dW, HBM-bound, next to
  // 18912 short dX tiles) runs better in its own launch, split to fill the machine there
  // (C4 backward layer, ncu serialized: 1.88 ms grouped vs 1.69 ms as two launches;
  // profiles/r02_c2_gemm.md)
  if (all && n > 1 && knob("TP_GEMM_GROUP_LONGK") && gemm_tc2_group_splits_member(gs, n)) all = false;
  if (all && n > 1) return gemm_tc2_group(gs, n, s);
  for (int i = 0; i < n; ++i) TP_TRY(gemm(gs[i], s));
  return TP_OK;
}

tp_status gemm_pair(const GemmArgs& a, const GemmArgs& b, cudaStream_t s) {
  const GemmArgs gs[2] = {a, b};
  return gemm_group(gs, 2, s);
}

}  // namespace tp
