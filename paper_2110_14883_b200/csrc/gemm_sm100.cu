// tcgen05 / TMEM / TMA bf16 GEMM for sm_100a — the local shard product of every TP mode
// ("NN / NT / TN on row-major shards ... bf16 x bf16 -> fp32 accumulate";
// P:L389 "tensor parallelism is mainly applied to matrix-matrix multiplication").
//
//   D[M,N] = alpha * (op(A) . op(B) + C) + bias[col]
//
// Design (B200-first):
//   * persistent: grid = min(#tiles, #SMs), static strided tile schedule, grouped raster
//     (bands of 16 M-blocks) so a wave's A/B panels stay in the 126 MB L2;
//   * warp-specialised, 192 threads: warp 0 = TMA producer (one lane), warp 1 = TMEM
//     allocator + MMA issuer (one lane), warps 2..5 = epilogue (TMEM -> regs -> global);
//   * operands staged by TMA with 128-byte swizzle into a 4-6 stage smem ring
//     (mbarrier full/empty pairs); op(A)/op(B) transposes are NOT copies: the smem
//     descriptor + instruction descriptor select K-major or MN-major operands;
//   * tcgen05.mma.cta_group::1.kind::f16, M=128 x N=BN (128|256) x K=16, fp32 accumulator
//     in TMEM, double-buffered (2 x BN columns) so the epilogue of tile i overlaps the
//     mainloop of tile i+1;
//   * epilogue fuses alpha, the fp32 accumulate-in (SUMMA steps), bias and the bf16/fp32
//     conversion.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <cstring>
#include <mutex>

#include "sm100_ptx.cuh"
#include "tp_internal.h"

namespace tp {
namespace {

constexpr int BM = 128;
constexpr int BK = 64;  // one 128-byte swizzle atom of bf16 along K
constexpr int kThreads = 192;

template <int BN>
struct Cfg {
  static constexpr int kStages = (BN == 256) ? 4 : 6;
  static constexpr int kABytes = BM * BK * 2;
  static constexpr int kBBytes = BN * BK * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kTmemCols = 2 * BN;
  static constexpr int kBarBytes = 256;
  static constexpr int kOutBytes = 4 * 2 * 4096;  // epilogue staging: 4 warps x 2 x [32 rows][128 B]
  static constexpr int kSmem = kStages * kStageBytes + kOutBytes + 1024 + kBarBytes;
};

struct EpiParams {
  void* D;
  const float* C;
  const void* bias;
  int64_t ldd, ldc;
  float alpha;
  int out_bf16;
  int vec_ok;  // D, C rows 16-byte aligned
  int tma;     // D written through smem staging + TMA bulk tensor stores (tmD)
};

// ------------------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE;\n"
      "bra LAB_WAIT;\n"
      "DONE:\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_prefetch(const CUtensorMap* m) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
}

__device__ __forceinline__ void tma_load_2d(const CUtensorMap* m, uint64_t* bar, void* dst, int c0,
                                            int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

// Shared-memory matrix descriptor (tcgen05), 128-byte swizzle, version 1.
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1) << 46;  // descriptor version (sm_100)
  d |= static_cast<uint64_t>(2) << 61;  // SWIZZLE_128B
  return d;
}

// Instruction descriptor: bf16 x bf16 -> f32, dense, M x N, operand majorness.
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N, bool a_mn, bool b_mn) {
  return (1u << 4)                                   // D format f32
         | (1u << 7)                                 // A format bf16
         | (1u << 10)                                // B format bf16
         | (static_cast<uint32_t>(a_mn) << 15)       // A major (0 K, 1 MN)
         | (static_cast<uint32_t>(b_mn) << 16)       // B major
         | (static_cast<uint32_t>(N >> 3) << 17)     // N / 8
         | (static_cast<uint32_t>(M >> 4) << 24);    // M / 16
}

__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15, "
      "%16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void tile_coords(int t, int num_m, int num_n, int& mb, int& nb) {
  constexpr int G = 16;  // M-blocks per raster band
  const int band = t / (G * num_n);
  const int m_start = band * G;
  const int band_m = min(G, num_m - m_start);
  const int idx = t - band * G * num_n;
  mb = m_start + idx % band_m;
  nb = idx / band_m;
}

__device__ __forceinline__ float bias_at(const void* bias, int out_bf16_in, int64_t col) {
  // bias has the operand dtype of this kernel (bf16)
  (void)out_bf16_in;
  return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(bias)[col]);
}

// Epilogue for 32 consecutive columns of one row.
__device__ __forceinline__ void epilogue_row32(const EpiParams& ep, const uint32_t (&r)[32],
                                               int64_t row, int64_t col0, int N) {
  float v[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
  const bool full = (col0 + 32 <= N) && ep.vec_ok;
  if (full) {
    if (ep.C) {
      const float4* c4 = reinterpret_cast<const float4*>(ep.C + row * ep.ldc + col0);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        float4 c = c4[i];
        v[4 * i + 0] += c.x;
        v[4 * i + 1] += c.y;
        v[4 * i + 2] += c.z;
        v[4 * i + 3] += c.w;
      }
    }
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] *= ep.alpha;
    if (ep.bias) {
      const uint4* b4 = reinterpret_cast<const uint4*>(
          reinterpret_cast<const __nv_bfloat16*>(ep.bias) + col0);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        uint4 u = b4[i];
        const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          float2 f = __bfloat1622float2(h[j]);
          v[8 * i + 2 * j] += f.x;
          v[8 * i + 2 * j + 1] += f.y;
        }
      }
    }
    if (ep.out_bf16) {
      uint4* d4 = reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(ep.D) + row * ep.ldd + col0);
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        uint4 u;
        __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
        for (int j = 0; j < 4; ++j) h[j] = __floats2bfloat162_rn(v[8 * i + 2 * j], v[8 * i + 2 * j + 1]);
        d4[i] = u;
      }
    } else {
      float4* d4 = reinterpret_cast<float4*>(reinterpret_cast<float*>(ep.D) + row * ep.ldd + col0);
#pragma unroll
      for (int i = 0; i < 8; ++i)
        d4[i] = make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
    }
  } else {
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const int64_t col = col0 + i;
      if (col < N) {
        float x = v[i];
        if (ep.C) x += ep.C[row * ep.ldc + col];
        x *= ep.alpha;
        if (ep.bias) x += bias_at(ep.bias, 0, col);
        if (ep.out_bf16)
          reinterpret_cast<__nv_bfloat16*>(ep.D)[row * ep.ldd + col] = __float2bfloat16_rn(x);
        else
          reinterpret_cast<float*>(ep.D)[row * ep.ldd + col] = x;
      }
    }
  }
}

// alpha * (acc + C) + bias for 32 consecutive columns of one row (TMA-store epilogue).
__device__ __forceinline__ void finish32(const EpiParams& ep, float (&v)[32], int64_t row, int64_t col0,
                                         int M, int N) {
  const bool in_row = row < M;
  const bool full = (col0 + 32 <= N) && ep.vec_ok;
  if (ep.C && in_row) {
    if (full) {
      const float4* c4 = reinterpret_cast<const float4*>(ep.C + row * ep.ldc + col0);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float4 c = c4[i];
        v[4 * i] += c.x;
        v[4 * i + 1] += c.y;
        v[4 * i + 2] += c.z;
        v[4 * i + 3] += c.w;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (col0 + i < N) v[i] += ep.C[row * ep.ldc + col0 + i];
    }
  }
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] *= ep.alpha;
  if (ep.bias) {
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (col0 + i < N) v[i] += bias_at(ep.bias, 0, col0 + i);
  }
}

// ------------------------------------------------------------------------------ the kernel
template <int BN, bool A_MN, bool B_MN>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmD, const EpiParams ep, int M, int N, int K,
                   int num_m, int num_n) {
  using C = Cfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + C::kStages * C::kABytes;
  uint8_t* sOut = sB + C::kStages * C::kBBytes;  // epilogue staging
  uint64_t* full = reinterpret_cast<uint64_t*>(sOut + C::kOutBytes);
  uint64_t* empty = full + C::kStages;
  uint64_t* tfull = empty + C::kStages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  const int num_tiles = num_m * num_n;
  const int num_k = (K + BK - 1) / BK;

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    if (ep.tma) tma_prefetch(&tmD);
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tslot)),
                 "r"(C::kTmemCols)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tslot;
  // programmatic dependent launch: prologue above overlaps the previous kernel's tail
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");

  if (warp == 0) {
    {
      // ===== TMA producer: whole warp, one elected lane issues (warp-uniform values stay in
      // uniform registers; a lone thread's instruction latency would pace the pipeline) =====
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        int mb, nb;
        tile_coords(t, num_m, num_n, mb, nb);
        for (int kb = 0; kb < num_k; ++kb) {
          mbar_wait(&empty[stage], phase ^ 1);
          if (ptx::elect_one()) {
          mbar_expect_tx(&full[stage], C::kStageBytes);
          uint8_t* a_dst = sA + stage * C::kABytes;
          uint8_t* b_dst = sB + stage * C::kBBytes;
          if (!A_MN) {
            tma_load_2d(&tmA, &full[stage], a_dst, kb * BK, mb * BM);
          } else {
#pragma unroll
            for (int c = 0; c < BM / 64; ++c)
              tma_load_2d(&tmA, &full[stage], a_dst + c * (BK * 128), mb * BM + c * 64, kb * BK);
          }
          if (!B_MN) {
            tma_load_2d(&tmB, &full[stage], b_dst, kb * BK, nb * BN);
          } else {
#pragma unroll
            for (int c = 0; c < BN / 64; ++c)
              tma_load_2d(&tmB, &full[stage], b_dst + c * (BK * 128), nb * BN + c * 64, kb * BK);
          }
          }
          __syncwarp();
          if (++stage == C::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    {
      // ===== MMA issuer (whole warp, one elected lane issues) =====
      constexpr uint32_t idesc = idesc_bf16(BM, BN, A_MN, B_MN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        __syncwarp();
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * BN);
        for (int kb = 0; kb < num_k; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a_base = smem_u32(sA + stage * C::kABytes);
          const uint32_t b_base = smem_u32(sB + stage * C::kBBytes);
          if (ptx::elect_one()) {
#pragma unroll
            for (int k = 0; k < BK / 16; ++k) {
              // K-major: +32 B per 16-element K step inside the 128 B swizzle atom (SBO = 8
              // rows). MN-major: +16 rows x 128 B per K step; LBO = one 64-wide MN chunk.
              const uint64_t ad = A_MN ? sdesc(a_base + k * 2048, BK * 128, 1024)
                                       : sdesc(a_base + k * 32, 16, 1024);
              const uint64_t bd = B_MN ? sdesc(b_base + k * 2048, BK * 128, 1024)
                                       : sdesc(b_base + k * 32, 16, 1024);
              umma_bf16(d_tmem, ad, bd, idesc, (kb | k) != 0 ? 1u : 0u);
            }
            umma_commit(&empty[stage]);  // smem slot free once these MMAs retire
          }
          __syncwarp();
          if (++stage == C::kStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (ptx::elect_one()) umma_commit(&tfull[acc]);  // accumulator ready for the epilogue
        __syncwarp();
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else {
    // ===== epilogue warps 2..5: TMEM lane quadrant = warp % 4 =====
    const int quad = warp & 3;
    int nbox = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = blockIdx.x; t < num_tiles; t += gridDim.x) {
      int mb, nb;
      tile_coords(t, num_m, num_n, mb, nb);
      if (lane == 0) mbar_wait(&tfull[acc], acc_phase);  // one poller per warp
      __syncwarp();
      tc_fence_after();
      const int64_t row0 = static_cast<int64_t>(mb) * BM + quad * 32;  // warp's first row
      const int64_t row = row0 + lane;
      const uint32_t tq = tmem_base + (static_cast<uint32_t>(quad * 32) << 16) +
                          static_cast<uint32_t>(acc * BN);
      if (ep.tma) {
        // TMEM -> registers -> alpha / C / bias / cast -> 128-byte-swizzled smem box [32 rows]
        // [128 B] (explicit st.shared) -> TMA bulk tensor store; two boxes per warp in flight
        constexpr int kCols = 64;  // bf16: 64 columns per box; fp32: 32 (two boxes per step)
#pragma unroll 1
        for (int c64 = 0; c64 < BN / kCols; ++c64) {
          uint32_t r0[32], r1[32];
          tmem_ld32(tq + c64 * 64, r0);
          tmem_ld32(tq + c64 * 64 + 32, r1);
          float v0[32], v1[32];
#pragma unroll
          for (int i = 0; i < 32; ++i) {
            v0[i] = __uint_as_float(r0[i]);
            v1[i] = __uint_as_float(r1[i]);
          }
          const int64_t col0 = static_cast<int64_t>(nb) * BN + c64 * 64;
          finish32(ep, v0, row, col0, M, N);
          finish32(ep, v1, row, col0 + 32, M, N);
#pragma unroll 1
          for (int h = 0; h < (ep.out_bf16 ? 1 : 2); ++h) {
            uint8_t* buf = sOut + (warp - 2) * 2 * 4096 + (nbox & 1) * 4096;
            if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
            __syncwarp();
            const uint32_t rowp = smem_u32(buf) + lane * 128;
            if (ep.out_bf16) {
#pragma unroll
              for (int j = 0; j < 8; ++j) {
                const float* src = j < 4 ? v0 + 8 * j : v1 + 8 * (j - 4);
                uint32_t u[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                  __nv_bfloat162 b2 = __floats2bfloat162_rn(src[2 * k], src[2 * k + 1]);
                  u[k] = *reinterpret_cast<uint32_t*>(&b2);
                }
                ptx::sts128(rowp + ((j ^ (lane & 7)) << 4), u[0], u[1], u[2], u[3]);
              }
            } else {
              const float* src = h == 0 ? v0 : v1;
#pragma unroll
              for (int j = 0; j < 8; ++j)
                ptx::sts128(rowp + ((j ^ (lane & 7)) << 4), __float_as_uint(src[4 * j]),
                            __float_as_uint(src[4 * j + 1]), __float_as_uint(src[4 * j + 2]),
                            __float_as_uint(src[4 * j + 3]));
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) {
              ptx::tma_store_2d(&tmD, buf, static_cast<int>(col0 + h * 32), static_cast<int>(row0));
              asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
            ++nbox;
          }
        }
      } else {
#pragma unroll 1
        for (int ch = 0; ch < BN / 32; ++ch) {
          uint32_t r[32];
          tmem_ld32(tq + ch * 32, r);
          const int64_t col0 = static_cast<int64_t>(nb) * BN + ch * 32;
          if (row < M && col0 < N) epilogue_row32(ep, r, row, col0, N);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
    // the staging boxes must outlive the bulk stores' shared-memory reads
    if (ep.tma && lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(C::kTmemCols)
                 : "memory");
  }
}

// ------------------------------------------------------------------------------ host side
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// 2-D bf16 tensor map: `inner` contiguous elements per row, `outer` rows, row stride ld.
tp_status make_map(CUtensorMap* m, const void* base, uint64_t inner, uint64_t outer, uint64_t ld,
                   uint32_t box_inner, uint32_t box_outer, bool fp32 = false) {
  auto fn = encode_fn();
  if (!fn) return fail(TP_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld * (fp32 ? 4 : 2)};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, fp32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                  const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(TP_ERR_SHAPE, "cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) +
                                  "): inner=" + std::to_string(inner) + " outer=" +
                                  std::to_string(outer) + " ld=" + std::to_string(ld));
  return TP_OK;
}

int num_sms(int dev) {
  static int cache[64] = {0};
  if (dev < 0 || dev >= 64) return 148;
  if (!cache[dev]) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = n > 0 ? n : 148;
  }
  return cache[dev];
}

template <int BN, bool A_MN, bool B_MN>
tp_status launch(const GemmArgs& g, cudaStream_t s) {
  using C = Cfg<BN>;
  CUtensorMap ta, tb;
  // A: K-major -> rows of K contiguous (box 64 x 128); MN-major -> stored [K,M] (box 64 x 64)
  if (!A_MN)
    TP_TRY(make_map(&ta, g.A, g.K, g.M, g.lda, BK, BM));
  else
    TP_TRY(make_map(&ta, g.A, g.M, g.K, g.lda, 64, BK));
  if (!B_MN)
    TP_TRY(make_map(&tb, g.B, g.K, g.N, g.ldb, BK, BN));
  else
    TP_TRY(make_map(&tb, g.B, g.N, g.K, g.ldb, 64, BK));

  int dev = 0;
  TP_CUDA(cudaGetDevice(&dev));
  auto kern = gemm_tc_kernel<BN, A_MN, B_MN>;
  TP_CUDA(set_smem_attr(reinterpret_cast<const void*>(kern), C::kSmem));
  const int num_m = static_cast<int>((g.M + BM - 1) / BM);
  const int num_n = static_cast<int>((g.N + BN - 1) / BN);
  const int tiles = num_m * num_n;
  int cap = num_sms(dev);
  if (g.reserve_sms > 0) cap = std::max(1, cap - g.reserve_sms);  // room for concurrent NCCL
  const int grid = tiles < cap ? tiles : cap;
  EpiParams ep;
  ep.D = g.D;
  ep.C = g.C;
  ep.bias = g.bias;
  ep.ldd = g.ldd;
  ep.ldc = g.ldc;
  ep.alpha = g.alpha;
  ep.out_bf16 = g.out_dtype == TP_BF16;
  const size_t osz = dtype_size(g.out_dtype);
  ep.vec_ok = ((reinterpret_cast<uintptr_t>(g.D) % 16) == 0) && ((g.ldd * osz) % 16 == 0) &&
              (!g.C || (((reinterpret_cast<uintptr_t>(g.C) % 16) == 0) && ((g.ldc * 4) % 16 == 0))) &&
              (!g.bias || (reinterpret_cast<uintptr_t>(g.bias) % 16) == 0);
  // D through TMA stores when its rows are 16-byte aligned (bf16 box 64 x 32, fp32 32 x 32)
  CUtensorMap td;
  std::memset(&td, 0, sizeof(td));
  const int env_tma = knob("TP_GEMM_V1_TMA_STORE");
  // A TMA store writes whole 16-byte granules of the inner dimension: when a row of D does not
  // end on a granule (N * osz % 16 != 0) it would also write zeros to the columns between N and
  // the next granule - elements outside D (measured: tools/gemm_probe_ragged.py). Those
  // problems take the guarded per-element epilogue instead.
  ep.tma = env_tma && (reinterpret_cast<uintptr_t>(g.D) % 16) == 0 && (g.ldd * osz) % 16 == 0 &&
           (g.N * osz) % 16 == 0;
  if (ep.tma)
    TP_TRY(make_map(&td, g.D, g.N, g.M, g.ldd, ep.out_bf16 ? 64 : 32, 32, !ep.out_bf16));
  const int tok = prof_begin(0, s, 2.0 * double(g.M) * double(g.N) * double(g.K));
  TP_CUDA(launch_pdl(kern, dim3(grid), dim3(kThreads), C::kSmem, s, ta, tb, td, ep,
                     static_cast<int>(g.M), static_cast<int>(g.N), static_cast<int>(g.K), num_m,
                     num_n));
  count_launch();
  prof_end(tok, s);
  TP_CUDA(cudaGetLastError());
  return TP_OK;
}

}  // namespace

tp_status gemm_tc_bf16(const GemmArgs& g, cudaStream_t s) {
  const bool a_mn = g.trans_a;   // A stored [K,M]: M contiguous
  const bool b_mn = !g.trans_b;  // B stored [K,N]: N contiguous
  // BN = 256 when there are enough 128x256 tiles to fill the machine, else 128.
  int dev = 0;
  TP_CUDA(cudaGetDevice(&dev));
  const int64_t tiles256 = ((g.M + BM - 1) / BM) * ((g.N + 255) / 256);
  const int force_bn = knob("TP_GEMM_V1_BN");
  // measured (profiles/r01_gemm_v2_summary.md): 128x256 tiles win once ~120+ of them exist
  const bool wide = force_bn ? force_bn == 256 : tiles256 >= (num_sms(dev) * 13) / 16;
  if (wide) {
    if (!a_mn && !b_mn) return launch<256, false, false>(g, s);
    if (!a_mn && b_mn) return launch<256, false, true>(g, s);
    if (a_mn && !b_mn) return launch<256, true, false>(g, s);
    return launch<256, true, true>(g, s);
  }
  if (!a_mn && !b_mn) return launch<128, false, false>(g, s);
  if (!a_mn && b_mn) return launch<128, false, true>(g, s);
  if (a_mn && !b_mn) return launch<128, true, false>(g, s);
  return launch<128, true, true>(g, s);
}

}  // namespace tp
