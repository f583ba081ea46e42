// Fused attention backward for sm_100a (the attention core of the block
// "with scores kept out of HBM"). For one problem (batch x head) with P = softmax(Q K^T scale):
//   dV = P^T dO,  dP = dO V^T,  dS = P (dP - Delta) scale,  Delta = rowsum(dO o O),
//   dQ = dS K,    dK = dS^T Q                                  (reading N4: the chain rule)
// with P recomputed from the forward's per-row log-sum-exp: P = exp2(S scale log2e - lse).
//
// One CTA per (problem, 128-key tile j), looping over the 128-query tiles i; 320 threads:
//   warp 0    TMA: K_j, V_j once; Q_i, dO_i per tile (NS-stage ring)
//   warp 1    tcgen05 MMA issuer (cta_group::1), all products 128 x 128 / 128 x d tiles:
//             S^T = K_j Q_i^T, dP^T = V_j dO_i^T (TMEM), dV += P^T dO_i, dK += dS^T Q_i (TMEM,
//             resident for the CTA), dQ_i = dS K_j (TMEM)
//   warps 2-5 one key row each (TMEM lane): P^T row = exp2(S^T row * c - lse) -> bf16 smem,
//             dS^T row = P (dP^T row - Delta) scale -> bf16 smem; at the end dK, dV -> HBM
//   warps 6-9 one query row each: dQ_i rows from TMEM added into the fp32 dQ accumulator in
//             HBM (red.global.add.v4.f32: the key tiles of a query row meet there)
// Every smem tile is stored once, K-major ([64-column chunk][128 rows][128 B], 128-byte
// swizzle) and read by the MMAs in whichever majorness the product needs (an MN-major operand
// over the same tile: LBO = 16 KB between 64-wide chunks, 2048 B per 16-row K step).
// TMEM: dV [0, d), dK [d, 2d), S^T [2d, +128), dP^T [2d+128, +128), dQ: [2d+256, +d) for
// d = 64; for d = 128 it reuses S^T's columns (free once the key rows have their P).
// Keys / queries past the sequence end: their P is 0 (lse = +inf), their rows are not stored.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include <cmath>
#include <mutex>

#include "sched.h"
#include "sm100_ptx.cuh"
#include "tp_internal.h"

namespace tp {
namespace {

using namespace ptx;

constexpr int kT = 128;           // keys per CTA, queries per tile
constexpr int kTileB = kT * 128;  // one [128 rows][128 B] chunk

template <int D>
struct BC {
  static constexpr int NS = 2;                         // Q / dO ring stages
  static constexpr int Chunk = D / 64;                 // 64-wide column chunks of a [128 x D] tile
  static constexpr int TileBytes = kT * D * 2;         // K, V, Q, dO tiles
  static constexpr int PBytes = kT * kT * 2;           // P^T, dS^T tiles (two 64-query chunks)
  // d = 128: P^T and dS^T share one smem tile (dS^T overwrites P^T once the dV MMA read it)
  static constexpr bool SharePdS = D != 64;
  static constexpr int Smem = 2 * TileBytes + NS * 2 * TileBytes + (SharePdS ? 1 : 2) * PBytes +
                              2 * kT * 4 + 1024 + 256;  // d = 128: 231,680 B of the 232,448
  static constexpr uint32_t TDV = 0, TDK = D, TS = 2 * D, TDP = 2 * D + 128;
  // d = 128: TMEM is full, dQ_i reuses dP^T's columns (free once the key rows formed dS_i)
  static constexpr uint32_t TDQ = D == 64 ? 2 * D + 256 : TDP;
  static constexpr bool Alias = D != 64;
};

struct BParams {
  CUtensorMap tmQ, tmK, tmV, tmdO;
  const float* lse;    // [problems*s] scaled log2 units
  const float* delta;  // [problems*s]
  float* dq_acc;       // [problems*s, D] fp32 (zeroed)
  __nv_bfloat16 *dk, *dv;
  float *dk32, *dv32;  // non-null: dK / dV written in fp32 here instead (ring partials)
  int no_dq;           // diagnostics (knob TP_FB_NODQ): skip the dQ accumulation
  int64_t s;
  float scale, scale_log2;
};

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ void red_add_v4(float* p, float a, float b, float c, float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(a), "f"(b), "f"(c),
               "f"(d)
               : "memory");
}

// write 32 bf16 values (16 packed words) of row r, columns [c0, c0+32), into a K-major tile
// [col/64 chunk][128 rows][128 B] with the 128-byte swizzle
__device__ __forceinline__ void sts_row32(uint8_t* tile, int r, int c0, const uint32_t (&pk)[16]) {
  const uint32_t rowp = smem_u32(tile) + (c0 / 64) * kTileB + r * 128;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int chunk = ((c0 % 64) / 32) * 4 + q;
    sts128(rowp + ((chunk ^ (r & 7)) << 4), pk[4 * q], pk[4 * q + 1], pk[4 * q + 2], pk[4 * q + 3]);
  }
}

template <int D>
__global__ void __launch_bounds__(320, 1) flash_bwd_kernel(const __grid_constant__ BParams F) {
  using C = BC<D>;
  constexpr int NS = C::NS;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sK = smem;
  uint8_t* sV = sK + C::TileBytes;
  uint8_t* sQ = sV + C::TileBytes;              // [NS]
  uint8_t* sdO = sQ + NS * C::TileBytes;        // [NS]
  uint8_t* sP = sdO + NS * C::TileBytes;
  uint8_t* sdS = C::SharePdS ? sP : sP + C::PBytes;
  float* sLD = reinterpret_cast<float*>(sdS + C::PBytes);  // [lse 128 | delta 128] of the tile
  uint64_t* bars = reinterpret_cast<uint64_t*>(sLD + 2 * kT);
  uint64_t* kv_full = bars;
  uint64_t* q_full = kv_full + 1;     // [NS]
  uint64_t* q_empty = q_full + NS;    // [NS]
  uint64_t* s_full = q_empty + NS;
  uint64_t* s_free = s_full + 1;
  uint64_t* dp_full = s_free + 1;
  uint64_t* dp_free = dp_full + 1;
  uint64_t* p_full = dp_free + 1;
  uint64_t* p_free = p_full + 1;
  uint64_t* ds_full = p_free + 1;
  uint64_t* ds_free = ds_full + 1;
  uint64_t* dq_full = ds_free + 1;
  uint64_t* dq_free = dq_full + 1;
  uint64_t* kv_done = dq_free + 1;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(kv_done + 1);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int64_t prob = blockIdx.y;
  const int64_t key0 = int64_t(blockIdx.x) * kT;
  const int64_t row_base = prob * F.s;
  const int nq = static_cast<int>((F.s + kT - 1) / kT);

  if (threadIdx.x == 0) {
    tma_prefetch(&F.tmQ);
    tma_prefetch(&F.tmK);
    tma_prefetch(&F.tmV);
    tma_prefetch(&F.tmdO);
    mbar_init(kv_full, 1);
    for (int i = 0; i < NS; ++i) {
      mbar_init(&q_full[i], 1);
      mbar_init(&q_empty[i], 1);
    }
    mbar_init(s_full, 1);
    mbar_init(s_free, 4);
    mbar_init(dp_full, 1);
    mbar_init(dp_free, 4);
    mbar_init(p_full, 4);
    mbar_init(p_free, 1);
    mbar_init(ds_full, 4);
    mbar_init(ds_free, 1);
    mbar_init(dq_full, 1);
    mbar_init(dq_free, 4);
    mbar_init(kv_done, 1);
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_cg1(tslot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;

  if (warp == 0) {
    if (elect_one()) {
      // ---- TMA producer
      mbar_expect_tx(kv_full, 2 * C::TileBytes);
      for (int c = 0; c < C::Chunk; ++c) {
        tma_load_2d(&F.tmK, kv_full, sK + c * kTileB, c * 64, static_cast<int>(row_base + key0));
        tma_load_2d(&F.tmV, kv_full, sV + c * kTileB, c * 64, static_cast<int>(row_base + key0));
      }
      for (int i = 0; i < nq; ++i) {
        const int st = i % NS;
        mbar_wait(&q_empty[st], ((i / NS) & 1) ^ 1);
        mbar_expect_tx(&q_full[st], 2 * C::TileBytes);
        const int r0 = static_cast<int>(row_base + int64_t(i) * kT);
        for (int c = 0; c < C::Chunk; ++c) {
          tma_load_2d(&F.tmQ, &q_full[st], sQ + st * C::TileBytes + c * kTileB, c * 64, r0);
          tma_load_2d(&F.tmdO, &q_full[st], sdO + st * C::TileBytes + c * kTileB, c * 64, r0);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (elect_one()) {
      // ---- MMA issuer
      constexpr uint32_t idSS = idesc_bf16_f32(128, kT, false, false);   // S^T, dP^T
      constexpr uint32_t idKV = idesc_bf16_f32(128, D, false, true);     // dV, dK
      constexpr uint32_t idQ = idesc_bf16_f32(128, D, true, true);       // dQ
      const uint64_t kd = sdesc_sw128(smem_u32(sK), 16, 1024);
      const uint64_t vd = sdesc_sw128(smem_u32(sV), 16, 1024);
      const uint64_t pd = sdesc_sw128(smem_u32(sP), 16, 1024);
      const uint64_t dsd = sdesc_sw128(smem_u32(sdS), 16, 1024);
      const uint64_t dsd_mn = sdesc_sw128(smem_u32(sdS), kTileB, 1024);  // dS (M = queries) MN-major
      const uint64_t kd_mn = sdesc_sw128(smem_u32(sK), kTileB, 1024);    // K_j as MN-major B
      mbar_wait(kv_full, 0);
      for (int i = 0; i < nq; ++i) {
        const int st = i % NS;
        const uint32_t ph = i & 1, php = (i - 1) & 1;
        mbar_wait(&q_full[st], (i / NS) & 1);
        const uint64_t qd = sdesc_sw128(smem_u32(sQ + st * C::TileBytes), 16, 1024);
        const uint64_t qd_mn = sdesc_sw128(smem_u32(sQ + st * C::TileBytes), kTileB, 1024);
        const uint64_t od = sdesc_sw128(smem_u32(sdO + st * C::TileBytes), 16, 1024);
        const uint64_t od_mn = sdesc_sw128(smem_u32(sdO + st * C::TileBytes), kTileB, 1024);
        // S^T = K_j Q_i^T   (the key rows took tile i-1's scores)
        if (i > 0) mbar_wait(s_free, php);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint32_t off = (k / 4) * (kTileB / 16) + (k % 4) * 2;
          umma_bf16_cg1(tmem + C::TS, kd + off, qd + off, idSS, k > 0 ? 1u : 0u);
        }
        umma_commit_cg1(s_full);
        // dP^T = V_j dO_i^T   (d = 128: dQ_{i-1}, in the same columns, drained)
        if (i > 0) {
          mbar_wait(dp_free, php);
          if (C::Alias) mbar_wait(dq_free, php);
        }
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < D / 16; ++k) {
          const uint32_t off = (k / 4) * (kTileB / 16) + (k % 4) * 2;
          umma_bf16_cg1(tmem + C::TDP, vd + off, od + off, idSS, k > 0 ? 1u : 0u);
        }
        umma_commit_cg1(dp_full);
        // dV += P^T dO_i   (K = queries: P^T K-major, dO_i MN-major)
        mbar_wait(p_full, ph);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < kT / 16; ++k) {
          const uint32_t offa = (k / 4) * (kTileB / 16) + (k % 4) * 2;
          umma_bf16_cg1(tmem + C::TDV, pd + offa, od_mn + k * (2048 / 16), idKV, (i > 0 || k > 0) ? 1u : 0u);
        }
        umma_commit_cg1(p_free);
        // dQ_i = dS K_j first (its drain then overlaps the dK MMA), then dK += dS^T Q_i
        mbar_wait(ds_full, ph);
        if (!C::Alias && i > 0) mbar_wait(dq_free, php);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < kT / 16; ++k)
          umma_bf16_cg1(tmem + C::TDQ, dsd_mn + k * (2048 / 16), kd_mn + k * (2048 / 16), idQ, k > 0 ? 1u : 0u);
        umma_commit_cg1(dq_full);
#pragma unroll
        for (int k = 0; k < kT / 16; ++k) {
          const uint32_t offa = (k / 4) * (kTileB / 16) + (k % 4) * 2;
          umma_bf16_cg1(tmem + C::TDK, dsd + offa, qd_mn + k * (2048 / 16), idKV, (i > 0 || k > 0) ? 1u : 0u);
        }
        umma_commit_cg1(ds_free);
        umma_commit_cg1(&q_empty[st]);
      }
      umma_commit_cg1(kv_done);
    }
    __syncwarp();
  } else if (warp < 6) {
    // ---- key-row warps: thread = key row r of the tile (TMEM lane quadrant warp % 4)
    const int quad = warp & 3;
    const int r = quad * 32 + lane;
    const int t = (warp - 2) * 32 + lane;  // 0..127: this thread's query slot for lse / delta
    const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
    const bool key_ok = key0 + r < F.s;
    // this thread's lse / delta slot of the next query tile, loaded one tile ahead
    float nl = t < F.s ? F.lse[row_base + t] : INFINITY;
    float nd = t < F.s ? F.delta[row_base + t] : 0.f;
    for (int i = 0; i < nq; ++i) {
      const uint32_t ph = i & 1, php = (i - 1) & 1;
      float* L = sLD;
      if (i > 0) named_barrier_sync(1, 128);  // every key row is done with tile i-1's values
      L[t] = nl;
      L[kT + t] = nd;
      named_barrier_sync(1, 128);
      {
        const int64_t q = int64_t(i + 1) * kT + t;
        nl = q < F.s ? F.lse[row_base + q] : INFINITY;
        nd = q < F.s ? F.delta[row_base + q] : 0.f;
      }
      // P^T row = exp2(S^T row c - lse[q])
      mbar_wait(s_full, ph);
      tc_fence_after();
      uint32_t pk[kT / 2];
#pragma unroll
      for (int c = 0; c < kT / 32; ++c) {
        uint32_t sv[32];
        tmem_ld32(tmem + C::TS + lane_off + c * 32, sv);
        tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int q = c * 32 + 2 * j;
          float p0 = ex2(fmaf(__uint_as_float(sv[2 * j]), F.scale_log2, -L[q]));
          float p1 = ex2(fmaf(__uint_as_float(sv[2 * j + 1]), F.scale_log2, -L[q + 1]));
          if (!key_ok) p0 = p1 = 0.f;
          __nv_bfloat162 h = __floats2bfloat162_rn(p0, p1);
          pk[c * 16 + j] = *reinterpret_cast<uint32_t*>(&h);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(s_free);
      // the P^T tile is free: the dV MMA of tile i-1 read it (and, shared with dS^T, the dQ / dK
      // MMAs of tile i-1 read dS^T)
      if (i > 0) mbar_wait(C::SharePdS ? ds_free : p_free, php);
#pragma unroll
      for (int c = 0; c < kT / 32; ++c) {
        uint32_t w[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) w[j] = pk[c * 16 + j];
        sts_row32(sP, r, c * 32, w);
      }
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(p_full);
      // dS^T row = P (dP^T row - delta[q]) scale
      mbar_wait(dp_full, ph);
      tc_fence_after();
      // the dS^T tile is free: shared with P^T, once the dV MMA of THIS tile read P^T; else once
      // the dQ / dK MMAs of tile i-1 read dS^T
      if (C::SharePdS) mbar_wait(p_free, ph);
      else if (i > 0) mbar_wait(ds_free, php);
#pragma unroll
      for (int c = 0; c < kT / 32; ++c) {
        uint32_t dv[32];
        tmem_ld32(tmem + C::TDP + lane_off + c * 32, dv);
        tmem_wait_ld();
        uint32_t w[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int q = c * 32 + 2 * j;
          const float2 p = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&pk[c * 16 + j]));
          const float d0 = p.x * (__uint_as_float(dv[2 * j]) - L[kT + q]) * F.scale;
          const float d1 = p.y * (__uint_as_float(dv[2 * j + 1]) - L[kT + q + 1]) * F.scale;
          __nv_bfloat162 h = __floats2bfloat162_rn(d0, d1);
          w[j] = *reinterpret_cast<uint32_t*>(&h);
        }
        sts_row32(sdS, r, c * 32, w);
      }
      tc_fence_before();
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(dp_free);
        mbar_arrive(ds_full);
      }
    }
    // ---- dK, dV rows -> HBM (bf16)
    mbar_wait(kv_done, 0);
    tc_fence_after();
#pragma unroll 1
    for (int which = 0; which < 2; ++which) {
      __nv_bfloat16* dst = (which == 0 ? F.dv : F.dk) + (row_base + key0 + r) * D;
      float* dst32 = F.dk32 ? (which == 0 ? F.dv32 : F.dk32) + (row_base + key0 + r) * D : nullptr;
      const uint32_t col0 = which == 0 ? C::TDV : C::TDK;
#pragma unroll 1
      for (int c = 0; c < D / 32; ++c) {
        uint32_t v[32];
        tmem_ld32(tmem + col0 + lane_off + c * 32, v);
        tmem_wait_ld();
        if (key_ok && dst32) {
#pragma unroll
          for (int k = 0; k < 32; k += 4)
            *reinterpret_cast<float4*>(dst32 + c * 32 + k) =
                make_float4(__uint_as_float(v[k]), __uint_as_float(v[k + 1]), __uint_as_float(v[k + 2]),
                            __uint_as_float(v[k + 3]));
        } else if (key_ok) {
#pragma unroll
          for (int k = 0; k < 32; k += 8) {
            uint4 u;
            __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
            for (int e = 0; e < 4; ++e)
              h[e] = __floats2bfloat162_rn(__uint_as_float(v[k + 2 * e]), __uint_as_float(v[k + 2 * e + 1]));
            *reinterpret_cast<uint4*>(dst + c * 32 + k) = u;
          }
        }
      }
    }
  } else {
    // ---- dQ warps: thread = query row of tile i (lane quadrant warp % 4)
    const int quad = warp & 3;
    const int r = quad * 32 + lane;
    const uint32_t lane_off = static_cast<uint32_t>(quad * 32) << 16;
    for (int i = 0; i < nq; ++i) {
      if (lane == 0) mbar_wait_sleep(dq_full, i & 1, 64);
      __syncwarp();
      tc_fence_after();
      const int64_t q = int64_t(i) * kT + r;
      float* dst = F.dq_acc + (row_base + q) * D;
#pragma unroll 1
      for (int c = 0; c < D / 32; ++c) {
        uint32_t v[32];
        tmem_ld32(tmem + C::TDQ + lane_off + c * 32, v);
        tmem_wait_ld();
        if (q < F.s && !F.no_dq) {
#pragma unroll
          for (int k = 0; k < 32; k += 4)
            red_add_v4(dst + c * 32 + k, __uint_as_float(v[k]), __uint_as_float(v[k + 1]),
                       __uint_as_float(v[k + 2]), __uint_as_float(v[k + 3]));
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(dq_free);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_cg1(tmem, 512);
  }
}

// Delta[row] = sum_c dO[row, c] O[row, c] (fp32), one warp per row.
__global__ void flash_bwd_delta(const __nv_bfloat16* __restrict__ o, const __nv_bfloat16* __restrict__ dout,
                                int64_t rows, int d, float* __restrict__ delta) {
  const int64_t row = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x % 32;
  if (row >= rows) return;
  float acc = 0.f;
  for (int c = lane * 8; c < d; c += 32 * 8) {
    const uint4 a = *reinterpret_cast<const uint4*>(o + row * d + c);
    const uint4 b = *reinterpret_cast<const uint4*>(dout + row * d + c);
    const __nv_bfloat162* ha = reinterpret_cast<const __nv_bfloat162*>(&a);
    const __nv_bfloat162* hb = reinterpret_cast<const __nv_bfloat162*>(&b);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 x = __bfloat1622float2(ha[e]), y = __bfloat1622float2(hb[e]);
      acc = fmaf(x.x, y.x, fmaf(x.y, y.y, acc));
    }
  }
#pragma unroll
  for (int o2 = 16; o2 > 0; o2 >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o2);
  if (lane == 0) delta[row] = acc;
}

__global__ void flash_bwd_cast(const float* __restrict__ src, int64_t n, __nv_bfloat16* __restrict__ dst) {
  const int64_t i = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) * 4;
  if (i + 3 < n) {
    const float4 v = *reinterpret_cast<const float4*>(src + i);
    __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
    uint2 u;
    u.x = *reinterpret_cast<uint32_t*>(&a);
    u.y = *reinterpret_cast<uint32_t*>(&b);
    *reinterpret_cast<uint2*>(dst + i) = u;
  } else {
    for (int64_t k = i; k < n; ++k) dst[k] = __float2bfloat16_rn(src[k]);
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_b() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

tp_status map_b(CUtensorMap* m, const void* base, uint64_t rows, int D) {
  auto fn = encode_b();
  if (!fn) return fail(TP_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {static_cast<cuuint64_t>(D), rows};
  cuuint64_t strides[1] = {static_cast<cuuint64_t>(D) * 2};
  cuuint32_t box[2] = {64, kT};
  cuuint32_t es[2] = {1, 1};
  if (fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
         CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
         CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return fail(TP_ERR_SHAPE, "flash bwd: tensor map encode failed");
  return TP_OK;
}

template <int D>
tp_status launch_bwd(const BParams& F, int64_t problems, cudaStream_t s) {
  using C = BC<D>;
  auto k = flash_bwd_kernel<D>;
  TP_CUDA(set_smem_attr(reinterpret_cast<const void*>(k), C::Smem));
  dim3 grid(static_cast<unsigned>((F.s + kT - 1) / kT), static_cast<unsigned>(problems));
  k<<<grid, 320, C::Smem, s>>>(F);
  count_launch();
  TP_CUDA(cudaGetLastError());
  return TP_OK;
}

}  // namespace

tp_status flash_bwd_delta_launch(int64_t rows, int64_t d, const void* o, const void* dout,
                                 float* delta, cudaStream_t st) {
  if (!rows) return TP_OK;
  const unsigned G = static_cast<unsigned>((rows * 32 + 255) / 256);
  flash_bwd_delta<<<G, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(o),
                                      static_cast<const __nv_bfloat16*>(dout), rows, static_cast<int>(d), delta);
  count_launch();
  TP_CUDA(cudaGetLastError());
  return TP_OK;
}

tp_status flash_bwd_cast_launch(const float* src, int64_t n, void* dst, cudaStream_t st) {
  if (!n) return TP_OK;
  const unsigned G = static_cast<unsigned>((n / 4 + 255) / 256 + 1);
  flash_bwd_cast<<<G, 256, 0, st>>>(src, n, static_cast<__nv_bfloat16*>(dst));
  count_launch();
  TP_CUDA(cudaGetLastError());
  return TP_OK;
}

// One ring step of the fused backward: local queries q / dout / lse / delta against the visiting
// key block k / v; dQ added into dq_acc (fp32, not zeroed here), dK / dV of the visiting block
// written in fp32 to dk32 / dv32.
tp_status flash_bwd_step(int64_t problems, int64_t s, int64_t d, const void* q, const void* k,
                         const void* v, const void* dout, const float* lse, const float* delta,
                         float* dq_acc, float* dk32, float* dv32, float scale, cudaStream_t st) {
  if (!problems || !s) return TP_OK;
  if (d != 64 && d != 128) return fail(TP_ERR_UNSUPPORTED, "flash bwd: d must be 64 or 128");
  if (problems > 65535) return fail(TP_ERR_UNSUPPORTED, "flash bwd: too many problems for one grid");
  const int64_t rows = problems * s;
  BParams F{};
  TP_TRY(map_b(&F.tmQ, q, uint64_t(rows), static_cast<int>(d)));
  TP_TRY(map_b(&F.tmK, k, uint64_t(rows), static_cast<int>(d)));
  TP_TRY(map_b(&F.tmV, v, uint64_t(rows), static_cast<int>(d)));
  TP_TRY(map_b(&F.tmdO, dout, uint64_t(rows), static_cast<int>(d)));
  F.lse = lse;
  F.delta = delta;
  F.dq_acc = dq_acc;
  F.dk32 = dk32;
  F.dv32 = dv32;
  F.s = s;
  F.scale = scale;
  F.scale_log2 = scale * 1.4426950408889634f;
  return d == 64 ? launch_bwd<64>(F, problems, st) : launch_bwd<128>(F, problems, st);
}

size_t flash_bwd_ws_bytes(int64_t problems, int64_t s, int64_t d) {
  const size_t rows = size_t(problems) * size_t(s);
  return ((rows * size_t(d) * 4 + 255) & ~size_t(255)) + ((rows * 4 + 255) & ~size_t(255));
}

tp_status flash_attn_bwd(int64_t problems, int64_t s, int64_t d, const void* q, const void* k,
                         const void* v, const void* o, const void* dout, const float* lse,
                         void* dq, void* dk, void* dv, float scale, void* ws, cudaStream_t st) {
  if (!problems || !s) return TP_OK;
  if (d != 64 && d != 128) return fail(TP_ERR_UNSUPPORTED, "flash bwd: d must be 64 or 128");
  if (problems > 65535) return fail(TP_ERR_UNSUPPORTED, "flash bwd: too many problems for one grid");
  const int64_t rows = problems * s;
  float* dq_acc = static_cast<float*>(ws);
  float* delta = reinterpret_cast<float*>(static_cast<char*>(ws) + ((size_t(rows) * d * 4 + 255) & ~size_t(255)));
  TP_CUDA(cudaMemsetAsync(dq_acc, 0, size_t(rows) * d * 4, st));
  {
    const unsigned G = static_cast<unsigned>((rows * 32 + 255) / 256);
    flash_bwd_delta<<<G, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(o),
                                        static_cast<const __nv_bfloat16*>(dout), rows, static_cast<int>(d), delta);
    count_launch();
    TP_CUDA(cudaGetLastError());
  }
  BParams F{};
  TP_TRY(map_b(&F.tmQ, q, uint64_t(rows), static_cast<int>(d)));
  TP_TRY(map_b(&F.tmK, k, uint64_t(rows), static_cast<int>(d)));
  TP_TRY(map_b(&F.tmV, v, uint64_t(rows), static_cast<int>(d)));
  TP_TRY(map_b(&F.tmdO, dout, uint64_t(rows), static_cast<int>(d)));
  F.lse = lse;
  F.delta = delta;
  F.dq_acc = dq_acc;
  F.dk = static_cast<__nv_bfloat16*>(dk);
  F.dv = static_cast<__nv_bfloat16*>(dv);
  F.s = s;
  F.scale = scale;
  F.scale_log2 = scale * 1.4426950408889634f;
  F.no_dq = knob("TP_FB_NODQ");
  TP_TRY(d == 64 ? launch_bwd<64>(F, problems, st) : launch_bwd<128>(F, problems, st));
  const int64_t n = rows * d;
  const unsigned G = static_cast<unsigned>((n / 4 + 255) / 256 + 1);
  flash_bwd_cast<<<G, 256, 0, st>>>(dq_acc, n, static_cast<__nv_bfloat16*>(dq));
  count_launch();
  TP_CUDA(cudaGetLastError());
  return TP_OK;
}

}  // namespace tp
