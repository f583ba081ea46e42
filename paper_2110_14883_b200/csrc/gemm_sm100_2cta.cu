// CTA-pair (tcgen05 cta_group::2) bf16 GEMM for sm_100a — the main local-GEMM kernel of every
// TP mode:   D[M,N] = alpha * (op(A).op(B) + C) + bias[col].
//
// Why a pair (profiles/r01_gemm_v1_summary.md): on one SM, shared memory feeds both the TMA
// writes and the UMMA operand reads. A 1-CTA 128x128 K=16 step moves 8 KB in + 8 KB out per 64
// MMA cycles (2x the ~128 B/clk port) and measured 47% tensor-pipe activity. A CTA pair
// computes a 256x256 tile: each CTA stages its own 128 rows of A and 128 of the 256 columns of
// B, the leader issues M=256 N=256 MMAs that read both CTAs' smem, each CTA keeps its 128
// accumulator rows (256 fp32 columns) in its own TMEM. Per CTA: 8 KB read + 8 KB written per
// 128 MMA cycles = the port's rate.
//
//   * cluster (2,1,1); persistent over pair-tiles (grouped raster), 192 threads per CTA:
//     warp 0 TMA producer (both CTAs; bytes signalled on the leader's `full` barrier),
//     warp 1 TMEM allocator (both) + MMA issuer (leader), warps 2..5 epilogue (both);
//   * 6-stage smem ring (32 KB/stage/CTA), BK = 64 with 128-byte swizzle; K-major or MN-major
//     operands by descriptor (no transposes); TMEM accumulator double-buffered (2 x 256 cols);
//   * split-K for grids with fewer pair-tiles than SM pairs (e.g. M = 512): every split writes
//     an fp32 partial tile, the last split to arrive (per-tile counter) sums the partials in
//     split order (deterministic) and runs the epilogue;
//   * epilogue: TMEM -> registers -> alpha / C / bias / cast -> 128-byte-swizzled smem staging
//     -> TMA bulk tensor store (full-line writes, asynchronous).
#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <mutex>

#include "sm100_ptx.cuh"
#include "tp_internal.h"

namespace tp {
unsigned long long* g_gemm_trace = nullptr;  // set by tp_gemm_trace (tools only)
namespace {

using namespace ptx;

constexpr int kBM = 128;  // A rows per CTA (pair tile: 256 rows)
constexpr int kBK = 64;
constexpr int kABytes = kBM * kBK * 2;
constexpr int kOutBytes = 32 * 128;  // per epilogue warp: 32 rows x 128 B staging
constexpr int kThreads = 192;

// Pair-tile width BNP (256 or 128): B columns per CTA, ring depth, TMEM, smem.
template <int BNP>
struct PC {
  static constexpr int BNC = BNP / 2;
  static constexpr int Stages = BNP == 256 ? 6 : 8;
  static constexpr int BBytes = BNC * kBK * 2;
  static constexpr int StageBytes = kABytes + BBytes;
  static constexpr int TmemCols = 2 * BNP;
  static constexpr int Smem = Stages * StageBytes + 8 * kOutBytes + 1024 + 256;
  static constexpr int TileElems = 256 * BNP;
};

struct Epi2 {
  const float* C;
  const void* bias;
  float* part;
  int* counters;
  int64_t ldc;
  float alpha;
  int out_bf16;
  int M, N;
  int splits, kb_per_split;
  int c_vec;     // C rows 16-byte aligned
  int prefetch;  // L2 prefetch distance in k-blocks (0 = off)
  unsigned long long* trace;  // optional per-CTA wait-cycle counters (TP_GEMM_TRACE)
};

__device__ __forceinline__ void tile_coords(int t, int num_m, int num_n, int& mb, int& nb) {
  constexpr int G = 8;  // pair-tile rows per raster band
  const int band = t / (G * num_n);
  const int m_start = band * G;
  const int band_m = min(G, num_m - m_start);
  const int idx = t - band * G * num_n;
  mb = m_start + idx % band_m;
  nb = idx / band_m;
}

// alpha*(acc + C) + bias for `cw` consecutive columns starting at col0 of one row.
template <int CW>
__device__ __forceinline__ void finish_vals(const Epi2& ep, float (&v)[CW], int64_t row, int64_t col0) {
  const bool in_row = row < ep.M;
  const bool full = col0 + CW <= ep.N;
  if (ep.C && in_row) {
    const float* c = ep.C + row * ep.ldc + col0;
    if (full && ep.c_vec) {
#pragma unroll
      for (int i = 0; i < CW / 4; ++i) {
        float4 x = reinterpret_cast<const float4*>(c)[i];
        v[4 * i] += x.x;
        v[4 * i + 1] += x.y;
        v[4 * i + 2] += x.z;
        v[4 * i + 3] += x.w;
      }
    } else {
#pragma unroll
      for (int i = 0; i < CW; ++i)
        if (col0 + i < ep.N) v[i] += c[i];
    }
  }
#pragma unroll
  for (int i = 0; i < CW; ++i) v[i] *= ep.alpha;
  if (ep.bias) {
    const __nv_bfloat16* b = reinterpret_cast<const __nv_bfloat16*>(ep.bias) + col0;
#pragma unroll
    for (int i = 0; i < CW; ++i)
      if (col0 + i < ep.N) v[i] += __bfloat162float(b[i]);
  }
}

// Stage one 32-row x 128-byte box (row = lane) with the 128-byte swizzle the TMA store expects.
template <int CW>
__device__ __forceinline__ void stage_row(uint8_t* stg, int lane, const float (&v)[CW], int out_bf16) {
  uint8_t* rowp = stg + lane * 128;
  if (out_bf16) {  // CW == 64
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      uint4 u;
      __nv_bfloat162* h = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
      for (int k = 0; k < 4; ++k) h[k] = __floats2bfloat162_rn(v[8 * j + 2 * k], v[8 * j + 2 * k + 1]);
      *reinterpret_cast<uint4*>(rowp + ((j ^ (lane & 7)) << 4)) = u;
    }
  } else {  // CW == 32
#pragma unroll
    for (int j = 0; j < 8; ++j)
      *reinterpret_cast<float4*>(rowp + ((j ^ (lane & 7)) << 4)) =
          make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
  }
}

// Each epilogue warp owns two 4 KB staging buffers used alternately: before refilling one,
// wait until at most one bulk store (the other buffer's) is still reading shared memory.
template <int CW>
__device__ __forceinline__ void store_box(const CUtensorMap* tmD, uint8_t* stg, int& nbox, int lane,
                                          float (&v)[CW], const Epi2& ep, int64_t row, int64_t col0,
                                          int64_t row0) {
  finish_vals<CW>(ep, v, row, col0);
  uint8_t* buf = stg + (nbox & 1) * kOutBytes;
  if (lane == 0) bulk_wait_read1();
  __syncwarp();
  stage_row<CW>(buf, lane, v, ep.out_bf16);
  fence_proxy_async_smem();
  __syncwarp();
  if (lane == 0) {
    tma_store_2d(tmD, buf, static_cast<int>(col0), static_cast<int>(row0));
    bulk_commit();
  }
  ++nbox;
}

// Unit u of a cluster -> (pair-tile row mb, pair-tile column nb of this CTA's pair, K split).
// Cluster shapes (MC): 1 = one CTA pair; 2 = two pairs side by side in N sharing (multicasting)
// their A rows; 3 = two pairs stacked in M sharing their B columns. A "super tile" is the
// cluster's pair-tiles.
constexpr int pairs_of(int MC) { return MC == 1 ? 1 : 2; }
struct Unit {
  int mb, nb, split, ptile;
};
template <int MC>
__device__ __forceinline__ Unit unit_of(int u, int splits, int num_m, int num_n, int pair) {
  Unit x;
  const int st = u / splits;
  x.split = u % splits;
  if (MC == 3) {
    int mbs;
    tile_coords(st, (num_m + 1) / 2, num_n, mbs, x.nb);
    x.mb = mbs * 2 + pair;
  } else {
    const int num_ns = (num_n + MC - 1) / MC;
    int nbs;
    tile_coords(st, num_m, num_ns, x.mb, nbs);
    x.nb = nbs * MC + pair;
  }
  x.ptile = st * pairs_of(MC) + pair;  // dense pair-tile id (split-K partials / counters)
  return x;
}
__host__ __device__ constexpr int super_tiles(int MC, int num_m, int num_n) {
  return MC == 1 ? num_m * num_n
                 : MC == 2 ? num_m * ((num_n + 1) / 2) : ((num_m + 1) / 2) * num_n;
}

template <int BNP, int MC, bool A_MN, bool B_MN>
__global__ void __cluster_dims__(2 * pairs_of(MC), 1, 1) __launch_bounds__(kThreads, 1)
    gemm_tc2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const __grid_constant__ CUtensorMap tmD, const Epi2 ep, int K, int num_m,
                    int num_n) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = sA + PC<BNP>::Stages * kABytes;
  uint8_t* sOut = sB + PC<BNP>::Stages * PC<BNP>::BBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sOut + 8 * kOutBytes);
  uint64_t* empty = full + PC<BNP>::Stages;
  uint64_t* tfull = empty + PC<BNP>::Stages;
  uint64_t* tempty = tfull + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);
  int* sflag = reinterpret_cast<int*>(tslot + 1);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t crank = cluster_rank();
  const uint32_t rank = crank & 1;        // position in the CTA pair
  const int pair = static_cast<int>(crank >> 1);
  const uint32_t lead = crank & ~1u;      // this pair's leader (issues the MMAs)
  const bool leader = rank == 0;
  constexpr int NP = pairs_of(MC);
  const int cid = blockIdx.x / (2 * NP), ncl = gridDim.x / (2 * NP);
  const int num_units = super_tiles(MC, num_m, num_n) * ep.splits;
  const int num_k = (K + kBK - 1) / kBK;
  constexpr uint16_t kAllMask = static_cast<uint16_t>((1u << (2 * NP)) - 1);
  const uint16_t pair_mask = static_cast<uint16_t>(0x3u << (2 * pair));

  if (warp == 0 && lane == 0) {
    tma_prefetch(&tmA);
    tma_prefetch(&tmB);
    tma_prefetch(&tmD);
    for (int s = 0; s < PC<BNP>::Stages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], pairs_of(MC));  // free once every pair's MMAs read it (multicast)
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 8);  // 4 epilogue warps x 2 CTAs (leader's copy is the one used)
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_cg2(tslot, PC<BNP>::TmemCols);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tslot;

  if (warp == 0) {
    if (lane == 0) {
      // ===== TMA producer (both CTAs) =====
      int stage = 0;
      uint32_t phase = 0;
      unsigned long long t_wait = 0, t_begin = clock64();
      for (int u = cid; u < num_units; u += ncl) {
        const Unit t = unit_of<MC>(u, ep.splits, num_m, num_n, pair);
        const int kb0 = t.split * ep.kb_per_split;
        const int kb1 = min(num_k, kb0 + ep.kb_per_split);
        const int m0 = t.mb * 256 + static_cast<int>(rank) * kBM;
        const int n0 = t.nb * BNP + static_cast<int>(rank) * PC<BNP>::BNC;
        for (int kb = kb0; kb < kb1; ++kb) {
          {
            const unsigned long long t0 = clock64();
            mbar_wait(&empty[stage], phase ^ 1);
            t_wait += clock64() - t0;
          }
          if (leader) mbar_expect_tx(&full[stage], 2 * PC<BNP>::StageBytes);
          uint8_t* a_dst = sA + stage * kABytes;
          uint8_t* b_dst = sB + stage * PC<BNP>::BBytes;
          const uint16_t xmask = static_cast<uint16_t>((1u << rank) | (1u << (2 + rank)));
          if (MC != 2) {
            if (!A_MN) {
              tma_load_2d_pair(&tmA, &full[stage], a_dst, kb * kBK, m0);
            } else {
#pragma unroll
              for (int c = 0; c < kBM / 64; ++c)
                tma_load_2d_pair(&tmA, &full[stage], a_dst + c * (kBK * 128), m0 + c * 64, kb * kBK);
            }
          } else {
            // A rows are the same for both pairs of the cluster: pair p fetches the p-th 64-row
            // half of this CTA's 128-row A tile and multicasts it to the same-rank CTA of every
            // pair (halves the TMA issue and L2 reads of A)
            if (!A_MN)
              tma_load_2d_pair_mc(&tmA, &full[stage], a_dst + pair * 64 * 128, kb * kBK,
                                  m0 + pair * 64, xmask);
            else
              tma_load_2d_pair_mc(&tmA, &full[stage], a_dst + pair * (kBK * 128), m0 + pair * 64,
                                  kb * kBK, xmask);
          }
          if (MC != 3) {
            if (!B_MN) {
              tma_load_2d_pair(&tmB, &full[stage], b_dst, kb * kBK, n0);
            } else {
#pragma unroll
              for (int c = 0; c < PC<BNP>::BNC / 64; ++c)
                tma_load_2d_pair(&tmB, &full[stage], b_dst + c * (kBK * 128), n0 + c * 64, kb * kBK);
            }
          } else {
            // B columns are the same for both pairs (stacked in M): pair p fetches half of this
            // CTA's B tile and multicasts it to the same-rank CTA of both pairs
            constexpr int BNC = PC<BNP>::BNC;
            if (!B_MN) {  // stored [N,K]: half the N rows
              tma_load_2d_pair_mc(&tmB, &full[stage], b_dst + pair * (BNC / 2) * 128, kb * kBK,
                                  n0 + pair * (BNC / 2), xmask);
            } else if (BNC >= 128) {  // stored [K,N]: one of the 64-column chunks
              tma_load_2d_pair_mc(&tmB, &full[stage], b_dst + pair * (kBK * 128), n0 + pair * 64,
                                  kb * kBK, xmask);
            } else {  // a single 64-column chunk: half of its K rows
              tma_load_2d_pair_mc(&tmB, &full[stage], b_dst + pair * (kBK / 2) * 128, n0,
                                  kb * kBK + pair * (kBK / 2), xmask);
            }
          }
          if (++stage == PC<BNP>::Stages) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
      if (ep.trace) {
        ep.trace[blockIdx.x * 8 + 0] = t_wait;
        ep.trace[blockIdx.x * 8 + 1] = clock64() - t_begin;
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      // ===== MMA issuer (leader) =====
      constexpr uint32_t idesc = idesc_bf16_f32(256, BNP, A_MN, B_MN);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      unsigned long long t_full = 0, t_temp = 0, t_begin = clock64();
      for (int u = cid; u < num_units; u += ncl) {
        const int split = u % ep.splits;  // same K range for every pair of the cluster
        const int kb0 = split * ep.kb_per_split;
        const int kb1 = min(num_k, kb0 + ep.kb_per_split);
        {
          const unsigned long long t0 = clock64();
          mbar_wait_cluster(&tempty[acc], acc_phase ^ 1);
          t_temp += clock64() - t0;
        }
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * BNP);
        for (int kb = kb0; kb < kb1; ++kb) {
          {
            const unsigned long long t0 = clock64();
            mbar_wait(&full[stage], phase);
            t_full += clock64() - t0;
          }
          tc_fence_after();
          const uint32_t a_base = smem_u32(sA + stage * kABytes);
          const uint32_t b_base = smem_u32(sB + stage * PC<BNP>::BBytes);
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) {
            const uint64_t ad = A_MN ? sdesc_sw128(a_base + k * 2048, kBK * 128, 1024)
                                     : sdesc_sw128(a_base + k * 32, 16, 1024);
            const uint64_t bd = B_MN ? sdesc_sw128(b_base + k * 2048, kBK * 128, 1024)
                                     : sdesc_sw128(b_base + k * 32, 16, 1024);
            umma_bf16_cg2(d_tmem, ad, bd, idesc, (kb > kb0 || k > 0) ? 1u : 0u);
          }
          umma_commit_cg2_mc(&empty[stage], kAllMask);
          if (++stage == PC<BNP>::Stages) {
            stage = 0;
            phase ^= 1;
          }
        }
        umma_commit_cg2_mc(&tfull[acc], pair_mask);
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
      if (ep.trace) {
        ep.trace[blockIdx.x * 8 + 2] = t_full;
        ep.trace[blockIdx.x * 8 + 3] = t_temp;
        ep.trace[blockIdx.x * 8 + 4] = clock64() - t_begin;
      }
    }
  } else {
    // ===== epilogue warps 2..5 (both CTAs): TMEM lane quadrant = warp % 4 =====
    const int quad = warp & 3;
    uint8_t* stg = sOut + (warp - 2) * 2 * kOutBytes;
    int nbox = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    unsigned long long t_tf = 0, t_part = 0, t_begin = clock64();
    for (int u = cid; u < num_units; u += ncl) {
      const Unit t = unit_of<MC>(u, ep.splits, num_m, num_n, pair);
      const int tile = t.ptile, mb = t.mb, nb = t.nb;
      const int64_t rloc = static_cast<int64_t>(rank) * kBM + quad * 32;  // row within pair tile
      const int64_t row0 = static_cast<int64_t>(mb) * 256 + rloc;          // first row of warp
      const int64_t row = row0 + lane;
      const int64_t n0 = static_cast<int64_t>(nb) * BNP;
      {
        const unsigned long long t0 = clock64();
        mbar_wait(&tfull[acc], acc_phase);
        t_tf += clock64() - t0;
      }
      tc_fence_after();
      const uint32_t t_row = tmem_base + (static_cast<uint32_t>(quad * 32) << 16) +
                             static_cast<uint32_t>(acc * BNP);
      if (ep.splits == 1) {
        if (ep.out_bf16) {
#pragma unroll 1
          for (int sub = 0; sub < BNP / 64; ++sub) {
            uint32_t r0[32], r1[32];
            tmem_ld32(t_row + sub * 64, r0);
            tmem_ld32(t_row + sub * 64 + 32, r1);
            tmem_wait_ld();
            float v[64];
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              v[i] = __uint_as_float(r0[i]);
              v[32 + i] = __uint_as_float(r1[i]);
            }
            store_box<64>(&tmD, stg, nbox, lane, v, ep, row, n0 + sub * 64, row0);
          }
        } else {
#pragma unroll 1
          for (int sub = 0; sub < BNP / 32; ++sub) {
            uint32_t r0[32];
            tmem_ld32(t_row + sub * 32, r0);
            tmem_wait_ld();
            float v[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r0[i]);
            store_box<32>(&tmD, stg, nbox, lane, v, ep, row, n0 + sub * 32, row0);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(&tempty[acc], lead);
      } else {
        // ---- split-K: publish this split's fp32 partial, the last split reduces ----
        // partial layout per CTA half: float4 slot f (column/4) major, row minor, so a
        // warp's 32 rows of one slot are 512 contiguous bytes (coalesced store and reload)
        float4* mypart = reinterpret_cast<float4*>(ep.part + static_cast<int64_t>(tile * ep.splits + t.split) *
                                                                 PC<BNP>::TileElems +
                                                   rank * (kBM * BNP)) + quad * 32 + lane;
        const unsigned long long tp0 = clock64();
#pragma unroll 1
        for (int ch = 0; ch < BNP / 32; ++ch) {
          uint32_t r0[32];
          tmem_ld32(t_row + ch * 32, r0);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 8; ++i)
            mypart[(ch * 8 + i) * kBM] =
                make_float4(__uint_as_float(r0[4 * i]), __uint_as_float(r0[4 * i + 1]),
                            __uint_as_float(r0[4 * i + 2]), __uint_as_float(r0[4 * i + 3]));
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(&tempty[acc], lead);  // TMEM free for the next unit
        __threadfence();
        named_barrier_sync(1, 128);
        t_part += clock64() - tp0;
        if (threadIdx.x == 64) {
          int* cnt = ep.counters + tile * 2 + rank;
          const int old = atomicAdd(cnt, 1);
          const int last = old == ep.splits - 1;
          if (last) *cnt = 0;  // ready for the next launch
          *sflag = last;
        }
        named_barrier_sync(1, 128);
        const int last = *sflag;
        named_barrier_sync(1, 128);
        if (last) {
          __threadfence();
          const float4* base =
              reinterpret_cast<const float4*>(ep.part + static_cast<int64_t>(tile) * ep.splits * PC<BNP>::TileElems +
                                              rank * (kBM * BNP)) + quad * 32 + lane;
          constexpr int kSplitStride4 = PC<BNP>::TileElems / 4;
          constexpr int CWB = 64;
          if (ep.out_bf16) {
#pragma unroll 1
            for (int sub = 0; sub < BNP / CWB; ++sub) {
              float v[CWB];
#pragma unroll
              for (int i = 0; i < CWB; ++i) v[i] = 0.f;
              if (ep.splits == 2) {
                float4 x0[CWB / 4], x1[CWB / 4];
                const float4* p0 = base + (sub * (CWB / 4)) * kBM;
                const float4* p1 = p0 + kSplitStride4;
#pragma unroll
                for (int i = 0; i < CWB / 4; ++i) {
                  x0[i] = __ldcg(p0 + i * kBM);
                  x1[i] = __ldcg(p1 + i * kBM);
                }
#pragma unroll
                for (int i = 0; i < CWB / 4; ++i) {
                  v[4 * i] = x0[i].x + x1[i].x;
                  v[4 * i + 1] = x0[i].y + x1[i].y;
                  v[4 * i + 2] = x0[i].z + x1[i].z;
                  v[4 * i + 3] = x0[i].w + x1[i].w;
                }
              } else {
                for (int s = 0; s < ep.splits; ++s) {
                  const float4* p = base + s * kSplitStride4 + (sub * (CWB / 4)) * kBM;
                  float4 x[CWB / 4];
#pragma unroll
                  for (int i = 0; i < CWB / 4; ++i) x[i] = __ldcg(p + i * kBM);
#pragma unroll
                  for (int i = 0; i < CWB / 4; ++i) {
                    v[4 * i] += x[i].x;
                    v[4 * i + 1] += x[i].y;
                    v[4 * i + 2] += x[i].z;
                    v[4 * i + 3] += x[i].w;
                  }
                }
              }
              store_box<CWB>(&tmD, stg, nbox, lane, v, ep, row, n0 + sub * CWB, row0);
            }
          } else {
#pragma unroll 1
            for (int sub = 0; sub < BNP / 32; ++sub) {
              float v[32];
#pragma unroll
              for (int i = 0; i < 32; ++i) v[i] = 0.f;
              for (int s = 0; s < ep.splits; ++s) {
                const float4* p = base + s * kSplitStride4 + (sub * 8) * kBM;
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                  float4 x = __ldcg(p + i * kBM);
                  v[4 * i] += x.x;
                  v[4 * i + 1] += x.y;
                  v[4 * i + 2] += x.z;
                  v[4 * i + 3] += x.w;
                }
              }
              store_box<32>(&tmD, stg, nbox, lane, v, ep, row, n0 + sub * 32, row0);
            }
          }
        }
      }
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
    if (lane == 0) bulk_wait0();
    if (ep.trace && warp == 2 && lane == 0) {
      ep.trace[blockIdx.x * 8 + 5] = t_tf;
      ep.trace[blockIdx.x * 8 + 6] = clock64() - t_begin;
      ep.trace[blockIdx.x * 8 + 7] = t_part;
    }
  }

  tc_fence_before();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_cg2(tmem_base, PC<BNP>::TmemCols);
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

tp_status make_map2(CUtensorMap* m, CUtensorMapDataType dt, size_t esz, const void* base,
                    uint64_t inner, uint64_t outer, uint64_t ld, uint32_t box_inner,
                    uint32_t box_outer) {
  auto fn = encode_fn();
  if (!fn) return fail(TP_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld * esz};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(m, dt, 2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return fail(TP_ERR_SHAPE, "cuTensorMapEncodeTiled (pair kernel) failed: " + std::to_string(int(r)));
  return TP_OK;
}

int sm_count() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

struct Plan2 {
  int num_m, num_n, splits, kbps, grid;
};

// Max co-resident clusters of a kernel (cluster size 4 may strand SMs on some GPCs).
template <typename Kern>
int max_clusters(Kern kern, int csize, int smem) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(csize * 64);
  cfg.blockDim = dim3(kThreads);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = csize;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  int n = 0;
  if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess || n <= 0) {
    cudaGetLastError();
    n = sm_count() / csize;
  }
  return n;
}

template <int BNP, int MC>
Plan2 plan2(const GemmArgs& g, size_t ws_bytes, int clusters) {
  Plan2 p;
  p.num_m = static_cast<int>((g.M + 255) / 256);
  p.num_n = static_cast<int>((g.N + BNP - 1) / BNP);
  const int supers = super_tiles(MC, p.num_m, p.num_n);
  const int ptiles = supers * pairs_of(MC);
  const int num_k = static_cast<int>((g.K + kBK - 1) / kBK);
  int S = 1;
  static const int allow_split = [] {
    const char* e = std::getenv("TP_GEMM_SPLITK");
    return e ? std::atoi(e) : 1;
  }();
  // split-K only when the grid would leave more than half of the clusters idle
  for (int s = 2; s <= 4 && allow_split; ++s) {
    const size_t need = size_t(ptiles) * s * PC<BNP>::TileElems * 4 + size_t(ptiles) * 2 * 4 + 256;
    if (2 * supers <= clusters && supers * s <= clusters && num_k >= 4 * s && need <= ws_bytes) S = s;
  }
  int kbps = (num_k + S - 1) / S;
  S = (num_k + kbps - 1) / kbps;  // no empty split
  if (S < 1) S = 1;
  p.splits = S;
  p.kbps = S > 1 ? kbps : num_k;
  const int units = supers * S;
  p.grid = 2 * pairs_of(MC) * (units < clusters ? units : clusters);
  return p;
}

template <int BNP, int MC, bool A_MN, bool B_MN>
tp_status launch2(const GemmArgs& g, cudaStream_t s) {
  using P = PC<BNP>;
  auto kern = gemm_tc2_kernel<BNP, MC, A_MN, B_MN>;
  static int clusters = 0;
  {
    static std::mutex mu;
    std::lock_guard<std::mutex> lk(mu);
    if (!clusters) {
      TP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, P::Smem));
      clusters = max_clusters(kern, 2 * pairs_of(MC), P::Smem);
    }
  }
  Plan2 pl = plan2<BNP, MC>(g, g.ws_bytes, clusters);
  CUtensorMap ta, tb, td;
  const auto BF = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  // multicast halves: MC 2 loads half of the A rows per pair, MC 3 half of the B tile
  const uint32_t a_rows = MC == 2 ? kBM / 2 : kBM;
  if (!A_MN)
    TP_TRY(make_map2(&ta, BF, 2, g.A, g.K, g.M, g.lda, kBK, a_rows));
  else
    TP_TRY(make_map2(&ta, BF, 2, g.A, g.M, g.K, g.lda, 64, kBK));
  if (!B_MN)
    TP_TRY(make_map2(&tb, BF, 2, g.B, g.K, g.N, g.ldb, kBK, MC == 3 ? P::BNC / 2 : P::BNC));
  else
    TP_TRY(make_map2(&tb, BF, 2, g.B, g.N, g.K, g.ldb, 64,
                     (MC == 3 && P::BNC < 128) ? kBK / 2 : kBK));
  if (g.out_dtype == TP_BF16)
    TP_TRY(make_map2(&td, BF, 2, g.D, g.N, g.M, g.ldd, 64, 32));
  else
    TP_TRY(make_map2(&td, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, g.D, g.N, g.M, g.ldd, 32, 32));

  Epi2 ep;
  ep.C = g.C;
  ep.bias = g.bias;
  ep.ldc = g.ldc;
  ep.alpha = g.alpha;
  ep.out_bf16 = g.out_dtype == TP_BF16;
  ep.M = static_cast<int>(g.M);
  ep.N = static_cast<int>(g.N);
  ep.splits = pl.splits;
  ep.kb_per_split = pl.kbps;
  ep.c_vec = !g.C || ((reinterpret_cast<uintptr_t>(g.C) % 16 == 0) && (g.ldc % 4 == 0));
  ep.part = nullptr;
  ep.counters = nullptr;
  ep.prefetch = 0;
  ep.trace = g_gemm_trace;
  if (pl.splits > 1) {
    const int ptiles = super_tiles(MC, pl.num_m, pl.num_n) * pairs_of(MC);
    char* w = static_cast<char*>(g.ws);
    ep.counters = reinterpret_cast<int*>(w);
    ep.part = reinterpret_cast<float*>(w + 256 * ((ptiles * 2 * 4 + 255) / 256));
    TP_CUDA(cudaMemsetAsync(ep.counters, 0, ptiles * 2 * sizeof(int), s));
  }
  const int tok = prof_begin(0, s, 2.0 * double(g.M) * double(g.N) * double(g.K));
  kern<<<pl.grid, kThreads, P::Smem, s>>>(ta, tb, td, ep, static_cast<int>(g.K), pl.num_m,
                                          pl.num_n);
  count_launch();
  prof_end(tok, s);
  TP_CUDA(cudaGetLastError());
  return TP_OK;
}

template <int BNP, int MC>
tp_status dispatch2(const GemmArgs& g, cudaStream_t s) {
  const bool a_mn = g.trans_a;
  const bool b_mn = !g.trans_b;
  if (!a_mn && !b_mn) return launch2<BNP, MC, false, false>(g, s);
  if (!a_mn && b_mn) return launch2<BNP, MC, false, true>(g, s);
  if (a_mn && !b_mn) return launch2<BNP, MC, true, false>(g, s);
  return launch2<BNP, MC, true, true>(g, s);
}

}  // namespace

bool gemm_tc2_supported(const GemmArgs& g) {
  const size_t osz = dtype_size(g.out_dtype);
  return g.M > 128 && (reinterpret_cast<uintptr_t>(g.D) % 16 == 0) && ((g.ldd * osz) % 16 == 0) &&
         (!g.bias || reinterpret_cast<uintptr_t>(g.bias) % 2 == 0);
}

size_t gemm_tc2_ws_bytes() {
  // split-K scratch upper bound: pair-tiles*splits <= #SMs/2 (74 on B200, +1 ragged super
  // tile), 256x256 fp32 each, plus counters
  return size_t(76) * PC<256>::TileElems * 4 + 76 * 2 * 4 * 4 + 1024;
}

tp_status gemm_tc2_bf16(const GemmArgs& g, cudaStream_t s) {
  // Pair tile 256x256 when those tiles fill the SM pairs, else 256x128 (twice the tiles).
  // Two pairs per cluster (A multicast) whenever there are >= 2 pair-tile columns.
  static const int force_bn = [] {
    const char* e = std::getenv("TP_GEMM_BN");
    return e ? std::atoi(e) : 0;
  }();
  static const int force_mc = [] {
    const char* e = std::getenv("TP_GEMM_MC");
    return e ? std::atoi(e) : 0;
  }();
  const int64_t tiles256 = ((g.M + 255) / 256) * ((g.N + 255) / 256);
  const int pairs = sm_count() / 2;
  const bool wide = force_bn ? force_bn == 256 : tiles256 >= pairs;
  // cluster shape: share the operand that is re-read more (B when few pair-tile rows)
  const int64_t nrows = (g.M + 255) / 256;
  const int64_t ncols = wide ? (g.N + 255) / 256 : (g.N + 127) / 128;
  int mc = 1;
  if (force_mc) mc = force_mc;
  else if (!wide && nrows >= 2 && nrows <= 4) mc = 3;
  if (wide) {
    if (mc == 2 && ncols >= 2) return dispatch2<256, 2>(g, s);
    if (mc == 3 && nrows >= 2) return dispatch2<256, 3>(g, s);
    return dispatch2<256, 1>(g, s);
  }
  if (mc == 2 && ncols >= 2) return dispatch2<128, 2>(g, s);
  if (mc == 3 && nrows >= 2) return dispatch2<128, 3>(g, s);
  return dispatch2<128, 1>(g, s);
}

}  // namespace tp
