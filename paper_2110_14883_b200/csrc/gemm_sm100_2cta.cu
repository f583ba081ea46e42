// CTA-pair (tcgen05 cta_group::2) bf16 GEMM for sm_100a — the main local-GEMM kernel of every
// TP mode:   D[M,N] = alpha * (op(A).op(B) + C) + bias[col],
// for ONE problem or a GROUP of two independent problems in one persistent launch (e.g. the
// backward's dX = dY.W^T and dW = X^T.dY, whose tiles together fill the machine).
//
// Design (profiles/r01_gemm_v1_summary.md, r01_gemm_v2_summary.md):
//   * a CTA pair computes a 256 x BNP tile (BNP 256 or 128): each CTA stages its 128 rows of
//     A and BNP/2 of the B columns, the leader issues M=256 N=BNP MMAs reading both CTAs'
//     shared memory, each CTA keeps its 128 accumulator rows in its own TMEM;
//   * cluster of 1 pair, or 2 pairs sharing an operand by TMA multicast (MC 2: pairs side by
//     side in N share A; MC 3: pairs stacked in M share B);
//   * persistent over units (problem, pair-tile, K split), 192 threads per CTA: warp 0 TMA
//     producer (both CTAs; bytes land on the pair leader's `full` barrier), warp 1 TMEM
//     allocator (both) + MMA issuer (leader), warps 2..5 epilogue (both);
//   * 6-8 stage smem ring, BK = 64 with 128-byte swizzle; operand majorness (K- or MN-major)
//     is per problem at run time (descriptors + instruction descriptor), so transposes are
//     never copies; TMEM accumulator double-buffered so the epilogue overlaps the next unit;
//   * split-K when a single problem has too few tiles: every split writes an fp32 partial,
//     the last split to arrive sums the partials in split order (deterministic);
//   * epilogue: TMEM -> registers -> alpha / C / bias / cast -> 128-byte-swizzled smem staging
//     (two buffers per warp) -> TMA bulk tensor store;
//   * programmatic dependent launch: the prologue overlaps the previous kernel's tail.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <climits>
#include <cstdlib>
#include <mutex>
#include <queue>
#include <vector>

#include "sm100_ptx.cuh"
#include "tp_internal.h"

// per-k-block clock64 instrumentation of the main loops (tools/gemm_trace.py); off by default
#ifndef TP_LOOP_CLOCKS
#define TP_LOOP_CLOCKS 0
#endif
// per-unit timeline of the pair kernel (tools/gemm_timeline.py); off by default. Slots per CTA
// (kTlStride, after the 300 x 16 wait-counter block of the trace buffer): 0 entry, 1 after the
// prologue, 2 exit, 3 / 4 producer's first / last TMA issue; per unit i < 16: 8+i first MMA issued,
// 24+i accumulator commit issued, 40+i epilogue saw the accumulator, 56+i epilogue released it
// (warp 2); 72..75 epilogue phase sums of warp 2: TMEM load, staging-buffer wait, stage + fence,
// store issue.
#ifndef TP_TIMELINE
#define TP_TIMELINE 0
#endif
#if TP_TIMELINE
#define TL_SET(slot, v) do { if (G.trace) G.trace[300 * 16 + blockIdx.x * 128 + (slot)] = (v); } while (0)
#define TL_ADD(slot, v) do { if (G.trace) G.trace[300 * 16 + blockIdx.x * 128 + (slot)] += (v); } while (0)
#else
#define TL_SET(slot, v) do { } while (0)
#define TL_ADD(slot, v) do { } while (0)
#endif

namespace tp {
unsigned long long* g_gemm_trace = nullptr;  // set by tp_gemm_trace (tools only)
namespace {

using namespace ptx;

constexpr int kBM = 128;  // A rows per CTA (pair tile: 256 rows)
constexpr int kBK = 64;
constexpr int kABytes = kBM * kBK * 2;
constexpr int kOutBytes = 32 * 128;  // per epilogue warp and buffer: 32 rows x 128 B staging
// Epilogue warps EW: 4 (one per TMEM lane quadrant) or 8 (two per quadrant, each half of the
// columns; one ring stage less). 8 wins only where the epilogue is everything (1-2 k-blocks per
// tile: C3's 16384^2 x 64 dW 132 -> 113 us) and loses elsewhere (C2 891 -> 860 TFLOP/s;
// profiles/r01_attention_summary.md), so the dispatcher picks it per problem.
// release / acquire at GPU scope for the split-K partial hand-off (each writer fences before the
// CTA barrier that precedes the counter atomic; the reader fences after observing the count).
// __threadfence() is fence.sc.gpu, a heavier sequentially consistent fence than this needs.
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }

template <int EW>
constexpr int threads_of() { return 64 + 32 * EW; }  // warp 0 TMA, warp 1 MMA, warps 2.. epilogue
constexpr int kMaxProbs = 4;
constexpr int kMaxPanels = 4;  // K-panels per problem (peer shards of a fused SUMMA)
constexpr int kMaxDPanels = 8;  // D row-panels per problem (fused 1D reduce-scatter slots)

// Pair-tile width BNP (256 or 128): B columns per CTA, ring depth, TMEM, smem. MC 5 (K-split
// pair cluster) gives one ring stage to the 32 KB DSMEM receive buffer of the split reduction.
constexpr int kRxBytes = 2 * 32 * kBM * 4;  // MC 5: two [32 cols][128 rows] fp32 chunks
// shared-memory copy of the problems' scalars (512 B) and of this cluster's unit list (256 B)
constexpr int kScalBytes = 1024;
template <int BNP, int MC = 1, int EW = 4>
struct PC {
  static constexpr int BNC = BNP / 2;
  static constexpr int Stages = EW == 8 ? (BNP == 256 ? (MC == 5 ? 4 : 5) : (MC == 5 ? 5 : 6))
                                               : (BNP == 256 ? (MC == 5 ? 5 : 6) : (MC == 5 ? 6 : 8));
  static constexpr int BBytes = BNC * kBK * 2;
  static constexpr int StageBytes = kABytes + BBytes;
  static constexpr int TmemCols = 2 * BNP;
  static constexpr int Rx = MC == 5 ? kRxBytes : 0;
  static constexpr int Smem = Stages * StageBytes + 2 * EW * kOutBytes + Rx + kScalBytes + 1024 + 256;
  static constexpr int TileElems = 256 * BNP;
};

// Per-problem scalars. The pair kernel copies them into shared memory once per CTA: the loops
// read them per unit (unit decode, descriptors, epilogue parameters), and indexed loads from the
// ~11 KB parameter block missed the constant cache (~1K clocks between units, tools/gemm_timeline).
struct ProbS {
  int d_rows;                                      // rows per D panel (0: a single D)
  const float* C;
  const void* bias;
  float* part;
  int* counters;
  int64_t ldc;
  float alpha;
  int out_bf16;
  int M, N, K;
  int a_mn, b_mn;
  int num_m, num_n;
  int splits, kb_per_split;
  int c_vec;
  int owner_wait;  // split-K: split 0 keeps its tile in TMEM and waits for the other splits
  int ptiles;      // pair tiles of this problem (split-K flag layout)
  int npanels, kb_panel, num_kb;  // K = npanels panels of kb_panel 64-wide k-blocks
  int unit0;  // first unit of this problem in the launch's unit space
  int narrow_nb;  // n-tile index computed as a half-width (N = 128) pair tile, -1 none
  int a_box64;    // K-major A loaded as two 64-row boxes (TP_GEMM_ABOX64, measurement knob)
};
struct Prob : ProbS {
  CUtensorMap tmA[kMaxPanels], tmB[kMaxPanels];  // one A/B map per K-panel
  CUtensorMap tmD[kMaxDPanels];                   // one D map per row-panel (usually 1)
};
constexpr int kMaxClusterUnits = 128;  // scheduled units per cluster held in shared memory
static_assert(sizeof(ProbS) * kMaxProbs <= 512, "problem scalars exceed their smem slot");

// Unit schedule: cluster c runs units sched_order[sched_start[c] .. sched_start[c + 1]) when
// `sched` is set (a host-side longest-processing-time assignment for launches whose units differ
// in length, e.g. the backward's long-K dX tiles next to many short dW tiles), else the static
// round robin u = c, c + #clusters, ...
constexpr int kMaxSchedClusters = 80;   // >= 148 / 2 pair clusters
constexpr int kMaxSchedUnits = 1024;
struct Group {
  Prob p[kMaxProbs];
  int nprob;
  int total_units;
  int raster;  // pair-tile rows per raster band (8; TP_GEMM_RASTER for measurements)
  unsigned long long* trace;  // optional per-CTA wait-cycle counters (tp_gemm_trace)
  int sched;
  int epi_diag;  // TP_TIMELINE builds only: 1 = epilogue skips the TMA stores, 2 = also the staging
  uint16_t sched_start[kMaxSchedClusters + 1];
  uint16_t sched_order[kMaxSchedUnits];
};

__device__ __forceinline__ int units_of_cluster(const Group& G, int cid, int ncl) {
  if (G.sched) return G.sched_start[cid + 1] - G.sched_start[cid];
  return cid < G.total_units ? (G.total_units - cid + ncl - 1) / ncl : 0;
}
__device__ __forceinline__ int unit_at(const Group& G, int cid, int ncl, int i) {
  return G.sched ? static_cast<int>(G.sched_order[G.sched_start[cid] + i]) : cid + i * ncl;
}
// the same from the shared-memory copy of the cluster's list (pair kernel)
__device__ __forceinline__ int unit_at_s(int sched, const uint16_t* ulist, int cid, int ncl, int i) {
  return sched ? static_cast<int>(ulist[i]) : cid + i * ncl;
}

__device__ __forceinline__ void tile_coords(int t, int num_m, int num_n, int& mb, int& nb, int G) {
  // G = pair-tile rows per raster band (Group::raster)
  const int band = t / (G * num_n);
  const int m_start = band * G;
  const int band_m = min(G, num_m - m_start);
  const int idx = t - band * G * num_n;
  mb = m_start + idx % band_m;
  nb = idx / band_m;
}

// Cluster shapes (MC): 1 = one CTA pair; 2 = two pairs side by side in N sharing their A rows;
// 3 = two pairs stacked in M sharing their B columns. A "super tile" = the cluster's tiles.
// 4 = 2x2 pairs (cluster of 8): A shared along N and B along M, both by multicast.
// 5 = K-split pair cluster: both pairs compute the SAME tile, pair 0 over the first half of K,
//     pair 1 over the second; pair 1 streams its fp32 accumulator into pair 0's shared memory
//     (DSMEM, 32-column chunks, double-buffered) and pair 0 adds it and stores the tile. Fills
//     the machine for few-tile (small-M) products without a global split-K round trip.
__host__ __device__ constexpr int pairs_of(int MC) { return MC == 1 ? 1 : MC == 4 ? 4 : 2; }
__host__ __device__ constexpr bool mc_a(int MC) { return MC == 2 || MC == 4; }  // A multicast
__host__ __device__ constexpr bool mc_b(int MC) { return MC == 3 || MC == 4; }  // B multicast
__host__ __device__ constexpr int super_tiles(int MC, int num_m, int num_n) {
  return (MC == 1 || MC == 5) ? num_m * num_n
         : MC == 2 ? num_m * ((num_n + 1) / 2)
         : MC == 3 ? ((num_m + 1) / 2) * num_n
                   : ((num_m + 1) / 2) * ((num_n + 1) / 2);
}

struct Unit {
  int prob, mb, nb, split, ptile;
};

template <int MC>
__device__ __forceinline__ Unit unit_of(const ProbS* sp, int nprob, int raster, int u, int pair) {
  Unit x;
  x.prob = 0;
#pragma unroll
  for (int i = 1; i < kMaxProbs; ++i)
    if (i < nprob && u >= sp[i].unit0) x.prob = i;
  const ProbS& P = sp[x.prob];
  const int lu = u - P.unit0;
  const int st = lu / P.splits;
  x.split = lu % P.splits;
  if (MC == 5) {  // both pairs on the same tile; `split` = which half of K
    tile_coords(st, P.num_m, P.num_n, x.mb, x.nb, raster);
    x.split = pair;
    x.ptile = st;
    return x;
  } else if (MC == 4) {
    int mbs, nbs;
    tile_coords(st, (P.num_m + 1) / 2, (P.num_n + 1) / 2, mbs, nbs, raster);
    x.mb = mbs * 2 + (pair >> 1);
    x.nb = nbs * 2 + (pair & 1);
  } else if (MC == 3) {
    int mbs;
    tile_coords(st, (P.num_m + 1) / 2, P.num_n, mbs, x.nb, raster);
    x.mb = mbs * 2 + pair;
  } else {
    const int num_ns = (P.num_n + MC - 1) / MC;
    int nbs;
    tile_coords(st, P.num_m, num_ns, x.mb, nbs, raster);
    x.nb = nbs * MC + pair;
  }
  x.ptile = st * pairs_of(MC) + pair;  // dense pair-tile id (split-K partials / counters)
  return x;
}

// alpha*(acc + C) + bias for CW consecutive columns starting at col0 of one row.
template <int CW>
__device__ __forceinline__ void finish_vals(const ProbS& ep, float (&v)[CW], int64_t row, int64_t col0) {
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
__device__ __forceinline__ void stage_row(uint8_t* stg, int lane, const float (&v)[CW]) {
  const uint32_t rowp = smem_u32(stg) + lane * 128;
  if (CW == 64) {  // bf16
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      uint32_t u[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        __nv_bfloat162 h = __floats2bfloat162_rn(v[8 * j + 2 * k], v[8 * j + 2 * k + 1]);
        u[k] = *reinterpret_cast<uint32_t*>(&h);
      }
      sts128(rowp + ((j ^ (lane & 7)) << 4), u[0], u[1], u[2], u[3]);
    }
  } else {  // fp32, CW == 32
#pragma unroll
    for (int j = 0; j < 8; ++j)
      sts128(rowp + ((j ^ (lane & 7)) << 4), __float_as_uint(v[4 * j]), __float_as_uint(v[4 * j + 1]),
             __float_as_uint(v[4 * j + 2]), __float_as_uint(v[4 * j + 3]));
  }
}

// Two staging buffers per warp used alternately: before refilling one, wait until at most one
// bulk store (the other buffer's) is still reading shared memory.
template <int CW>
__device__ __forceinline__ void store_box(const ProbS& ep, const CUtensorMap* tmD, uint8_t* stg, int& nbox, int lane,
                                          float (&v)[CW], int64_t row, int64_t col0, int64_t row0,
                                          unsigned long long* tl = nullptr, int diag = 0) {
#if TP_TIMELINE
  const unsigned long long cf = clock64();
#endif
  finish_vals<CW>(ep, v, row, col0);
  uint8_t* buf = stg + (nbox & 1) * kOutBytes;
#if TP_TIMELINE
  unsigned long long c0 = clock64();
  if (tl && lane == 0) tl[5] += c0 - cf;
  if (diag == 2) {  // keep the values live, skip staging and store
    if (v[0] == 12345.f && v[CW - 1] == -1.f) stg[lane] = 1;
    ++nbox;
    return;
  }
#endif
  if (lane == 0) bulk_wait_read1();
  __syncwarp();
#if TP_TIMELINE
  unsigned long long c1 = clock64();
#endif
  stage_row<CW>(buf, lane, v);
  fence_proxy_async_smem();
  __syncwarp();
#if TP_TIMELINE
  unsigned long long c2 = clock64();
  if (tl && lane == 0) {
    tl[1] += c1 - c0;
    tl[2] += c2 - c1;
  }
#endif
#if TP_TIMELINE
  if (diag == 1) {
    ++nbox;
    return;
  }
#endif
  if (lane == 0) {
    const int pi = ep.d_rows ? static_cast<int>(row0 / ep.d_rows) : 0;
    if (pi < kMaxDPanels) {
      tma_store_2d(&tmD[pi], buf, static_cast<int>(col0),
                   static_cast<int>(row0 - int64_t(pi) * ep.d_rows));
      bulk_commit();
    }
  }
#if TP_TIMELINE
  if (tl && lane == 0) tl[3] += clock64() - c2;
#endif
  ++nbox;
}

// CW output columns (sub-chunk `sub`) of this thread's row, straight from TMEM.
template <int CW>
__device__ __forceinline__ void tmem_cols(uint32_t t_row, int sub, float (&v)[CW]) {
  uint32_t r0[32];
  tmem_ld32(t_row + sub * CW, r0);
  if (CW == 64) {
    uint32_t r1[32];
    tmem_ld32(t_row + sub * CW + 32, r1);
    tmem_wait_ld();
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      v[i] = __uint_as_float(r0[i]);
      v[(CW == 64 ? 32 : 0) + i] = __uint_as_float(r1[i]);
    }
  } else {
    tmem_wait_ld();
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r0[i]);
  }
}

// Last split: sum the S fp32 partials of this thread's row for sub-chunk `sub`, split order.
template <int CW>
__device__ __forceinline__ void sum_partials(const float4* base, int splits, int split_stride4,
                                             int sub, float (&v)[CW]) {
#pragma unroll
  for (int i = 0; i < CW; ++i) v[i] = 0.f;
  if (splits == 2) {
    float4 x0[CW / 4], x1[CW / 4];
    const float4* p0 = base + (sub * (CW / 4)) * kBM;
    const float4* p1 = p0 + split_stride4;
#pragma unroll
    for (int i = 0; i < CW / 4; ++i) {
      x0[i] = __ldcg(p0 + i * kBM);
      x1[i] = __ldcg(p1 + i * kBM);
    }
#pragma unroll
    for (int i = 0; i < CW / 4; ++i) {
      v[4 * i] = x0[i].x + x1[i].x;
      v[4 * i + 1] = x0[i].y + x1[i].y;
      v[4 * i + 2] = x0[i].z + x1[i].z;
      v[4 * i + 3] = x0[i].w + x1[i].w;
    }
  } else {
    for (int s = 0; s < splits; ++s) {
      const float4* p = base + s * split_stride4 + (sub * (CW / 4)) * kBM;
      float4 x[CW / 4];
#pragma unroll
      for (int i = 0; i < CW / 4; ++i) x[i] = __ldcg(p + i * kBM);
#pragma unroll
      for (int i = 0; i < CW / 4; ++i) {
        v[4 * i] += x[i].x;
        v[4 * i + 1] += x[i].y;
        v[4 * i + 2] += x[i].z;
        v[4 * i + 3] += x[i].w;
      }
    }
  }
}

// v += partials of splits 1..S-1 (split order) for sub-chunk `sub` of this thread's row. All
// loads of one split are issued before use (memory-level parallelism: the partials are L2-hot).
template <int CW>
__device__ __forceinline__ void add_partials(const float4* base, int splits, int split_stride4,
                                             int sub, float (&v)[CW]) {
  for (int sp = 1; sp < splits; ++sp) {
    const float4* p = base + sp * split_stride4 + (sub * (CW / 4)) * kBM;
    float4 x[CW / 4];
#pragma unroll
    for (int i = 0; i < CW / 4; ++i) x[i] = __ldcg(p + i * kBM);
#pragma unroll
    for (int i = 0; i < CW / 4; ++i) {
      v[4 * i] += x[i].x;
      v[4 * i + 1] += x[i].y;
      v[4 * i + 2] += x[i].z;
      v[4 * i + 3] += x[i].w;
    }
  }
}

template <int BNP, int MC, int EW>
__global__ void __cluster_dims__(2 * pairs_of(MC), 1, 1) __launch_bounds__(threads_of<EW>(), 1)
    gemm_tc2_kernel(const __grid_constant__ Group G) {
  using P = PC<BNP, MC, EW>;
  constexpr int NP = pairs_of(MC);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = sA + P::Stages * kABytes;
  uint8_t* sOut = sB + P::Stages * P::BBytes;
  float* rx = reinterpret_cast<float*>(sOut + 2 * EW * kOutBytes);  // MC 5: [2][32][128]
  ProbS* sp = reinterpret_cast<ProbS*>(sOut + 2 * EW * kOutBytes + P::Rx);
  uint64_t* full = reinterpret_cast<uint64_t*>(sOut + 2 * EW * kOutBytes + P::Rx + kScalBytes);
  uint64_t* empty = full + P::Stages;
  uint64_t* tfull = empty + P::Stages;
  uint64_t* tempty = tfull + 2;
  uint64_t* rxf = tempty + 2;  // MC 5, in pair 0: the sender's chunks landed (tx bytes)
  uint64_t* rxe = rxf + 2;     // MC 5, in pair 1: the owner consumed them (4 owner warps)
  uint32_t* tslot = reinterpret_cast<uint32_t*>(rxe + 2);
  int* sflag = reinterpret_cast<int*>(tslot + 1);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (G.trace && threadIdx.x == 0) {  // entry timestamps (tools only)
    G.trace[blockIdx.x * 16 + 7] = globaltimer();
    G.trace[blockIdx.x * 16 + 10] = clock64();
    TL_SET(0, clock64());
  }
  const uint32_t crank = cluster_rank();
  const uint32_t rank = crank & 1;   // position in the CTA pair
  const int pair = static_cast<int>(crank >> 1);
  const uint32_t lead = crank & ~1u;  // this pair's leader (issues the MMAs)
  const bool leader = rank == 0;
  const int cid = blockIdx.x / (2 * NP), ncl = gridDim.x / (2 * NP);
  constexpr uint16_t kAllMask = static_cast<uint16_t>((1u << (2 * NP)) - 1);
  const uint16_t pair_mask = static_cast<uint16_t>(0x3u << (2 * pair));
  // multicast partners (same rank in the pair): MC 2/3 the other pair; MC 4 (pair = 2*pm + pn)
  // A goes to the pairs of the same pair-row pm, B to the pairs of the same pair-column pn
  const int a_idx = MC == 4 ? (pair & 1) : pair;   // which half of the shared A box this pair loads
  const int b_idx = MC == 4 ? (pair >> 1) : pair;  // which half of the shared B box
  const uint16_t xmask_a = static_cast<uint16_t>(
      MC == 4 ? (1u << (4 * (pair >> 1) + rank)) | (1u << (4 * (pair >> 1) + 2 + rank))
              : (1u << rank) | (1u << (2 + rank)));
  const uint16_t xmask_b = static_cast<uint16_t>(
      MC == 4 ? (1u << (2 * (pair & 1) + rank)) | (1u << (4 + 2 * (pair & 1) + rank))
              : (1u << rank) | (1u << (2 + rank)));

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < G.nprob; ++i) {
      for (int k = 0; k < G.p[i].npanels; ++k) {
        tma_prefetch(&G.p[i].tmA[k]);
        tma_prefetch(&G.p[i].tmB[k]);
      }
      tma_prefetch(&G.p[i].tmD[0]);
    }
    for (int s = 0; s < P::Stages; ++s) {
      mbar_init(&full[s], 1);
      // free once every pair's MMAs have read it (multicast); MC 5 pairs share nothing
      mbar_init(&empty[s], MC == 5 ? 1 : NP);
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], 2 * EW);  // epilogue warps x 2 CTAs (the leader's copy is used)
      mbar_init(&rxf[a], 1);  // MC 5 owner: its own expect_tx arrive + the sender's bulk bytes
      mbar_init(&rxe[a], 4);  // MC 5 sender: the owner's 4 epilogue warps
    }
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_cg2(tslot, P::TmemCols);
  // launch parameters the loops read per unit go to shared memory / registers here, under the
  // barrier init and TMEM allocation (first reads of the parameter block miss the constant cache)
  uint16_t* ulist = reinterpret_cast<uint16_t*>(reinterpret_cast<uint8_t*>(sp) + 512);
  const int sched = G.sched;
  const int nu = units_of_cluster(G, cid, ncl);
  if (warp == 2 && lane < G.nprob) sp[lane] = static_cast<const ProbS&>(G.p[lane]);
  if (warp == 3 && sched) {
    const int base = G.sched_start[cid];
    for (int i = lane; i < nu; i += 32) ulist[i] = G.sched_order[base + i];
  }
  const int nprob = G.nprob, raster = G.raster;
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tslot;
  // the prologue above overlaps the previous kernel's tail (PDL); operands, C and outputs are
  // touched only once the previous kernel's results are visible
  pdl_launch_dependents();
  pdl_wait();
  if (G.trace && threadIdx.x == 0) G.trace[blockIdx.x * 16 + 8] = globaltimer();
#if TP_TIMELINE
  unsigned long long* tl = G.trace ? G.trace + 300 * 16 + blockIdx.x * 128 : nullptr;
  if (threadIdx.x == 0) TL_SET(1, clock64());
#else
  unsigned long long* tl = nullptr;
#endif
  (void)tl;

  if (warp == 0) {
    {
      // ===== TMA producer (both CTAs of every pair) =====
      // The whole warp runs the loop (its values stay warp-uniform, in uniform registers) and
      // one elected lane issues: a single thread's instruction latency would otherwise pace
      // the pipeline (profiles/r01_gemm_v3_summary.md).
      int stage = 0;
      uint32_t phase = 0;
      unsigned long long t_wait = 0, t_begin = clock64();
      for (int ui = 0; ui < nu; ++ui) {
        const int u = unit_at_s(sched, ulist, cid, ncl, ui);
        const Unit t = unit_of<MC>(sp, nprob, raster, u, pair);
        const ProbS& pr = sp[t.prob];
        const Prob& pm = G.p[t.prob];
        const int kb0 = t.split * pr.kb_per_split;  // MC 5: split = this pair's K half
        const int kb1 = min(pr.num_kb, kb0 + pr.kb_per_split);
        const int m0 = t.mb * 256 + static_cast<int>(rank) * kBM;
        // ragged last n-tile of <= BNP/2 columns: an N = BNP/2 pair tile (half the B bytes and
        // MMA time instead of a full tile whose second half is zero fill)
        const bool nar = MC == 1 && BNP == 256 && t.nb == pr.narrow_nb;
        const int n0 = t.nb * BNP + static_cast<int>(rank) * (nar ? P::BNC / 2 : P::BNC);
        // k-block kb lives in K-panel kb / kb_panel (its own tensor maps, e.g. a peer's shard);
        // the panel and in-panel column advance incrementally (no division in the loop: the
        // single producer thread's instruction latency is on the pipeline's critical path)
        const int kc_end = pr.kb_panel * kBK;
        int panel = kb0 / pr.kb_panel;
        int kc = (kb0 - panel * pr.kb_panel) * kBK;
        const CUtensorMap* mA = &pm.tmA[panel];
        const CUtensorMap* mB = &pm.tmB[panel];
        // copies: the asm "memory" clobbers below would otherwise force param-space reloads
        const bool a_mn = pr.a_mn != 0, b_mn = pr.b_mn != 0;
        const CUtensorMap* const tmA = pm.tmA;
        const CUtensorMap* const tmB = pm.tmB;
        for (int kb = kb0; kb < kb1; ++kb) {
#if TP_LOOP_CLOCKS
          {
            const unsigned long long t0 = clock64();
            mbar_wait(&empty[stage], phase ^ 1);
            t_wait += clock64() - t0;
          }
#else
          mbar_wait(&empty[stage], phase ^ 1);
#endif
          if (elect_one()) {
#if TP_TIMELINE
          if (ui == 0 && kb == kb0) TL_SET(3, clock64());
          TL_SET(4, clock64());
#endif
          if (leader) mbar_expect_tx(&full[stage], 2 * (nar ? kABytes + P::BBytes / 2 : P::StageBytes));
          uint8_t* a_dst = sA + stage * kABytes;
          uint8_t* b_dst = sB + stage * P::BBytes;
          // ---- A: this CTA's 128 rows (K-major: one box; MN-major: two 64-wide chunks)
          if (!mc_a(MC)) {
            if (!a_mn && pr.a_box64) {
              tma_load_2d_pair(mA, &full[stage], a_dst, kc, m0);
              tma_load_2d_pair(mA, &full[stage], a_dst + 64 * 128, kc, m0 + 64);
            } else if (!a_mn) {
              tma_load_2d_pair(mA, &full[stage], a_dst, kc, m0);
            } else {
              for (int c = 0; c < kBM / 64; ++c)
                tma_load_2d_pair(mA, &full[stage], a_dst + c * (kBK * 128), m0 + c * 64, kc);
            }
          } else {  // this pair fetches half a_idx and multicasts it to the A-sharing CTAs
            if (!a_mn)
              tma_load_2d_pair_mc(mA, &full[stage], a_dst + a_idx * 64 * 128, kc,
                                  m0 + a_idx * 64, xmask_a);
            else
              tma_load_2d_pair_mc(mA, &full[stage], a_dst + a_idx * (kBK * 128),
                                  m0 + a_idx * 64, kc, xmask_a);
          }
          // ---- B: this CTA's BNP/2 columns
          if (!mc_b(MC)) {
            if (!b_mn) {
              tma_load_2d_pair(nar ? &tmB[1] : mB, &full[stage], b_dst, kc, n0);  // [1]: 64-row box
            } else {
              for (int c = 0; c < (nar ? P::BNC / 128 : P::BNC / 64); ++c)
                tma_load_2d_pair(mB, &full[stage], b_dst + c * (kBK * 128), n0 + c * 64, kc);
            }
          } else {  // pairs stacked in M share B: this pair fetches half b_idx, multicasts it
            constexpr int BNC = P::BNC;
            if (!b_mn)
              tma_load_2d_pair_mc(mB, &full[stage], b_dst + b_idx * (BNC / 2) * 128, kc,
                                  n0 + b_idx * (BNC / 2), xmask_b);
            else if (BNC >= 128)
              tma_load_2d_pair_mc(mB, &full[stage], b_dst + b_idx * (kBK * 128), n0 + b_idx * 64,
                                  kc, xmask_b);
            else
              tma_load_2d_pair_mc(mB, &full[stage], b_dst + b_idx * (kBK / 2) * 128, n0,
                                  kc + b_idx * (kBK / 2), xmask_b);
          }
          }
          __syncwarp();
          if (++stage == P::Stages) {
            stage = 0;
            phase ^= 1;
          }
          kc += kBK;
          if (kc == kc_end) {
            kc = 0;
            ++panel;
            mA = &tmA[panel];
            mB = &tmB[panel];
          }
        }
      }
      if (G.trace && lane == 0) {
        G.trace[blockIdx.x * 16 + 0] = t_wait;
        G.trace[blockIdx.x * 16 + 1] = clock64() - t_begin;
      }
    }
  } else if (warp == 1) {
    if (leader) {
      // ===== MMA issuer (pair leader; whole warp, one elected lane issues) =====
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      unsigned long long t_full = 0, t_temp = 0, t_first = 0, t_unit0 = 0, t_steady = 0, n_steady = 0,
                         t_begin = clock64();
      for (int ui = 0; ui < nu; ++ui) {
        const int u = unit_at_s(sched, ulist, cid, ncl, ui);
        const Unit t = unit_of<MC>(sp, nprob, raster, u, pair);
        const ProbS& pr = sp[t.prob];
        const int num_k = pr.num_kb;
        const int kb0 = t.split * pr.kb_per_split;
        const int kb1 = min(num_k, kb0 + pr.kb_per_split);
        const bool nar = MC == 1 && BNP == 256 && t.nb == pr.narrow_nb;
        const uint32_t idesc = idesc_bf16_f32(256, nar ? BNP / 2 : BNP, pr.a_mn != 0, pr.b_mn != 0);
        // K-major: +32 B per 16-element K step inside the 128 B swizzle atom (SBO = 8 rows).
        // MN-major: +16 rows x 128 B per K step; LBO = one 64-wide MN chunk (BK rows).
        // Descriptors are built once per unit; per k-block / K step only the 16-byte-granular
        // start-address field (low 14 bits, no carry: smem < 256 KB) advances.
        const uint32_t a_step4 = pr.a_mn ? 2048u / 16 : 32u / 16;
        const uint32_t b_step4 = pr.b_mn ? 2048u / 16 : 32u / 16;
        const uint64_t a_desc0 = sdesc_sw128(smem_u32(sA), pr.a_mn ? kBK * 128 : 16, 1024);
        const uint64_t b_desc0 = sdesc_sw128(smem_u32(sB), pr.b_mn ? kBK * 128 : 16, 1024);
        {
          const unsigned long long t0 = clock64();
          mbar_wait(&tempty[acc], acc_phase ^ 1);
          t_temp += clock64() - t0;
        }
        __syncwarp();
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + static_cast<uint32_t>(acc * BNP);
        for (int kb = kb0; kb < kb1; ++kb) {
#if TP_LOOP_CLOCKS
          {
            const unsigned long long t0 = clock64();
            mbar_wait(&full[stage], phase);
            const unsigned long long t1 = clock64();
            const unsigned long long dt = t1 - t0;
            t_full += dt;
            if (kb == kb0) {
              t_first += dt;
              t_unit0 = t1;
            }
            if (kb == kb1 - 1) {  // steady-state cycles per k-block inside this unit
              t_steady += t1 - t_unit0;
              n_steady += kb1 - kb0 - 1;
            }
          }
#else
          mbar_wait(&full[stage], phase);
#endif
          tc_fence_after();
          const uint64_t ad = a_desc0 + static_cast<uint32_t>(stage * (kABytes / 16));
          const uint64_t bd = b_desc0 + static_cast<uint32_t>(stage * (P::BBytes / 16));
          if (elect_one()) {
#if TP_TIMELINE
            if (kb == kb0) {
              if (ui < 16) TL_SET(8 + ui, clock64());
            }
#endif
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k)
              umma_bf16_cg2(d_tmem, ad + k * a_step4, bd + k * b_step4, idesc,
                            (kb > kb0 || k > 0) ? 1u : 0u);
            // slot free once these MMAs retire (every sharing pair's CTAs; MC 5: own pair)
            umma_commit_cg2_mc(&empty[stage], MC == 5 ? pair_mask : kAllMask);
          }
          __syncwarp();
          if (++stage == P::Stages) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (elect_one()) umma_commit_cg2_mc(&tfull[acc], pair_mask);  // accumulator ready
#if TP_TIMELINE
        if (lane == 0 && ui < 16) TL_SET(24 + ui, clock64());
#endif
        __syncwarp();
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
      if (G.trace && lane == 0) {
        G.trace[blockIdx.x * 16 + 2] = t_full;
        G.trace[blockIdx.x * 16 + 3] = t_temp;
        G.trace[blockIdx.x * 16 + 4] = clock64() - t_begin;
        G.trace[blockIdx.x * 16 + 12] = t_first;
        G.trace[blockIdx.x * 16 + 13] = t_steady;
        G.trace[blockIdx.x * 16 + 14] = n_steady;
      }
    }
  } else {
    // ===== epilogue warps 2..9 (both CTAs): TMEM lane quadrant = warp % 4; the two warps of a
    // quadrant take the two halves of the tile's columns (`half`) =====
    const int quad = warp & 3;
    const int half = (warp - 2) / 4;
#if TP_TIMELINE
    unsigned long long tacc[8] = {0, 0, 0, 0, 0, 0, 0, 0};  // epilogue phase sums (warp 2)
    unsigned long long t_saw = 0, t_loop_end = 0;
#endif
    constexpr int kHalves = EW / 4;
    constexpr int kSub64 = BNP / 64, kSub32 = BNP / 32;  // column sub-chunks per tile
    const int s64_0 = half * (kSub64 / kHalves), s64_1 = s64_0 + kSub64 / kHalves;
    const int s32_0 = half * (kSub32 / kHalves), s32_1 = s32_0 + kSub32 / kHalves;
    uint8_t* stg = sOut + (warp - 2) * 2 * kOutBytes;
    int nbox = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    uint32_t rx_round = 0;  // MC 5: DSMEM chunk rounds so far (both pairs count alike)
    unsigned long long t_tf = 0, t_begin = clock64();
    unsigned long long t_pub = 0, t_xwait = 0;  // split exchange: publish / sibling-wait cycles
    for (int ui = 0; ui < nu; ++ui) {
        const int u = unit_at_s(sched, ulist, cid, ncl, ui);
      const Unit t = unit_of<MC>(sp, nprob, raster, u, pair);
      const ProbS& pr = sp[t.prob];
      const Prob& pm = G.p[t.prob];
      const int64_t rloc = static_cast<int64_t>(rank) * kBM + quad * 32;  // row within pair tile
      const int64_t row0 = static_cast<int64_t>(t.mb) * 256 + rloc;       // first row of warp
      const int64_t row = row0 + lane;
      const int64_t n0 = static_cast<int64_t>(t.nb) * BNP;
      {
        // one lane polls, the rest park at the warp barrier: 4 warps x 32 lanes spinning on
        // try_wait for the whole main loop would contend with the TMA/MMA smem traffic
        const unsigned long long t0 = clock64();
        if (lane == 0) mbar_wait_sleep(&tfull[acc], acc_phase, 200);
        __syncwarp();
        t_tf += clock64() - t0;
#if TP_TIMELINE
        if (warp == 2 && lane == 0 && ui < 16) TL_SET(40 + ui, clock64());
        t_saw = clock64();
#endif
      }
      tc_fence_after();
      const uint32_t t_row = tmem_base + (static_cast<uint32_t>(quad * 32) << 16) +
                             static_cast<uint32_t>(acc * BNP);
      if (MC == 5) {
        // ---- K-split pair: pair 1 streams its accumulator into pair 0's smem (DSMEM), pair 0
        // adds it in column chunks of 64 (two 32-column buffers) and stores the tile (the
        // first four epilogue warps; the other four only release TMEM)
        const uint32_t peer = crank ^ 2u;  // same rank, other pair
        const int rrow = quad * 32 + lane;
        if (half == 1) {
          // nothing: the round protocol below runs on one warp per lane quadrant
        } else if (pair == 1) {
          // sender: TMEM -> own staging (conflict-free [col][row]) -> one bulk copy per 32-col
          // chunk into the owner's buffer, completing as tx bytes on the owner's rxf
#pragma unroll 1
          for (int k = 0; k < BNP / 64; ++k, ++rx_round) {
            mbar_wait_cluster(&rxe[0], (rx_round & 1) ^ 1);  // owner done with the last round
            mbar_wait_cluster(&rxe[1], (rx_round & 1) ^ 1);
            uint32_t r0[32], r1[32];
            tmem_ld32(t_row + k * 64, r0);
            tmem_ld32(t_row + k * 64 + 32, r1);
            tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < 32; ++j) {
              rx[j * kBM + rrow] = __uint_as_float(r0[j]);
              rx[(32 + j) * kBM + rrow] = __uint_as_float(r1[j]);
            }
            fence_proxy_async_smem();
            named_barrier_sync(2, 128);  // the four working epilogue warps
            if (threadIdx.x == 64) {
              const uint32_t src = smem_u32(rx);
              bulk_s2s(mapa(src, peer), src, 32 * kBM * 4, mapa(smem_u32(&rxf[0]), peer));
              bulk_s2s(mapa(src + 32 * kBM * 4, peer), src + 32 * kBM * 4, 32 * kBM * 4,
                       mapa(smem_u32(&rxf[1]), peer));
            }
          }
        } else {
#pragma unroll 1
          for (int k = 0; k < BNP / 64; ++k, ++rx_round) {
            if (threadIdx.x == 64) {  // this round's two chunks: 16 KB each
              mbar_expect_tx(&rxf[0], 32 * kBM * 4);
              mbar_expect_tx(&rxf[1], 32 * kBM * 4);
            }
            float v[64];
            tmem_cols<64>(t_row, k, v);
            mbar_wait(&rxf[0], rx_round & 1);
            mbar_wait(&rxf[1], rx_round & 1);
            const float* q0 = rx + rrow;
#pragma unroll
            for (int j = 0; j < 64; ++j) v[j] += q0[j * kBM];
            __syncwarp();
            if (lane == 0) {
              mbar_arrive_cluster(&rxe[0], peer);
              mbar_arrive_cluster(&rxe[1], peer);
            }
            if (pr.out_bf16) {
              store_box<64>(pr, pm.tmD, stg, nbox, lane, v, row, n0 + k * 64, row0);
            } else {
              float lo[32], hi[32];
#pragma unroll
              for (int j = 0; j < 32; ++j) {
                lo[j] = v[j];
                hi[j] = v[32 + j];
              }
              store_box<32>(pr, pm.tmD, stg, nbox, lane, lo, row, n0 + k * 64, row0);
              store_box<32>(pr, pm.tmD, stg, nbox, lane, hi, row, n0 + k * 64 + 32, row0);
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(&tempty[acc], lead);
      } else if (pr.splits == 1) {
        // a narrow tile holds BNP/2 accumulator columns (the rest of the buffer is stale)
        const bool nar = MC == 1 && BNP == 256 && t.nb == pr.narrow_nb;
#if TP_TIMELINE
        tacc[4] += clock64() - t_saw;
#endif
        if (pr.out_bf16) {
#pragma unroll 1
          for (int sub = s64_0; sub < (nar ? min(s64_1, kSub64 / 2) : s64_1); ++sub) {
            float v[64];
#if TP_TIMELINE
            const unsigned long long c0 = clock64();
#endif
            tmem_cols<64>(t_row, sub, v);
#if TP_TIMELINE
            tacc[0] += clock64() - c0;
#endif
            store_box<64>(pr, pm.tmD, stg, nbox, lane, v, row, n0 + sub * 64, row0,
#if TP_TIMELINE
                          warp == 2 ? tacc : nullptr,
#else
                          nullptr,
#endif
                          G.epi_diag);
          }
#if TP_TIMELINE
          t_loop_end = clock64();
#endif
        } else {
#pragma unroll 1
          for (int sub = s32_0; sub < (nar ? min(s32_1, kSub32 / 2) : s32_1); ++sub) {
            float v[32];
            tmem_cols<32>(t_row, sub, v);
            store_box<32>(pr, pm.tmD, stg, nbox, lane, v, row, n0 + sub * 32, row0);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(&tempty[acc], lead);
#if TP_TIMELINE
        if (warp == 2 && lane == 0 && ui < 16) TL_SET(56 + ui, clock64());
        tacc[6] += clock64() - t_loop_end;
#endif
      } else if (EW == 4 && pr.owner_wait && pr.splits == 2) {
        // ---- split-K of two, co-resident, reduce-scatter style: split s keeps the columns
        // [s BNP/2, (s+1) BNP/2) of the tile. Each split publishes its fp32 partial of the OTHER
        // half, then adds its sibling's partial of its own half and stores it: both CTAs of the
        // tile move half the bytes at the same time instead of one writing all and the other
        // reading all. acc + partial is the same sum as split 0 + split 1 (fp add commutes).
        const int tile = t.ptile;
        const int me = t.split, other = 1 - t.split;
        float4* part_me = reinterpret_cast<float4*>(pr.part + (int64_t(tile) * 2 + me) * P::TileElems +
                                                    rank * (kBM * BNP)) + quad * 32 + lane;
        const float4* part_ot = reinterpret_cast<const float4*>(pr.part + (int64_t(tile) * 2 + other) * P::TileElems +
                                                                rank * (kBM * BNP)) + quad * 32 + lane;
        int* flags = pr.counters + 2 * pr.ptiles + (tile * 2 + rank) * 2;
        constexpr int kHalfChunks = BNP / 64;  // 32-column chunks per half tile
        const unsigned long long tx0 = clock64();
#pragma unroll 1
        for (int ch = other * kHalfChunks; ch < (other + 1) * kHalfChunks; ++ch) {
          uint32_t r0[32];
          tmem_ld32(t_row + ch * 32, r0);
          tmem_wait_ld();
#pragma unroll
          for (int i = 0; i < 8; ++i)
            part_me[(ch * 8 + i) * kBM] =
                make_float4(__uint_as_float(r0[4 * i]), __uint_as_float(r0[4 * i + 1]),
                            __uint_as_float(r0[4 * i + 2]), __uint_as_float(r0[4 * i + 3]));
        }
        fence_acq_rel_gpu();
        named_barrier_sync(1, (EW * 32));
        const unsigned long long tx1 = clock64();
        t_pub += tx1 - tx0;
        if (threadIdx.x == 64) {
          atomicAdd(&flags[me], 1);
          volatile int* f = &flags[other];
          while (*f < 1) __nanosleep(32);
          *f = 0;  // ready for the next launch
          fence_acq_rel_gpu();
        }
        named_barrier_sync(1, (EW * 32));
        t_xwait += clock64() - tx1;
        if (pr.out_bf16) {
#pragma unroll 1
          for (int sub = me * (BNP / 128); sub < (me + 1) * (BNP / 128); ++sub) {
            float v[64];
            tmem_cols<64>(t_row, sub, v);
            const float4* q = part_ot + (sub * 16) * kBM;
            float4 x[16];
#pragma unroll
            for (int i = 0; i < 16; ++i) x[i] = __ldcg(q + i * kBM);
#pragma unroll
            for (int i = 0; i < 16; ++i) {
              v[4 * i] += x[i].x;
              v[4 * i + 1] += x[i].y;
              v[4 * i + 2] += x[i].z;
              v[4 * i + 3] += x[i].w;
            }
            store_box<64>(pr, pm.tmD, stg, nbox, lane, v, row, n0 + sub * 64, row0);
          }
        } else {
#pragma unroll 1
          for (int ch = me * kHalfChunks; ch < (me + 1) * kHalfChunks; ++ch) {
            float v[32];
            tmem_cols<32>(t_row, ch, v);
            const float4* q = part_ot + (ch * 8) * kBM;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const float4 x = __ldcg(q + i * kBM);
              v[4 * i] += x.x;
              v[4 * i + 1] += x.y;
              v[4 * i + 2] += x.z;
              v[4 * i + 3] += x.w;
            }
            store_box<32>(pr, pm.tmD, stg, nbox, lane, v, row, n0 + ch * 32, row0);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(&tempty[acc], lead);
      } else if (pr.owner_wait && t.split == 0) {
        // ---- split-K, owner: every split is co-resident (one unit per cluster), so split 0
        // keeps its accumulator in TMEM, waits for the other splits' partials and adds them
        // in split order (deterministic), then stores the tile
        const int tile = t.ptile;
        const float4* base =
            reinterpret_cast<const float4*>(pr.part + static_cast<int64_t>(tile) * pr.splits * P::TileElems +
                                            rank * (kBM * BNP)) +
            quad * 32 + lane;
        constexpr int kSplitStride4 = P::TileElems / 4;
        if (threadIdx.x == 64) {
          volatile int* cnt = pr.counters + tile * 2 + rank;
          while (*cnt < pr.splits - 1) __nanosleep(64);
          fence_acq_rel_gpu();
          *cnt = 0;  // ready for the next launch
        }
        named_barrier_sync(1, (EW * 32));
        if (pr.out_bf16) {
#pragma unroll 1
          for (int sub = s64_0; sub < s64_1; ++sub) {
            float v[64];
            tmem_cols<64>(t_row, sub, v);
            add_partials<64>(base, pr.splits, kSplitStride4, sub, v);
            store_box<64>(pr, pm.tmD, stg, nbox, lane, v, row, n0 + sub * 64, row0);
          }
        } else {
#pragma unroll 1
          for (int sub = s32_0; sub < s32_1; ++sub) {
            float v[32];
            tmem_cols<32>(t_row, sub, v);
            add_partials<32>(base, pr.splits, kSplitStride4, sub, v);
            store_box<32>(pr, pm.tmD, stg, nbox, lane, v, row, n0 + sub * 32, row0);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(&tempty[acc], lead);
      } else {
        // ---- split-K: publish this split's fp32 partial; with owner_wait split 0 adds it,
        // otherwise the last split to arrive reduces all partials ----
        // partial layout per CTA half: float4 slot f (column/4) major, row minor, so a warp's
        // 32 rows of one slot are 512 contiguous bytes (coalesced store and reload)
        const int tile = t.ptile;
        float4* mypart =
            reinterpret_cast<float4*>(pr.part + static_cast<int64_t>(tile * pr.splits + t.split) *
                                                    P::TileElems +
                                      rank * (kBM * BNP)) +
            quad * 32 + lane;
#pragma unroll 1
        for (int ch = s32_0; ch < s32_1; ++ch) {
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
        if (lane == 0) mbar_arrive_remote(&tempty[acc], lead);  // TMEM free for the next unit
        fence_acq_rel_gpu();
        named_barrier_sync(1, (EW * 32));
        if (pr.owner_wait) {
          if (threadIdx.x == 64) atomicAdd(pr.counters + tile * 2 + rank, 1);
        } else if (threadIdx.x == 64) {
          int* cnt = pr.counters + tile * 2 + rank;
          const int old = atomicAdd(cnt, 1);
          const int last = old == pr.splits - 1;
          if (last) *cnt = 0;  // ready for the next launch
          *sflag = last;
        }
        named_barrier_sync(1, (EW * 32));
        const int last = pr.owner_wait ? 0 : *sflag;
        named_barrier_sync(1, (EW * 32));
        if (last) {
          fence_acq_rel_gpu();
          const float4* base =
              reinterpret_cast<const float4*>(pr.part + static_cast<int64_t>(tile) * pr.splits * P::TileElems +
                                              rank * (kBM * BNP)) +
              quad * 32 + lane;
          constexpr int kSplitStride4 = P::TileElems / 4;
          if (pr.out_bf16) {
#pragma unroll 1
            for (int sub = s64_0; sub < s64_1; ++sub) {
              float v[64];
              sum_partials<64>(base, pr.splits, kSplitStride4, sub, v);
              store_box<64>(pr, pm.tmD, stg, nbox, lane, v, row, n0 + sub * 64, row0);
            }
          } else {
#pragma unroll 1
            for (int sub = s32_0; sub < s32_1; ++sub) {
              float v[32];
              sum_partials<32>(base, pr.splits, kSplitStride4, sub, v);
              store_box<32>(pr, pm.tmD, stg, nbox, lane, v, row, n0 + sub * 32, row0);
            }
          }
        }
      }
      if (++acc == 2) {
        acc = 0;
        acc_phase ^= 1;
      }
    }
    // staging buffers must outlive the bulk stores' smem reads; the global writes complete with
    // the grid (as CUTLASS's store tail: wait_group.read, not a full-completion wait)
    if (lane == 0) bulk_wait_read0();
#if TP_TIMELINE
    if (warp == 2 && lane == 0 && tl)
      for (int i = 0; i < 7; ++i) tl[72 + i] = tacc[i];
#endif
    if (G.trace && warp == 2 && lane == 0) {
      G.trace[blockIdx.x * 16 + 5] = t_tf;
      G.trace[blockIdx.x * 16 + 15] = (t_xwait << 32) | (t_pub & 0xffffffffull);
      G.trace[blockIdx.x * 16 + 6] = clock64() - t_begin;
    }
  }

  tc_fence_before();
  __syncthreads();  // reconverge every warp (idle lanes park here) before the .aligned barrier
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_cg2(tmem_base, P::TmemCols);
  }
  if (G.trace && threadIdx.x == 0) {
    G.trace[blockIdx.x * 16 + 9] = globaltimer();
    G.trace[blockIdx.x * 16 + 11] = clock64();
    TL_SET(2, clock64());
  }
}

// ------------------------------------------------------------------ wide pair tiles (512 x 256)
// For the large products (C3-HEAD, C5: the per-rank GEMMs of the north-star configurations),
// which run at the 1 kW power cap: a CTA pair computes a 512 x 256 tile. Each CTA stages 256 rows
// of A and 128 columns of B per k-block, and the leader issues TWO M=256 N=256 MMAs per K step
// (A rows 0-127 and 128-255 of both CTAs) into the two 256-column halves of the 512-column TMEM,
// so every B k-block serves 512 rows: 25% fewer L2 -> SM bytes per flop than the 256 x 256 pair
// tile, and bigger tiles mean fewer distinct operand panels per wave (less DRAM traffic), i.e.
// less energy per flop - the currency at the power cap (profiles/r02_ncu_gemm_shapes.md).
// Single TMEM accumulator: the epilogue (4 warps per CTA, both row halves) drains it before the
// next unit's first MMA. No split-K, no K-panels / D row-panels (the caller checks).
constexpr int kWStages = 4;
constexpr int kWABytes = 2 * kBM * kBK * 2;  // 256 rows x 64 k
constexpr int kWBBytes = 128 * kBK * 2;      // 128 columns x 64 k (half of the pair's 256)
constexpr int kWStageBytes = kWABytes + kWBBytes;
constexpr int kWSmem = kWStages * kWStageBytes + 2 * 4 * kOutBytes + 1024 + 256;

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(threads_of<4>(), 1)
    gemm_tc2w_kernel(const __grid_constant__ Group G) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sA = smem;
  uint8_t* sB = sA + kWStages * kWABytes;
  uint8_t* sOut = sB + kWStages * kWBBytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sOut + 2 * 4 * kOutBytes);
  uint64_t* empty = full + kWStages;
  uint64_t* tfull = empty + kWStages;
  uint64_t* tempty = tfull + 1;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 1);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = cluster_rank() & 1;
  const bool leader = rank == 0;
  const int cid = blockIdx.x / 2, ncl = gridDim.x / 2;

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < G.nprob; ++i) {
      tma_prefetch(&G.p[i].tmA[0]);
      tma_prefetch(&G.p[i].tmB[0]);
      tma_prefetch(&G.p[i].tmD[0]);
    }
    for (int s = 0; s < kWStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(tfull, 1);
    mbar_init(tempty, 2 * 4);  // 4 epilogue warps x 2 CTAs
    fence_barrier_init();
  }
  if (warp == 1) tmem_alloc_cg2(tslot, 512);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tslot;
  pdl_launch_dependents();
  pdl_wait();

  auto unit_prob = [&](int u, int& lu) {
    int pi = 0;
#pragma unroll
    for (int i = 1; i < kMaxProbs; ++i)
      if (i < G.nprob && u >= G.p[i].unit0) pi = i;
    lu = u - G.p[pi].unit0;
    return pi;
  };

  if (warp == 0) {
    // ===== TMA producer (both CTAs; bytes land on the leader's `full`) =====
    int stage = 0;
    uint32_t phase = 0;
    for (int u = cid; u < G.total_units; u += ncl) {
      int lu;
      const Prob& pr = G.p[unit_prob(u, lu)];
      int mb, nb;
      tile_coords(lu, pr.num_m, pr.num_n, mb, nb, G.raster);
      const int m0 = mb * 512 + static_cast<int>(rank) * 256;
      const int n0 = nb * 256 + static_cast<int>(rank) * 128;
      const bool a_mn = pr.a_mn != 0, b_mn = pr.b_mn != 0;
      const CUtensorMap* mA = &pr.tmA[0];
      const CUtensorMap* mB = &pr.tmB[0];
      for (int kb = 0; kb < pr.num_kb; ++kb) {
        const int kc = kb * kBK;
        mbar_wait(&empty[stage], phase ^ 1);
        if (elect_one()) {
          if (leader) mbar_expect_tx(&full[stage], 2 * kWStageBytes);
          uint8_t* a_dst = sA + stage * kWABytes;
          uint8_t* b_dst = sB + stage * kWBBytes;
          if (!a_mn) {
            tma_load_2d_pair(mA, &full[stage], a_dst, kc, m0);  // one [256 rows][128 B] box
          } else {
            for (int c = 0; c < 4; ++c)
              tma_load_2d_pair(mA, &full[stage], a_dst + c * (kBK * 128), m0 + c * 64, kc);
          }
          if (!b_mn) {
            tma_load_2d_pair(mB, &full[stage], b_dst, kc, n0);
          } else {
            for (int c = 0; c < 2; ++c)
              tma_load_2d_pair(mB, &full[stage], b_dst + c * (kBK * 128), n0 + c * 64, kc);
          }
        }
        __syncwarp();
        if (++stage == kWStages) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    if (leader) {
      // ===== MMA issuer: two M=256 N=256 MMAs per K step (row halves 0 / 1 of each CTA) =====
      int stage = 0;
      uint32_t phase = 0, acc_phase = 0;
      for (int u = cid; u < G.total_units; u += ncl) {
        int lu;
        const Prob& pr = G.p[unit_prob(u, lu)];
        const uint32_t idesc = idesc_bf16_f32(256, 256, pr.a_mn != 0, pr.b_mn != 0);
        const uint32_t a_step4 = pr.a_mn ? 2048u / 16 : 32u / 16;
        const uint32_t b_step4 = pr.b_mn ? 2048u / 16 : 32u / 16;
        // second row half: +128 rows x 128 B (K-major) = +2 MN chunks of 64 x 128 B (MN-major)
        constexpr uint32_t a_half4 = (kBM * 128) / 16;
        const uint64_t a_desc0 = sdesc_sw128(smem_u32(sA), pr.a_mn ? kBK * 128 : 16, 1024);
        const uint64_t b_desc0 = sdesc_sw128(smem_u32(sB), pr.b_mn ? kBK * 128 : 16, 1024);
        mbar_wait(tempty, acc_phase ^ 1);  // the epilogue drained the previous unit
        __syncwarp();
        tc_fence_after();
        for (int kb = 0; kb < pr.num_kb; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t ad = a_desc0 + static_cast<uint32_t>(stage * (kWABytes / 16));
          const uint64_t bd = b_desc0 + static_cast<uint32_t>(stage * (kWBBytes / 16));
          if (elect_one()) {
#pragma unroll
            for (int k = 0; k < kBK / 16; ++k) {
              const uint32_t acc = (kb > 0 || k > 0) ? 1u : 0u;
              umma_bf16_cg2(tmem_base, ad + k * a_step4, bd + k * b_step4, idesc, acc);
              umma_bf16_cg2(tmem_base + 256, ad + a_half4 + k * a_step4, bd + k * b_step4, idesc, acc);
            }
            umma_commit_cg2_mc(&empty[stage], 0x3);
          }
          __syncwarp();
          if (++stage == kWStages) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (elect_one()) umma_commit_cg2_mc(tfull, 0x3);
        __syncwarp();
        acc_phase ^= 1;
      }
    }
  } else {
    // ===== epilogue warps 2..5 (both CTAs): lane quadrant warp % 4, both row halves =====
    const int quad = warp & 3;
    uint8_t* stg = sOut + (warp - 2) * 2 * kOutBytes;
    int nbox = 0;
    uint32_t acc_phase = 0;
    for (int u = cid; u < G.total_units; u += ncl) {
      int lu;
      const Prob& pr = G.p[unit_prob(u, lu)];
      int mb, nb;
      tile_coords(lu, pr.num_m, pr.num_n, mb, nb, G.raster);
      const int64_t n0 = static_cast<int64_t>(nb) * 256;
      if (lane == 0) mbar_wait_sleep(tfull, acc_phase, 200);
      __syncwarp();
      tc_fence_after();
#pragma unroll 1
      for (int h = 0; h < 2; ++h) {
        const int64_t row0 = static_cast<int64_t>(mb) * 512 + rank * 256 + h * 128 + quad * 32;
        const int64_t row = row0 + lane;
        const uint32_t t_row = tmem_base + (static_cast<uint32_t>(quad * 32) << 16) +
                               static_cast<uint32_t>(h * 256);
        if (pr.out_bf16) {
#pragma unroll 1
          for (int sub = 0; sub < 4; ++sub) {
            float v[64];
            tmem_cols<64>(t_row, sub, v);
            store_box<64>(pr, pr.tmD, stg, nbox, lane, v, row, n0 + sub * 64, row0);
          }
        } else {
#pragma unroll 1
          for (int sub = 0; sub < 8; ++sub) {
            float v[32];
            tmem_cols<32>(t_row, sub, v);
            store_box<32>(pr, pr.tmD, stg, nbox, lane, v, row, n0 + sub * 32, row0);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(tempty, 0);
      acc_phase ^= 1;
    }
    if (lane == 0) bulk_wait_read0();
  }

  tc_fence_before();
  __syncthreads();
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc_cg2(tmem_base, 512);
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

// L2 sector promotion of the operand loads (TP_GEMM_L2PROMO: 0 none, 1 64 B, 2 128 B, 3 256 B)
CUtensorMapL2promotion l2_promotion() {
  switch (knob("TP_GEMM_L2PROMO")) {
    case 0: return CU_TENSOR_MAP_L2_PROMOTION_NONE;
    case 1: return CU_TENSOR_MAP_L2_PROMOTION_L2_64B;
    case 2: return CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
    default: return CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  }
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
                  l2_promotion(), CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
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

// Max co-resident clusters of a kernel (clusters of 4 may strand SMs on some GPCs).
template <typename Kern>
int max_clusters(Kern kern, int csize, int smem, int threads) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(csize * 64);
  cfg.blockDim = dim3(threads);
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

// Fill one problem's maps, epilogue params and its split-K choice.
template <int BNP, int MC>
tp_status setup_prob(const GemmArgs& g, Prob& pr, int clusters, int split_mode, char*& ws,
                     size_t& ws_left, cudaStream_t s) {
  using P = PC<BNP, MC>;
  const auto BF = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  pr.a_mn = g.trans_a ? 1 : 0;
  pr.b_mn = g.trans_b ? 0 : 1;
  pr.narrow_nb = -1;
  // multicast halves: MC 2 loads half of the A rows per pair, MC 3 half of the B tile
  pr.npanels = g.npanels > 1 ? g.npanels : 1;
  if (pr.npanels > kMaxPanels) return fail(TP_ERR_UNSUPPORTED, "gemm: more than 4 K-panels");
  for (int k = 0; k < pr.npanels; ++k) {
    const void* A = pr.npanels > 1 ? g.Ap[k] : g.A;
    const void* B = pr.npanels > 1 ? g.Bp[k] : g.B;
    pr.a_box64 = (!mc_a(MC) && !pr.a_mn && knob("TP_GEMM_ABOX64")) ? 1 : 0;
    if (!pr.a_mn)
      TP_TRY(make_map2(&pr.tmA[k], BF, 2, A, g.K, g.M, g.lda, kBK,
                       (mc_a(MC) || pr.a_box64) ? kBM / 2 : kBM));
    else
      TP_TRY(make_map2(&pr.tmA[k], BF, 2, A, g.M, g.K, g.lda, 64, kBK));
    if (!pr.b_mn)
      TP_TRY(make_map2(&pr.tmB[k], BF, 2, B, g.K, g.N, g.ldb, kBK, mc_b(MC) ? P::BNC / 2 : P::BNC));
    else
      TP_TRY(make_map2(&pr.tmB[k], BF, 2, B, g.N, g.K, g.ldb, 64,
                       (mc_b(MC) && P::BNC < 128) ? kBK / 2 : kBK));
  }
  pr.kb_panel = static_cast<int>((g.K + kBK - 1) / kBK);
  pr.num_kb = pr.kb_panel * pr.npanels;
  const int dp = g.dpanels > 1 ? g.dpanels : 1;
  if (dp > kMaxDPanels) return fail(TP_ERR_UNSUPPORTED, "gemm: more than 8 D row-panels");
  pr.d_rows = dp > 1 ? static_cast<int>(g.d_rows) : 0;
  for (int i = 0; i < dp; ++i) {
    void* D = dp > 1 ? g.Dp[i] : g.D;
    const uint64_t rows = dp > 1 ? uint64_t(g.d_rows) : uint64_t(g.M);
    if (g.out_dtype == TP_BF16)
      TP_TRY(make_map2(&pr.tmD[i], BF, 2, D, g.N, rows, g.ldd, 64, 32));
    else
      TP_TRY(make_map2(&pr.tmD[i], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, D, g.N, rows, g.ldd, 32, 32));
  }
  pr.C = g.C;
  pr.bias = g.bias;
  pr.ldc = g.ldc;
  pr.alpha = g.alpha;
  pr.out_bf16 = g.out_dtype == TP_BF16;
  pr.M = static_cast<int>(g.M);
  pr.N = static_cast<int>(g.N);
  pr.K = static_cast<int>(g.K);
  pr.num_m = static_cast<int>((g.M + 255) / 256);
  pr.num_n = static_cast<int>((g.N + BNP - 1) / BNP);
  pr.c_vec = !g.C || ((reinterpret_cast<uintptr_t>(g.C) % 16 == 0) && (g.ldc % 4 == 0));
  pr.part = nullptr;
  pr.counters = nullptr;
  pr.owner_wait = 0;
  const int supers = super_tiles(MC, pr.num_m, pr.num_n);
  const int ptiles = supers * pairs_of(MC);
  const int num_k = pr.num_kb;
  int S = 1;
  const int env_split = knob("TP_GEMM_SPLITK");
  // split_mode > 0: a single problem -- split K only when the grid would leave more than half
  // of the clusters idle (up to 16 ways, every split >= 4 k-blocks). split_mode < 0: a problem
  // of a group whose tiles are far longer than the group's per-cluster share of work
  // (-split_mode = that share in k-blocks): split so no unit exceeds ~ the share.
  // counters: per pair tile 2 ints (per CTA of the pair) + 4 flags (CTA x split, exchange path)
  const size_t cbytes = 256 * ((size_t(ptiles) * 24 + 255) / 256);
  const auto need_of = [&](int sp) { return size_t(ptiles) * sp * P::TileElems * 4 + cbytes; };
  if (split_mode > 0 && env_split) {
    for (int sp = 2; sp <= 16; ++sp)
      if (2 * supers <= clusters && supers * sp <= clusters && num_k >= 4 * sp && need_of(sp) <= ws_left)
        S = sp;
  } else if (split_mode < 0 && env_split) {
    const int share = -split_mode;
    const int want = std::min(16, (num_k + share - 1) / share);
    for (int sp = want; sp >= 2; --sp)
      if (supers * sp <= clusters && num_k >= 4 * sp && need_of(sp) <= ws_left) {
        S = sp;
        break;
      }
  }
  if (MC == 5) {  // the cluster's two pairs split K in halves; no global split-K
    if (num_k < 2) return fail(TP_ERR_UNSUPPORTED, "gemm: K-split pair cluster needs >= 2 k-blocks");
    pr.splits = 1;
    pr.kb_per_split = (num_k + 1) / 2;
    return TP_OK;
  }
  int kbps = (num_k + S - 1) / S;
  S = (num_k + kbps - 1) / kbps;  // no empty split
  if (S < 1) S = 1;
  pr.splits = S;
  pr.kb_per_split = S > 1 ? kbps : num_k;
  // half-width last n-tile (single pass only: the split-K paths move whole tiles); K-major B
  // loads it through a 64-row box map in the free second panel slot
  pr.narrow_nb = -1;
  const int64_t n_tail = g.N % BNP;
  if (MC == 1 && BNP == 256 && S == 1 && pr.npanels == 1 && n_tail > 0 && n_tail <= BNP / 2 &&
      knob("TP_GEMM_NARROW")) {
    pr.narrow_nb = pr.num_n - 1;
    if (!pr.b_mn) TP_TRY(make_map2(&pr.tmB[1], BF, 2, g.B, g.K, g.N, g.ldb, kBK, P::BNC / 2));
  }
  if (S > 1) {
    pr.counters = reinterpret_cast<int*>(ws);
    pr.ptiles = ptiles;
    pr.part = reinterpret_cast<float*>(ws + cbytes);
    const size_t used = cbytes + size_t(ptiles) * S * P::TileElems * 4;
    ws += used;
    ws_left -= used;
    TP_CUDA(cudaMemsetAsync(pr.counters, 0, cbytes, s));
  }
  return TP_OK;
}

// Longest-processing-time assignment of units to clusters when their lengths differ (a group
// whose members have different K, e.g. the C2 backward: 32 dX tiles of 64 k-blocks next to 256
// dW tiles of 8; round robin gave the first 32 clusters 88 k-blocks against a mean of 55).
// Unit cost = k-blocks x the measured clocks of one pair k-block (576 at 256 columns: the SM's
// operand ingress, not the 512-clock MMA, paces it) + a per-unit turnaround (TP_GEMM_SCHED_EPI
// clocks: the next unit's first k-block arriving, the exposed epilogue share; tools/
// gemm_timeline.py measured ~6.2K clocks per 8-k-block dW unit in the C2 group). Units longest
// first, each to the least-loaded cluster; a cluster runs its units in the order assigned.
template <int BNP>
void schedule_units(Group& G, int ncl) {
  const int units = G.total_units;
  if (!knob("TP_GEMM_SCHED") || ncl <= 0 || ncl > kMaxSchedClusters || units <= ncl ||
      units > kMaxSchedUnits)
    return;
  std::vector<int64_t> cost(units);
  int64_t cmin = INT64_MAX, cmax = 0;
  const int64_t epi = knob("TP_GEMM_SCHED_EPI");
  for (int i = 0; i < G.nprob; ++i) {
    const Prob& pr = G.p[i];
    if (pr.splits != 1) return;  // split-K units keep their co-residency rules
    const int nu = pr.num_m * pr.num_n;
    for (int t = 0; t < nu; ++t) {
      const int64_t c = int64_t(pr.num_kb) * 576 * BNP / 256 + epi;
      cost[pr.unit0 + t] = c;
      cmin = std::min(cmin, c);
      cmax = std::max(cmax, c);
    }
  }
  if (cmin == cmax) return;  // uniform units: round robin is already balanced
  // units in order of decreasing cost (stable), each to the least-loaded cluster (min-heap of
  // (load, cluster): ties go to the lower cluster index); host cost O(units log clusters)
  std::vector<int> ord(units);
  for (int u = 0; u < units; ++u) ord[u] = u;
  std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return cost[a] > cost[b]; });
  using LC = std::pair<int64_t, int>;
  std::priority_queue<LC, std::vector<LC>, std::greater<LC>> heap;
  for (int c = 0; c < ncl; ++c) heap.push(LC(0, c));
  std::vector<int> owner(units), count(ncl, 0);
  for (int u : ord) {
    LC top = heap.top();
    heap.pop();
    owner[u] = top.second;
    if (++count[top.second] > kMaxClusterUnits) return;
    top.first += cost[u];
    heap.push(top);
  }
  // per-cluster lists in assignment order (counting sort over the cost order)
  std::vector<int> pos(ncl + 1, 0);
  for (int c = 0; c < ncl; ++c) pos[c + 1] = pos[c] + count[c];
  for (int c = 0; c <= ncl; ++c) G.sched_start[c] = static_cast<uint16_t>(pos[c]);
  for (int u : ord) G.sched_order[pos[owner[u]]++] = static_cast<uint16_t>(u);
  G.sched = 1;
}

template <int BNP, int MC, int EW = 4>
tp_status launch2(const GemmArgs* gs, int n, cudaStream_t s) {
  using P = PC<BNP, MC, EW>;
  auto kern = gemm_tc2_kernel<BNP, MC, EW>;
  static int clusters_of[64] = {};  // co-resident clusters, per device
  int dev = 0;
  TP_CUDA(cudaGetDevice(&dev));
  int clusters = 0;
  {
    static std::mutex mu;
    std::lock_guard<std::mutex> lk(mu);
    int& c = clusters_of[dev & 63];
    if (!c) {
      TP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, P::Smem));
      c = max_clusters(kern, 2 * pairs_of(MC), P::Smem, threads_of<EW>());
    }
    clusters = c;
  }
  const int env_raster = std::max(1, knob("TP_GEMM_RASTER"));
  Group G;
  G.nprob = n;
  G.raster = env_raster;
  G.trace = g_gemm_trace;
  char* ws = static_cast<char*>(gs[0].ws);
  size_t ws_left = ws ? gs[0].ws_bytes : 0;
  int units = 0;
  double flops = 0;
  for (int i = 0; i < n; ++i) {
    // no split-K inside a group: measured slower (the partial round trip outweighs the balance
    // gain on the C2 backward, 0.135 vs 0.126 ms/step)
    const int group_split = knob("TP_GEMM_GROUP_SPLIT");
    int mode = n == 1 ? 1 : 0;
    if (n > 1 && group_split) {
      // per-cluster share of the group's work (tiles x k-blocks); a problem whose tiles are
      // more than twice as long is split (e.g. a long-K dW next to many short dX tiles)
      double work = 0;
      for (int j = 0; j < n; ++j) {
        const double tiles = double((gs[j].M + 255) / 256) * double((gs[j].N + BNP - 1) / BNP);
        const double kb = double((gs[j].K + kBK - 1) / kBK) * (gs[j].npanels > 1 ? gs[j].npanels : 1);
        work += tiles * kb;
      }
      const double share = work / clusters;
      const double kb_i = double((gs[i].K + kBK - 1) / kBK) * (gs[i].npanels > 1 ? gs[i].npanels : 1);
      if (kb_i > 2 * share && share >= 8) mode = -static_cast<int>(share);
    }
    TP_TRY((setup_prob<BNP, MC>(gs[i], G.p[i], clusters, mode, ws, ws_left, s)));
    G.p[i].unit0 = units;
    units += super_tiles(MC, G.p[i].num_m, G.p[i].num_n) * G.p[i].splits;
    flops += 2.0 * double(gs[i].M) * double(gs[i].N) * double(gs[i].K) * G.p[i].npanels;
  }
  G.total_units = units;
  // persistent grid; when a collective runs concurrently (SUMMA panel broadcast under this
  // GEMM) leave SMs for its kernels, else the NCCL CTAs cannot be resident until we finish
  int cap = clusters;
  if (gs[0].reserve_sms > 0)
    cap = std::max(1, std::min(cap, (sm_count() - gs[0].reserve_sms) / (2 * pairs_of(MC))));
  const int grid = 2 * pairs_of(MC) * (units < cap ? units : cap);
  G.sched = 0;
  if (MC == 1) schedule_units<BNP>(G, grid / 2);
  G.epi_diag = TP_TIMELINE ? knob("TP_GEMM_EPI_DIAG") : 0;
  // split 0 may wait for its sibling splits only when every unit has its own resident cluster
  const int env_owner = knob("TP_GEMM_SPLIT_OWNER");
  for (int i = 0; i < n; ++i)
    G.p[i].owner_wait = (env_owner && g_shared_device_grids.load() == 0 && G.p[i].splits > 1 &&
                         units <= grid / (2 * pairs_of(MC))) ? 1 : 0;
  const int tok = prof_begin(0, s, flops);
  TP_CUDA(launch_pdl(kern, dim3(grid), dim3(threads_of<EW>()), P::Smem, s, G));
  count_launch();
  prof_end(tok, s);
  TP_CUDA(cudaGetLastError());
  return TP_OK;
}

}  // namespace

// ---- wide pair tiles (gemm_tc2w_kernel): up to kMaxProbs problems, no split-K / panels
bool gemm_wide_ok(const GemmArgs& g) {
  return g.npanels <= 1 && g.dpanels <= 1 && g.K > 0 && gemm_tc2_supported(g);
}

tp_status launch_wide(const GemmArgs* gs, int n, cudaStream_t s) {
  if (n < 1 || n > kMaxProbs) return fail(TP_ERR_UNSUPPORTED, "wide gemm: 1..4 problems");
  auto kern = gemm_tc2w_kernel;
  static int clusters_of[64] = {};
  int dev = 0;
  TP_CUDA(cudaGetDevice(&dev));
  int clusters = 0;
  {
    static std::mutex mu;
    std::lock_guard<std::mutex> lk(mu);
    int& c = clusters_of[dev & 63];
    if (!c) {
      TP_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kWSmem));
      c = max_clusters(kern, 2, kWSmem, threads_of<4>());
    }
    clusters = c;
  }
  const int env_raster = std::max(1, knob("TP_GEMM_WIDE_RASTER"));
  Group G;
  G.nprob = n;
  G.raster = env_raster;
  G.trace = nullptr;
  G.sched = 0;
  G.epi_diag = 0;
  const auto BF = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  int units = 0;
  double flops = 0;
  for (int i = 0; i < n; ++i) {
    const GemmArgs& g = gs[i];
    Prob& pr = G.p[i];
    pr.a_mn = g.trans_a ? 1 : 0;
    pr.b_mn = g.trans_b ? 0 : 1;
    if (!pr.a_mn) TP_TRY(make_map2(&pr.tmA[0], BF, 2, g.A, g.K, g.M, g.lda, kBK, 2 * kBM));
    else TP_TRY(make_map2(&pr.tmA[0], BF, 2, g.A, g.M, g.K, g.lda, 64, kBK));
    if (!pr.b_mn) TP_TRY(make_map2(&pr.tmB[0], BF, 2, g.B, g.K, g.N, g.ldb, kBK, 128));
    else TP_TRY(make_map2(&pr.tmB[0], BF, 2, g.B, g.N, g.K, g.ldb, 64, kBK));
    if (g.out_dtype == TP_BF16)
      TP_TRY(make_map2(&pr.tmD[0], BF, 2, g.D, g.N, g.M, g.ldd, 64, 32));
    else
      TP_TRY(make_map2(&pr.tmD[0], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, g.D, g.N, g.M, g.ldd, 32, 32));
    pr.d_rows = 0;
    pr.C = g.C;
    pr.bias = g.bias;
    pr.ldc = g.ldc;
    pr.alpha = g.alpha;
    pr.out_bf16 = g.out_dtype == TP_BF16;
    pr.M = static_cast<int>(g.M);
    pr.N = static_cast<int>(g.N);
    pr.K = static_cast<int>(g.K);
    pr.num_m = static_cast<int>((g.M + 511) / 512);
    pr.num_n = static_cast<int>((g.N + 255) / 256);
    pr.c_vec = !g.C || ((reinterpret_cast<uintptr_t>(g.C) % 16 == 0) && (g.ldc % 4 == 0));
    pr.part = nullptr;
    pr.counters = nullptr;
    pr.owner_wait = 0;
    pr.splits = 1;
    pr.npanels = 1;
    pr.kb_panel = static_cast<int>((g.K + kBK - 1) / kBK);
    pr.num_kb = pr.kb_panel;
    pr.kb_per_split = pr.num_kb;
    pr.ptiles = pr.num_m * pr.num_n;
    pr.narrow_nb = -1;
    pr.a_box64 = 0;
    pr.unit0 = units;
    units += pr.num_m * pr.num_n;
    flops += 2.0 * double(g.M) * double(g.N) * double(g.K);
  }
  G.total_units = units;
  int cap = clusters;
  if (gs[0].reserve_sms > 0) cap = std::max(1, std::min(cap, (sm_count() - gs[0].reserve_sms) / 2));
  const int env_np = knob("TP_GEMM_WIDE_NP");
  if (env_np && gs[0].reserve_sms <= 0) cap = units;
  const int grid = 2 * (units < cap ? units : cap);
  const int tok = prof_begin(0, s, flops);
  TP_CUDA(launch_pdl(kern, dim3(grid), dim3(threads_of<4>()), kWSmem, s, G));
  count_launch();
  prof_end(tok, s);
  TP_CUDA(cudaGetLastError());
  return TP_OK;
}

bool gemm_tc2_supported(const GemmArgs& g) {
  const size_t osz = dtype_size(g.out_dtype);
  if (g.dpanels > 1) {
    if (g.dpanels > kMaxDPanels || g.d_rows % 32 || g.d_rows * g.dpanels < g.M) return false;
    for (int i = 0; i < g.dpanels; ++i)
      if (!g.Dp[i] || reinterpret_cast<uintptr_t>(g.Dp[i]) % 16) return false;
  }
  // TMA-store epilogue only: rows of D must end on a 16-byte granule (a store of the last
  // granule of a ragged row would zero the columns past N, see gemm_sm100.cu)
  return g.M > 128 && (g.dpanels > 1 || reinterpret_cast<uintptr_t>(g.D) % 16 == 0) &&
         ((g.ldd * osz) % 16 == 0) && ((g.N * osz) % 16 == 0) &&
         (!g.bias || reinterpret_cast<uintptr_t>(g.bias) % 2 == 0);
}

size_t gemm_tc2_ws_bytes() {
  // split-K scratch upper bound: pair-tiles*splits <= #SMs/2 (74 on B200, + a ragged super
  // tile), 256x256 fp32 each, plus counters
  return size_t(76) * PC<256>::TileElems * 4 + 4096;
}

// Wide 512 x 256 pair tiles for the big products: two waves of tiles or more and a long K
// (>= 12288: the un-overlapped epilogue of the single TMEM accumulator is then ~1%, and the
// operand panels overflow L2). TP_GEMM_WIDE=0 turns it off (A/B measurements), =1 forces it.
static int wide_mode() {
  const int m = knob("TP_GEMM_WIDE");
  return m;
}

static bool want_wide(const GemmArgs* gs, int n) {
  const int mode = wide_mode();
  if (mode == 0) return false;
  int64_t units = 0, kmin = INT64_MAX;
  for (int i = 0; i < n; ++i) {
    if (!gemm_wide_ok(gs[i])) return false;
    units += ((gs[i].M + 511) / 512) * ((gs[i].N + 255) / 256);
    kmin = std::min<int64_t>(kmin, gs[i].K);
  }
  if (mode == 1) return true;
  // measured (interleaved A/B, profiles/r02_gemm_wide_ab.md): +10% on 16384^3 (NN / NT / TN,
  // = cuBLAS), neutral to -4% on the 8192-class shapes (operand panels mostly L2-resident)
  return units >= sm_count() && kmin >= 12288;
}

tp_status gemm_tc2_bf16(const GemmArgs& g, cudaStream_t s) {
  if (want_wide(&g, 1)) return launch_wide(&g, 1, s);
  // Pair tile 256x256 when those tiles fill the SM pairs, else 256x128 (twice the tiles).
  // TP_GEMM_BN / TP_GEMM_MC force a width / cluster shape (tests, A/B measurements).
  const int force_bn = knob("TP_GEMM_BN");
  const int force_mc = knob("TP_GEMM_MC");
  const int64_t tiles256 = ((g.M + 255) / 256) * ((g.N + 255) / 256);
  const int pairs = sm_count() / 2;
  const bool wide = force_bn ? force_bn == 256 : tiles256 >= pairs;
  const int64_t nrows = (g.M + 255) / 256;
  const int64_t ncols = wide ? (g.N + 255) / 256 : (g.N + 127) / 128;
  const int mc = force_mc ? force_mc : 1;
  const int64_t kblocks = (g.K + kBK - 1) / kBK * (g.npanels > 1 ? g.npanels : 1);
  if (mc == 5 && kblocks >= 2) return force_bn == 128 ? launch2<128, 5>(&g, 1, s) : launch2<256, 5>(&g, 1, s);
  if (wide) {
    if (mc == 4 && ncols >= 2 && nrows >= 2) return launch2<256, 4>(&g, 1, s);
    if (mc == 2 && ncols >= 2) return launch2<256, 2>(&g, 1, s);
    if (mc == 3 && nrows >= 2) return launch2<256, 3>(&g, 1, s);
    // epilogue-bound (1-2 k-blocks per tile, e.g. a dW over 64 tokens): 8 epilogue warps
    const int env_ew = knob("TP_GEMM_EPI_WARPS");
    const bool ew8 = env_ew ? env_ew == 8 : kblocks <= 2;
    if (ew8) return launch2<256, 1, 8>(&g, 1, s);
    return launch2<256, 1>(&g, 1, s);
  }
  if (mc == 4 && ncols >= 2 && nrows >= 2) return launch2<128, 4>(&g, 1, s);
  if (mc == 2 && ncols >= 2) return launch2<128, 2>(&g, 1, s);
  if (mc == 3 && nrows >= 2) return launch2<128, 3>(&g, 1, s);
  if (knob("TP_GEMM_EPI_WARPS") == 8) return launch2<128, 1, 8>(&g, 1, s);
  return launch2<128, 1>(&g, 1, s);
}

bool gemm_tc2_group_splits_member(const GemmArgs* gs, int n) {
  if (!knob("TP_GEMM_GROUP_SPLIT")) return false;  // the group would not split: keep it
  // the per-cluster share launch2<256, 1> computes for a group (tiles x k-blocks / clusters)
  const double clusters = sm_count() / 2;
  double work = 0;
  for (int j = 0; j < n; ++j) {
    const double tiles = double((gs[j].M + 255) / 256) * double((gs[j].N + 255) / 256);
    work += tiles * double((gs[j].K + kBK - 1) / kBK) * (gs[j].npanels > 1 ? gs[j].npanels : 1);
  }
  const double share = work / clusters;
  for (int i = 0; i < n; ++i) {
    const double kb = double((gs[i].K + kBK - 1) / kBK) * (gs[i].npanels > 1 ? gs[i].npanels : 1);
    if (kb > 2 * share && share >= 8) return true;
  }
  return false;
}

// Up to four independent problems in one launch, 256x256 pair tiles; problems with more K
// blocks per tile go first so the round-robin unit assignment front-loads the long units.
tp_status gemm_tc2_group(const GemmArgs* in, int n, cudaStream_t s) {
  if (n < 1 || n > kMaxProbs) return fail(TP_ERR_UNSUPPORTED, "gemm group: 1..4 problems");
  if (want_wide(in, n)) return launch_wide(in, n, s);
  GemmArgs gs[kMaxProbs];
  for (int i = 0; i < n; ++i) gs[i] = in[i];
  auto kblocks = [](const GemmArgs& g) { return g.K * (g.npanels > 1 ? g.npanels : 1); };
  std::stable_sort(gs, gs + n, [&](const GemmArgs& x, const GemmArgs& y) { return kblocks(x) > kblocks(y); });
  const int group_bn = knob("TP_GEMM_GROUP_BN");
  if (group_bn == 128) return launch2<128, 1>(gs, n, s);
  return launch2<256, 1>(gs, n, s);
}

}  // namespace tp
