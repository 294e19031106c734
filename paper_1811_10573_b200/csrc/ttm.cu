// ttm.cu — first-level TTM T = X ×_m A^(m) (PAPER.md P:78-80 Tree_Map_PP level 1; P:405-414
// the dimension-tree MTTKRP whose leading 4 s^N R cost is exactly these TTMs).
//
//   out[b][r][n] = Σ_x X[b][x][r] · F[x][n]      X viewed as [B][S][R], F = A^(m) (S x K)
//
// Contracting mode m of a row-major tensor: B = Π_{v<m} s_v, S = s_m, R = Π_{v>m} s_v.  The
// rank index n lands last (Def. 3.1).  Two orientations of the same GEMM:
//   R == 1  ("k-contiguous"): the natural unfolding X(B x S) · F — X rows are contiguous in x.
//   R  > 1  ("m-contiguous"): per batch b, X_b(S x R)^T · F — X rows are contiguous in r.
//
// sm_100a design:
//   * FP64 tensor cores: tcgen05 has no f64 kind, so the FP64 tensor path on sm_100a is the
//     warp-level DMMA (mma.sync.m8n8k4.f64 -> SASS DMMA.8x8x4).
//   * One CTA = 128 output rows x BN (= K rounded up to 16) columns, so X is streamed from HBM
//     exactly once.  8 consumer warps each own 16 rows x BN; 1 producer warp issues TMA.
//   * TMA (cp.async.bulk.tensor) stages 16-deep k slices of X and of a zero-padded copy of F
//     through a STAGES-deep mbarrier ring with 128-byte swizzle.
//   * Fragment loads are 16-byte LDS (two doubles) with a k-slot permutation and a row
//     permutation chosen so that every quarter-warp hits 8 distinct 16-byte bank groups under
//     the 128B swizzle (derivation in DESIGN.md): thread (g = lane/4, t = lane%4) uses
//     k = 8q + 2t + kk for MMA k-slot t in sub-step (q, kk).
#include "internal.h"

#include <cuda.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <mutex>

namespace cppp {
#ifdef CPPP_PROBE_TTM   // tools/probe_ttm only: per-unit (sm, start, end) global-timer stamps
__device__ unsigned long long g_ttm_trace[1 << 16][3];
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %smid;" : "=r"(r));
  return r;
}
#define TTM_STAMP_START(u)                                      \
  unsigned long long ttm_t0_ = 0;                               \
  if (threadIdx.x == 0) ttm_t0_ = gtimer()
#define TTM_STAMP_END(u)                                                     \
  if (threadIdx.x == 0 && (u) < (1 << 16)) {                                 \
    g_ttm_trace[u][0] = smid();                                              \
    g_ttm_trace[u][1] = ttm_t0_;                                             \
    g_ttm_trace[u][2] = gtimer();                                            \
  }
#else
#define TTM_STAMP_START(u) (void)0
#define TTM_STAMP_END(u) (void)0
#endif
namespace {

constexpr int BM = 128;
constexpr int BK = 16;
constexpr int NWARP = 16;   // consumer warps, 8 output rows each (4 per SM sub-partition)
constexpr int NTHREADS = (NWARP + 1) * 32;
// scratch layout (ttm_scratch_doubles): tile counter + split tickets (TTM_CTL doubles) | split
// partial sums (TTM_PART doubles) | padded factor (S x ttm_ld(K)) -- the control words sit at a
// fixed offset, so launches with different S never overwrite each other's tickets
constexpr int64_t TTM_CTL = 512;
constexpr int64_t TTM_TICKETS = 2 * (TTM_CTL - 8);   // unsigned words after the 8-double counter
constexpr int64_t TTM_PART = static_cast<int64_t>(8) << 20;   // 64 MiB of parked partial tiles

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      " selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(bar), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  while (!mbar_try_wait(bar, parity)) {
  }
}
// Every TMA load carries an L2 cache policy: X streams through once (evict_first, so the GEMM's
// output -- which the next tree level reads right away -- stays in L2 instead of X's dead lines),
// the factor tiles are read by every CTA (evict_last).
__device__ __forceinline__ uint64_t l2_policy_x() {
  uint64_t pol;
#ifdef CPPP_X_EVICT_NORMAL   // A/B builds
  asm volatile("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(pol));
#else
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
#endif
  return pol;
}
__device__ __forceinline__ uint64_t l2_policy_f() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ void tma_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                       uint32_t bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(bar), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tma_3d(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                       int c2, uint32_t bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(bar), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void tma_4d(uint32_t dst, const CUtensorMap* map, int c0, int c1,
                                       int c2, int c3, uint32_t bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
      " [%0], [%1, {%2, %3, %4, %5}], [%6], %7;" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(bar), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void lds2(double& x, double& y, uint32_t addr) {
  asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(x), "=d"(y) : "r"(addr));
}
__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// NT = number of 8-wide n-tiles (BN = 8 NT >= K); the factor is staged 16 columns per TMA box,
// so smem holds BNP = round_up(BN, 16) columns and the odd last tile (if any) is skipped.
template <int NT>
struct Cfg {
  static constexpr int BN = 8 * NT;
  static constexpr int BNP = ((BN + 15) / 16) * 16;
  static constexpr int XBYTES = BM * BK * 8;           // 16 KiB
  static constexpr int FBYTES = BK * BNP * 8;          // 2 KiB per 16 columns
  static constexpr int STAGE = XBYTES + FBYTES;
  static constexpr int MAX_STAGES = (200 * 1024) / STAGE > 8 ? 8 : (200 * 1024) / STAGE;
  static int smem(int stages) { return stages * STAGE + 2 * stages * 8 + 1024; }
};

// Persistent: CTA b processes tiles b, b + gridDim.x, ...; the producer warp runs ahead across
// tile boundaries (bounded by the ring), so the next tile's loads overlap this tile's epilogue.
// Work units: tiles [0, nfull) are whole; each of the nsplit tiles after them is cut into ks
// k chunks (units nfull + ks v + c).  Two uses: a last wave at most half full gets ks = 2 (it
// then costs half a tile instead of a whole one), and a GEMM with few tiles and a long
// reduction (the multi-mode first level, S = s^h) splits every tile.  The chunks of a split
// tile leave partial sums in `part`; the last to finish (ticket) adds them in chunk order
// (deterministic) and writes the tile.
struct Unit {
  long long tile;
  int k0, k1, chunk;   // chunk = -1 for a whole tile
  int nch;             // chunks of this tile
};
__device__ __forceinline__ Unit decode_unit(long long u, long long nfull, int nk, int ks) {
  if (u < nfull) return Unit{u, 0, nk, -1, 1};
  const long long v = u - nfull;
  const int c = static_cast<int>(v % ks);
  return Unit{nfull + v / ks, nk * c / ks, nk * (c + 1) / ks, c, ks};
}
// Stream-K split (skG > 0 CTAs): the ntiles x nk k slices, in (tile, k) order, are cut into skG
// equal ranges and CTA b runs range b, its pieces cut at tile boundaries; unit id = tile x skG +
// b.  Chunk c of tile t is the c-th range touching it (ranges are non-empty: T >= skG).
__device__ __forceinline__ long long sk_range_of(long long x, long long T, long long G) {
  return ((x + 1) * G + T - 1) / T - 1;   // the last range starting at or before slice x
}
__device__ __forceinline__ Unit decode_sk(long long u, int nk, long long T, long long G) {
  const long long t = u / G, b = u - t * G;
  const long long lo = b * T / G, hi = (b + 1) * T / G, t0 = t * nk;
  const long long fb = sk_range_of(t0, T, G), lb = sk_range_of(t0 + nk - 1, T, G);
  const int nch = static_cast<int>(lb - fb + 1);
  return Unit{t, static_cast<int>((lo > t0 ? lo : t0) - t0),
              static_cast<int>((hi < t0 + nk ? hi : t0 + nk) - t0),
              nch > 1 ? static_cast<int>(b - fb) : -1, nch};
}

template <int NT, bool MC, bool BATCH = false>
__global__ void __launch_bounds__(NTHREADS, 1)
    ttm_dmma_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmF,
                    const __grid_constant__ CUtensorMap tmX4,
                    double* __restrict__ out, int64_t Mrows, int64_t mtiles, int64_t nfull,
                    int64_t nsplit, int ks, int S, int K, int stages, int64_t Rflat,
                    unsigned long long* __restrict__ tile_counter, unsigned int* __restrict__ tickets,
                    double* __restrict__ part, int box8, int64_t Rm, int64_t skG) {
  using C = Cfg<NT>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(base + stages * C::STAGE);
  uint64_t* empty = full + stages;
  __shared__ long long stage_tile[16];   // unit id carried by the first k-stage of each unit
  __shared__ Unit stage_unit[16];        // ... its decoded form and tile origin (the consumers
  __shared__ long long stage_bm[16][2];  // skip the 64-bit divisions of decode / batch split)
  __shared__ int ticket_s;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < stages; ++s) {
      mbar_init(smem_u32(&full[s]), 1);
      mbar_init(smem_u32(&empty[s]), NWARP);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  pdl_wait();   // X, the padded factor and the scheduler words come from earlier kernels
  const int nk = (S + BK - 1) / BK;
  const long long nunits = skG ? nsplit * skG : nfull + static_cast<long long>(ks) * nsplit;
  const long long skT = nsplit * nk;   // stream-K: slices in all
  auto decode = [&](long long unit) {
    return skG ? decode_sk(unit, nk, skT, skG) : decode_unit(unit, nfull, nk, ks);
  };

  if (warp == NWARP) {  // ---------------- TMA producer
    if (lane == 0) {
      const uint64_t polX = l2_policy_x(), polF = l2_policy_f();
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmX)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmF)) : "memory");
      if (box8) asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmX4)) : "memory");
      if constexpr (!BATCH) {
        int64_t it = 0;
        int pst = 0;          // it % stages and (it / stages) & 1, kept incrementally (a runtime
        uint32_t pph = 0;     // divisor costs a division sequence per stage)
        long long sk_t = skG ? (blockIdx.x * skT / skG) / nk : 0;
        const long long sk_hi = skG ? (blockIdx.x + 1) * skT / skG : 0;
        while (true) {
          // dynamic tile scheduler: robust to SMs that are busy with other streams' work
          // (stream-K: this CTA's own pieces, in order)
          long long unit;
          if (skG) {
            unit = sk_t * nk < sk_hi ? sk_t * skG + blockIdx.x : nunits;
            ++sk_t;
          } else {
            unit = static_cast<long long>(atomicAdd(tile_counter, 1ull));
          }
          if (unit >= nunits) {
            if (it >= stages) mbar_wait(smem_u32(&empty[pst]), pph ^ 1);
            stage_tile[pst] = -1;
            mbar_arrive(smem_u32(&full[pst]));   // wake the consumers with the sentinel
            break;
          }
          const Unit un = decode(unit);
          const int64_t b = MC ? un.tile / mtiles : 0;
          const int64_t m0 = (un.tile - b * mtiles) * BM;
          // flattened rows: (batch, row) of the tile's first row, one division per unit
          const int64_t b_first = Rflat ? m0 / Rflat : 0;
          const int64_t r_first = Rflat ? m0 - b_first * Rflat : 0;
          for (int kt = un.k0; kt < un.k1; ++kt, ++it) {
            const int st = pst;
            const uint32_t ph = pph;
            if (++pst == stages) {
              pst = 0;
              pph ^= 1u;
            }
            if (it >= stages) mbar_wait(smem_u32(&empty[st]), ph ^ 1);
            if (kt == un.k0) stage_tile[st] = unit;
            const uint32_t fb = smem_u32(&full[st]);
            mbar_expect_tx(fb, C::STAGE);
            const uint32_t sx = smem_u32(base + st * C::STAGE);
            const uint32_t sf = sx + C::XBYTES;
            if (!MC) {
              tma_2d(sx, &tmX, kt * BK, static_cast<int>(m0), fb, polX);
            } else if (box8 && (Rflat ? r_first : m0) + BM <= Rm) {
              // R % 16 == 0 and the tile inside one batch: its eight 16-row boxes in one 4-D load
              tma_4d(sx, &tmX4, 0, kt * BK, static_cast<int>((Rflat ? r_first : m0) / 16),
                     static_cast<int>(Rflat ? b_first : b), fb, polX);
            } else if (Rflat == 0) {
#pragma unroll
              for (int c = 0; c < BM / 16; ++c)
                tma_3d(sx + c * 2048, &tmX, static_cast<int>(m0 + 16 * c), kt * BK,
                       static_cast<int>(b), fb, polX);
            } else {   // rows flattened over (b, r): each 16-row box has its own (b, r)
              int rc = static_cast<int>(r_first), bc = static_cast<int>(b_first);
#pragma unroll
              for (int c = 0; c < BM / 16; ++c) {
                tma_3d(sx + c * 2048, &tmX, rc, kt * BK, bc, fb, polX);
                rc += 16;
                if (rc >= Rflat) {   // R % 16 == 0: a box never straddles two batches
                  rc -= static_cast<int>(Rflat);
                  ++bc;
                }
              }
            }
            tma_3d(sf, &tmF, 0, kt * BK, 0, fb, polF);   // all BNP/16 column boxes in one load
          }
        }
      } else {
        // units with few k stages (short reductions): claimed UB = 4 at a time, the next batch
        // before this one's loads are issued, so the atomic's round trip is not paid per unit
        constexpr long long UB = 4;
        int64_t it = 0;
        int pst = 0;
        uint32_t pph = 0;
        auto issue = [&](long long unit) {
        const Unit un = decode_unit(unit, nfull, nk, ks);
        const int64_t b = MC ? un.tile / mtiles : 0;
        const int64_t m0 = (un.tile - b * mtiles) * BM;
        // flattened rows: (batch, row) of the tile's first row, one division per unit
        const int64_t b_first = Rflat ? m0 / Rflat : 0;
        const int64_t r_first = Rflat ? m0 - b_first * Rflat : 0;
        for (int kt = un.k0; kt < un.k1; ++kt, ++it) {
          const int st = pst;
          const uint32_t ph = pph;
          if (++pst == stages) {
            pst = 0;
            pph ^= 1u;
          }
          if (it >= stages) mbar_wait(smem_u32(&empty[st]), ph ^ 1);
          if (kt == un.k0) {
            stage_tile[st] = unit;
            stage_unit[st] = un;
            stage_bm[st][0] = b;
            stage_bm[st][1] = m0;
          }
          const uint32_t fb = smem_u32(&full[st]);
          mbar_expect_tx(fb, C::STAGE);
          const uint32_t sx = smem_u32(base + st * C::STAGE);
          const uint32_t sf = sx + C::XBYTES;
          if (!MC) {
            tma_2d(sx, &tmX, kt * BK, static_cast<int>(m0), fb, polX);
          } else if (box8 && (Rflat ? r_first : m0) + BM <= Rm) {
            // R % 16 == 0 and the tile inside one batch: its eight 16-row boxes in one 4-D load
            tma_4d(sx, &tmX4, 0, kt * BK, static_cast<int>((Rflat ? r_first : m0) / 16),
                   static_cast<int>(Rflat ? b_first : b), fb, polX);
          } else if (Rflat == 0) {
#pragma unroll
            for (int c = 0; c < BM / 16; ++c)
              tma_3d(sx + c * 2048, &tmX, static_cast<int>(m0 + 16 * c), kt * BK,
                     static_cast<int>(b), fb, polX);
          } else {   // rows flattened over (b, r): each 16-row box has its own (b, r)
            int rc = static_cast<int>(r_first), bc = static_cast<int>(b_first);
#pragma unroll
            for (int c = 0; c < BM / 16; ++c) {
              tma_3d(sx + c * 2048, &tmX, rc, kt * BK, bc, fb, polX);
              rc += 16;
              if (rc >= Rflat) {   // R % 16 == 0: a box never straddles two batches
                rc -= static_cast<int>(Rflat);
                ++bc;
              }
            }
          }
          tma_3d(sf, &tmF, 0, kt * BK, 0, fb, polF);   // all BNP/16 column boxes in one load
        }
        };
        long long next = static_cast<long long>(atomicAdd(tile_counter, (unsigned long long)UB));
        while (next < nunits) {
          const long long u0 = next, u1 = u0 + UB < nunits ? u0 + UB : nunits;
          next = static_cast<long long>(atomicAdd(tile_counter, (unsigned long long)UB));
          for (long long unit = u0; unit < u1; ++unit) issue(unit);
        }
        if (it >= stages) mbar_wait(smem_u32(&empty[pst]), pph ^ 1);
        stage_tile[pst] = -1;
        mbar_arrive(smem_u32(&full[pst]));   // wake the consumers with the sentinel
      }
    }
    return;
  }

  // ---------------- consumers: warp owns 8 output rows x all BN columns (one 8-row m-tile)
  const int g = lane >> 2, t = lane & 3;
  // k-contiguous A: fragment row g -> box row 8 warp + fm(g), fm(g) = (g>>1)|((g&1)<<2)
  const int fm = (g >> 1) | ((g & 1) << 2);
  // m-contiguous A: 16-row box (warp >> 1), rows 8 (warp & 1) + g within it
  const int mbox = warp >> 1, mrow = 8 * (warp & 1) + g;
  const bool pairs = (K % 2) == 0;
  int cst = 0;        // stage index and parity of the next k stage, kept incrementally
  uint32_t cph = 0;
  while (true) {
    mbar_wait(smem_u32(&full[cst]), cph);
    const long long unit = stage_tile[cst];
    if (unit < 0) break;
    // short units (BATCH): the producer's decoded unit; long ones decode it here (measured: the
    // shared-memory copy helps the S = 20 GEMM 272 -> 264 us and costs C2's 395 -> 399 us)
    const Unit un = BATCH ? stage_unit[cst] : decode(unit);
    TTM_STAMP_START(unit);
    const int64_t b = BATCH ? stage_bm[cst][0] : (MC ? un.tile / mtiles : 0);
    const int64_t m0 = BATCH ? stage_bm[cst][1] : (un.tile - b * mtiles) * BM;
    double acc[NT][2];
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[j][0] = acc[j][1] = 0.0;

    for (int kt = un.k0; kt < un.k1; ++kt) {
      const int st = cst;
      if (kt > un.k0) mbar_wait(smem_u32(&full[st]), cph);
      if (++cst == stages) {
        cst = 0;
        cph ^= 1u;
      }
      const uint32_t sx = smem_u32(base + st * C::STAGE);
      const uint32_t sf = sx + C::XBYTES;
      const int qmax = (S - kt * BK) > 8 ? 2 : 1;   // skip an all-zero k tail
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        if (q >= qmax) break;
        double a[2];  // [kk]
        if (!MC) {
          const int row = 8 * warp + fm;
          const int chunk = 4 * q + t;
          lds2(a[0], a[1], sx + row * 128 + ((chunk ^ (row & 7)) << 4));
        } else {
#pragma unroll
          for (int kk = 0; kk < 2; ++kk) {
            const int row = 8 * q + 2 * t + kk;
            asm volatile("ld.shared.f64 %0, [%1];"
                         : "=d"(a[kk])
                         : "r"(sx + mbox * 2048 + row * 128 + (((mrow >> 1) ^ (row & 7)) << 4) +
                               ((mrow & 1) << 3)));
          }
        }
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
          const int row = 8 * q + 2 * t + kk;
          const uint32_t frow = sf + row * 128 + ((g ^ (row & 7)) << 4);
#pragma unroll
          for (int c = 0; c < NT / 2; ++c) {   // tile pair: columns 16c + 2g (+1), interleaved
            double b0, b1;
            lds2(b0, b1, frow + c * 2048);
            dmma(acc[2 * c], a[kk], b0);
            dmma(acc[2 * c + 1], a[kk], b1);
          }
          if (NT & 1) {  // unpaired last tile: contiguous columns 16c + g, 8-byte loads
            constexpr int c = NT / 2;
            double b0;
            asm volatile("ld.shared.f64 %0, [%1];"
                         : "=d"(b0)
                         : "r"(sf + c * 2048 + row * 128 + (((g >> 1) ^ (row & 7)) << 4) + ((g & 1) << 3)));
            dmma(acc[NT - 1], a[kk], b0);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&empty[st]));
    }

    // ---------------- split tile: park this chunk; the last chunk to finish combines
    if (un.chunk >= 0) {
      const int64_t v = un.tile - nfull;
      double* mine = part + ((v * ks + un.chunk) * (NT * 2)) * (NWARP * 32) + threadIdx.x;
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        mine[(2 * j) * (NWARP * 32)] = acc[j][0];
        mine[(2 * j + 1) * (NWARP * 32)] = acc[j][1];
      }
      __threadfence();
      asm volatile("bar.sync 1, %0;" ::"r"(NWARP * 32) : "memory");   // consumer warps only
      if (threadIdx.x == 0) ticket_s = atomicAdd(tickets + v, 1u);
      asm volatile("bar.sync 1, %0;" ::"r"(NWARP * 32) : "memory");
      if (ticket_s != un.nch - 1) {   // another chunk finishes the tile
        TTM_STAMP_END(unit);
        continue;
      }
      __threadfence();
      const double* p0 = part + ((v * ks) * (NT * 2)) * (NWARP * 32) + threadIdx.x;
#pragma unroll
      for (int j = 0; j < NT; ++j) {
        acc[j][0] = __ldcg(p0 + (2 * j) * (NWARP * 32));
        acc[j][1] = __ldcg(p0 + (2 * j + 1) * (NWARP * 32));
      }
      for (int c = 1; c < un.nch; ++c) {
        const double* pc = p0 + c * (NT * 2) * (NWARP * 32);
#pragma unroll
        for (int j = 0; j < NT; ++j) {
          acc[j][0] += __ldcg(pc + (2 * j) * (NWARP * 32));
          acc[j][1] += __ldcg(pc + (2 * j + 1) * (NWARP * 32));
        }
      }
      if (threadIdx.x == 0) tickets[v] = 0u;
    }
    // ---------------- epilogue: thread holds row r x columns 16c + 4t + {0,1,2,3}
    {
      const int mloc = MC ? (16 * mbox + mrow) : (8 * warp + fm);
      const int64_t m = m0 + mloc;
      if (m < Mrows) {
        double* orow = out + (b * Mrows + m) * static_cast<int64_t>(K);
#pragma unroll
        for (int c = 0; c < NT / 2; ++c) {
          const int n0 = 16 * c + 4 * t;
          const double v0 = acc[2 * c][0], v1 = acc[2 * c + 1][0];
          const double v2 = acc[2 * c][1], v3 = acc[2 * c + 1][1];
          if (pairs && n0 + 3 < K) {
            double* p = orow + n0;
            if ((reinterpret_cast<uintptr_t>(p) & 31) == 0) {   // one full 32-byte sector
              asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(v0), "d"(v1),
                           "d"(v2), "d"(v3)
                           : "memory");
            } else {
              *reinterpret_cast<double2*>(p) = make_double2(v0, v1);
              *reinterpret_cast<double2*>(p + 2) = make_double2(v2, v3);
            }
          } else {
            if (n0 < K) orow[n0] = v0;
            if (n0 + 1 < K) orow[n0 + 1] = v1;
            if (n0 + 2 < K) orow[n0 + 2] = v2;
            if (n0 + 3 < K) orow[n0 + 3] = v3;
          }
        }
        if (NT & 1) {
          const int n0 = 16 * (NT / 2) + 2 * t;
          const double v0 = acc[NT - 1][0], v1 = acc[NT - 1][1];
          if (pairs && n0 + 1 < K) {
            *reinterpret_cast<double2*>(orow + n0) = make_double2(v0, v1);
          } else {
            if (n0 < K) orow[n0] = v0;
            if (n0 + 1 < K) orow[n0 + 1] = v1;
          }
        }
      }
    }
    TTM_STAMP_END(unit);
  }
  // the last CTA out resets the scheduler words for the next launch (no memset node, so
  // consecutive launches keep their programmatic dependency)
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(tile_counter + 1, 1ull) == gridDim.x - 1) {
      tile_counter[0] = 0ull;
      tile_counter[1] = 0ull;
      __threadfence();
    }
  }
}

// ---------------------------------------------------------------- fused level 1 -> level 2 (f1)
// The PP construction tree of an order-4 tensor without its s^3 K level-1 nodes in HBM (SURVEY
// NEXT f1; P:700-719 amortises exactly these contractions).  One GEMM contracts mode a of X
// (T = X ×_a A_p^(a), the level-1 node) and its epilogue contracts each 128-row tile of T
// once more, rank-diagonally, into two leaves:
//   * the FAST leaf contracts the last kept mode f: a tile is 128 consecutive x_f (s_f % 128 ==
//     0), so the tile's rows weighted by A_p^(f)[x_f][k] and summed give a partial of
//     M_p(kept \ f) for this x_f block; the nh = s_f / 128 block partials go to separate buffers
//     and are added in block order afterwards;
//   * the LOOP leaf contracts a second kept mode l: a unit is a run of tiles that differ only in
//     x_l (ascending), and each tile's rows, weighted by A_p^(l)[x_l][k], are accumulated into the
//     unit's slice of a partial of M_p(o, f) (o = the third kept mode) -- read-modify-write of a
//     128 x K slice that stays in L2; runs over nP x_l chunks leave nP partials added in order.
// Tile t of the GEMM (m-contiguous, R % 128 == 0: tiles never straddle a batch) covers the
// flattened kept index [128 t, 128 t + 128): t = x_o lstr_o + x_l lstr_l + h with the strides in
// tiles (the flattened row-major index of the kept modes / 128).  Deterministic: every sum has a
// fixed order (rows inside a tile by a fixed shuffle tree then warps in order, x_l ascending inside
// a run, blocks and runs by the combine kernel).
struct FusedArgs {
  int64_t o_str, l_str;          // tile strides of x_o and x_l
  int64_t n_o, n_l, nh;          // extents: x_o, x_l, fast blocks (s_f / 128)
  int64_t run;                   // tiles per unit (x_l chunk length)
  int64_t nP;                    // x_l chunks
  const double* Af;              // A_p^(f), s_f x K
  const double* Al;              // A_p^(l), s_l x K
  double* fast;                  // [nh][leaf rows][K]  (leaf (kept \ f))
  int64_t fl_o, fl_l;            // fast leaf row strides of x_o, x_l
  double* loop;                  // [nP][n_o * s_f][K]  (leaf (o, f))
  int64_t sf;                    // s_f
};

template <int NT>
__global__ void __launch_bounds__(NTHREADS, 1)
    ttm_fused_kernel(const __grid_constant__ CUtensorMap tmF, const __grid_constant__ CUtensorMap tmX4,
                     int64_t mtiles, int S, int K, int stages, unsigned long long* __restrict__ tile_counter,
                     const FusedArgs fa) {
  using C = Cfg<NT>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(base + stages * C::STAGE);
  uint64_t* empty = full + stages;
  double* red = reinterpret_cast<double*>(empty + stages);   // [NWARP][BN] fast-leaf partials
  double* lacc = red + NWARP * C::BN;                           // [BM][BN + 1] loop-leaf slice
  constexpr int LP = C::BN + 1;
  __shared__ long long stage_tile[16];
  __shared__ long long stage_meta[16][4];   // per unit's first stage of a tile: x_o, x_l, h, chunk
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int st = 0; st < stages; ++st) {
      mbar_init(smem_u32(&full[st]), 1);
      mbar_init(smem_u32(&empty[st]), NWARP);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  pdl_wait();
  const int nk = (S + BK - 1) / BK;
  const long long nunits = fa.n_o * fa.nh * fa.nP;
  // unit u -> (x_o, h, chunk p); tile i of the run -> x_l = p run + i
  auto tile_of = [&](long long u, int64_t i, int64_t* xl_out, int64_t* xo, int64_t* h, int64_t* p) {
    *p = u % fa.nP;
    const long long r = u / fa.nP;
    *h = r % fa.nh;
    *xo = r / fa.nh;
    const int64_t xl = *p * fa.run + i;
    *xl_out = xl;
    return *xo * fa.o_str + xl * fa.l_str + *h;
  };
  auto run_len = [&](int64_t p) {
    const int64_t lo = p * fa.run, hi = lo + fa.run < fa.n_l ? lo + fa.run : fa.n_l;
    return hi - lo;
  };
  if (warp == NWARP) {   // ---------------- TMA producer
    if (lane == 0) {
      const uint64_t polX = l2_policy_x(), polF = l2_policy_f();
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmX4)) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&tmF)) : "memory");
      int64_t it = 0;
      int pst = 0;   // it % stages, (it / stages) & 1 kept incrementally
      uint32_t pph = 0;
      while (true) {
        const long long unit = static_cast<long long>(atomicAdd(tile_counter, 1ull));
        if (unit >= nunits) {
          if (it >= stages) mbar_wait(smem_u32(&empty[pst]), pph ^ 1);
          stage_tile[pst] = -1;
          mbar_arrive(smem_u32(&full[pst]));
          break;
        }
        int64_t xl, xo, h, p;
        tile_of(unit, 0, &xl, &xo, &h, &p);
        const int64_t L = run_len(p);
        for (int64_t i = 0; i < L; ++i) {
          const int64_t t = tile_of(unit, i, &xl, &xo, &h, &p);
          const int64_t b = t / mtiles, m0 = (t - b * mtiles) * BM;
          for (int kt = 0; kt < nk; ++kt, ++it) {
            const int st = pst;
            const uint32_t ph = pph;
            if (++pst == stages) {
              pst = 0;
              pph ^= 1u;
            }
            if (it >= stages) mbar_wait(smem_u32(&empty[st]), ph ^ 1);
            if (kt == 0) {   // the consumers read the tile's coordinates (no 64-bit divisions)
              stage_tile[st] = i + (i + 1 == L ? 65536 : 0);
              stage_meta[st][0] = xo;
              stage_meta[st][1] = xl;
              stage_meta[st][2] = h;
              stage_meta[st][3] = p;
            }
            const uint32_t fb = smem_u32(&full[st]);
            mbar_expect_tx(fb, C::STAGE);
            const uint32_t sx = smem_u32(base + st * C::STAGE);
            tma_4d(sx, &tmX4, 0, kt * BK, static_cast<int>(m0 / 16), static_cast<int>(b), fb, polX);
            tma_3d(sx + C::XBYTES, &tmF, 0, kt * BK, 0, fb, polF);
          }
        }
      }
    }
    return;
  }
  // ---------------- consumers (the GEMM part is ttm_dmma_kernel's m-contiguous path)
  const int g = lane >> 2, t4 = lane & 3;
  const int mbox = warp >> 1, mrow = 8 * (warp & 1) + g;
  const int mloc = 16 * mbox + mrow;   // this thread's row of the tile
  int cst = 0;   // stage index and parity of the next k stage, kept incrementally
  uint32_t cph = 0;
  while (true) {
    mbar_wait(smem_u32(&full[cst]), cph);
    const int st0 = cst;
    const long long code = stage_tile[st0];
    if (code < 0) break;
    const int64_t i = code & 65535;
    const bool last = code >= 65536;   // the run's last tile: its loop-leaf slice goes out
    const int64_t xo = stage_meta[st0][0], xl = stage_meta[st0][1], h = stage_meta[st0][2],
                  p = stage_meta[st0][3];
    double acc[NT][2];
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[j][0] = acc[j][1] = 0.0;
    for (int kt = 0; kt < nk; ++kt) {
      const int st = cst;
      if (kt > 0) mbar_wait(smem_u32(&full[st]), cph);
      if (++cst == stages) {
        cst = 0;
        cph ^= 1u;
      }
      const uint32_t sx = smem_u32(base + st * C::STAGE);
      const uint32_t sf = sx + C::XBYTES;
      const int qmax = (S - kt * BK) > 8 ? 2 : 1;
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        if (q >= qmax) break;
        double a[2];
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
          const int row = 8 * q + 2 * t4 + kk;
          asm volatile("ld.shared.f64 %0, [%1];"
                       : "=d"(a[kk])
                       : "r"(sx + mbox * 2048 + row * 128 + (((mrow >> 1) ^ (row & 7)) << 4) +
                             ((mrow & 1) << 3)));
        }
#pragma unroll
        for (int kk = 0; kk < 2; ++kk) {
          const int row = 8 * q + 2 * t4 + kk;
          const uint32_t frow = sf + row * 128 + ((g ^ (row & 7)) << 4);
#pragma unroll
          for (int c = 0; c < NT / 2; ++c) {
            double b0, b1;
            lds2(b0, b1, frow + c * 2048);
            dmma(acc[2 * c], a[kk], b0);
            dmma(acc[2 * c + 1], a[kk], b1);
          }
          if (NT & 1) {
            constexpr int c = NT / 2;
            double b0;
            asm volatile("ld.shared.f64 %0, [%1];"
                         : "=d"(b0)
                         : "r"(sf + c * 2048 + row * 128 + (((g >> 1) ^ (row & 7)) << 4) + ((g & 1) << 3)));
            dmma(acc[NT - 1], a[kk], b0);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(smem_u32(&empty[st]));
    }
    // ---------------- epilogue: (row mloc) x (columns 16c + 4t4 + {0..3}, and 16(NT/2) + 2t4 + {0,1})
    const int64_t xf = h * BM + mloc;
    const double* af = fa.Af + xf * K;
    const double* al = fa.Al + xl * K;
    double* lrow = fa.loop + (p * fa.n_o * fa.sf + xo * fa.sf + xf) * static_cast<int64_t>(K);
    double* lsm = lacc + mloc * LP;   // this thread's row of the run's loop-leaf slice (smem)
    // value of (tile pair c, element e) -> column and accumulator
#pragma unroll
    for (int c = 0; c < (NT + 1) / 2; ++c) {
      const bool pair = 2 * c + 1 < NT;
      double v[4];
      int n[4];
      if (pair) {
        v[0] = acc[2 * c][0];
        v[1] = acc[2 * c + 1][0];
        v[2] = acc[2 * c][1];
        v[3] = acc[2 * c + 1][1];
        for (int e = 0; e < 4; ++e) n[e] = 16 * c + 4 * t4 + e;
      } else {
        v[0] = acc[2 * c][0];
        v[1] = acc[2 * c][1];
        v[2] = v[3] = 0.0;
        n[0] = 16 * c + 2 * t4;
        n[1] = n[0] + 1;
        n[2] = n[3] = K;   // none
      }
      double fsum[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const bool ok = n[e] < K;
        // loop leaf: x_l ascending inside the run (the first tile initialises the slice)
        if (ok) {
          const double w = __ldg(al + n[e]);
          const double x = i == 0 ? v[e] * w : fma(v[e], w, lsm[n[e]]);
          if (last) lrow[n[e]] = x;
          else lsm[n[e]] = x;
        }
        fsum[e] = ok ? v[e] * __ldg(af + n[e]) : 0.0;
      }
      // fast leaf: the warp's 8 rows (g) by a fixed xor tree, then the warps in order
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        fsum[e] += __shfl_xor_sync(0xffffffffu, fsum[e], 4);
        fsum[e] += __shfl_xor_sync(0xffffffffu, fsum[e], 8);
        fsum[e] += __shfl_xor_sync(0xffffffffu, fsum[e], 16);
      }
      if (g == 0) {
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (n[e] < K) red[warp * C::BN + n[e]] = fsum[e];
      }
    }
    asm volatile("bar.sync 1, %0;" ::"r"(NWARP * 32) : "memory");   // consumer warps only
    if (threadIdx.x < K) {
      const int n = threadIdx.x;
      double s = 0.0;
      // warps in row order: warp w holds rows 16 (w >> 1) + 8 (w & 1) + g
      for (int w = 0; w < NWARP; ++w) s += red[w * C::BN + n];
      fa.fast[(h * (fa.n_o * fa.n_l) + xo * fa.fl_o + xl * fa.fl_l) * static_cast<int64_t>(K) + n] = s;
    }
    asm volatile("bar.sync 1, %0;" ::"r"(NWARP * 32) : "memory");
  }
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(tile_counter + 1, 1ull) == gridDim.x - 1) {
      tile_counter[0] = 0ull;
      tile_counter[1] = 0ull;
      __threadfence();
    }
  }
}

// ---------------------------------------------------------------- SIMT fallback
// One thread per output (b, r, n); X read with r fastest across the warp.
__global__ void ttm_simt_kernel(const double* __restrict__ X, int64_t B, int64_t S, int64_t R,
                                const double* __restrict__ F, int K, double* __restrict__ out) {
  const int64_t total = B * R * K;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t n = e / (B * R);
    const int64_t br = e - n * (B * R);
    const int64_t b = br / R, r = br - b * R;
    const double* xp = X + b * S * R + r;
    double acc = 0.0;
    for (int64_t x = 0; x < S; ++x) acc = fma(xp[x * R], F[x * K + n], acc);
    out[br * K + n] = acc;
  }
}

// ---------------------------------------------------------------- skinny GEMMs (K <= 16)
// Shapes the TMA GEMM cannot take (an odd row stride: s = 25 for the compact Laplacian)
// with a small rank: 2 K flops per 8-byte element of X, far below the FP64 ridge (5.7 flop/B), so
// the bound is HBM and the tensor core has nothing to win -- what matters is streaming X once,
// coalesced.  KB >= K accumulators per thread, x in ascending order (as the GEMM).
//   m-contiguous (R > 1): thread per (b, r); a warp reads 32 consecutive r of one x row (a
//     coalesced 256-byte run), the factor row F[x][0..K) is a broadcast load.
template <int KB>
__global__ void __launch_bounds__(256)
    ttm_skinny_mc_kernel(const double* __restrict__ X, int64_t B, int64_t S, int64_t R,
                         const double* __restrict__ F, int K, double* __restrict__ out) {
  pdl_wait();
  const int64_t total = B * R;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t b = e / R, r = e - b * R;
    const double* xp = X + b * S * R + r;
    double acc[KB];
#pragma unroll
    for (int n = 0; n < KB; ++n) acc[n] = 0.0;
    int64_t x = 0;
    for (; x + 4 <= S; x += 4) {
      double v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = __ldcs(xp + (x + u) * R);
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int n = 0; n < KB; ++n)
          if (n < K) acc[n] = fma(v[u], __ldg(F + (x + u) * K + n), acc[n]);
    }
    for (; x < S; ++x) {
      const double v = __ldcs(xp + x * R);
#pragma unroll
      for (int n = 0; n < KB; ++n)
        if (n < K) acc[n] = fma(v, __ldg(F + x * K + n), acc[n]);
    }
    double* o = out + e * K;
#pragma unroll
    for (int n = 0; n < KB; ++n)
      if (n < K) o[n] = acc[n];
  }
}

//   k-contiguous (R == 1, rows of S doubles): a CTA stages SK_ROWS consecutive rows -- one
//     contiguous run of X -- through shared memory with coalesced loads, then thread = row
//     (odd row pitch S: conflict-free for odd S), the factor in shared memory.
constexpr int SK_ROWS = 128;
template <int KB>
__global__ void __launch_bounds__(SK_ROWS)
    ttm_skinny_kc_kernel(const double* __restrict__ X, int64_t B, int S, const double* __restrict__ F,
                         int K, double* __restrict__ out) {
  pdl_wait();
  extern __shared__ double sk[];   // [SK_ROWS * S] rows | [S * K] factor
  double* fs = sk + (int64_t)SK_ROWS * S;
  for (int e = threadIdx.x; e < S * K; e += SK_ROWS) fs[e] = F[e];
  for (int64_t b0 = (int64_t)blockIdx.x * SK_ROWS; b0 < B; b0 += (int64_t)gridDim.x * SK_ROWS) {
    const int nr = static_cast<int>(B - b0 < SK_ROWS ? B - b0 : SK_ROWS);
    const double* src = X + b0 * S;
    __syncthreads();
    for (int e = threadIdx.x; e < nr * S; e += SK_ROWS) sk[e] = __ldcs(src + e);
    __syncthreads();
    if (threadIdx.x < nr) {
      const double* row = sk + threadIdx.x * S;
      double acc[KB];
#pragma unroll
      for (int n = 0; n < KB; ++n) acc[n] = 0.0;
      for (int x = 0; x < S; ++x) {
        const double v = row[x];
#pragma unroll
        for (int n = 0; n < KB; ++n)
          if (n < K) acc[n] = fma(v, fs[x * K + n], acc[n]);
      }
      double* o = out + (b0 + threadIdx.x) * K;
#pragma unroll
      for (int n = 0; n < KB; ++n)
        if (n < K) o[n] = acc[n];
    }
  }
}

//   k-contiguous with long rows (the Khatri-Rao first level: S = s^3 = 15625 for LAP): warp per
//     row, lanes on consecutive x (coalesced), the lane partials added by a fixed xor tree.
template <int KB>
__global__ void __launch_bounds__(256)
    ttm_skinny_rows_kernel(const double* __restrict__ X, int64_t B, int64_t S, const double* __restrict__ F,
                           int K, double* __restrict__ out) {
  pdl_wait();
  const int lane = threadIdx.x & 31;
  const int64_t w0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t b = w0; b < B; b += nw) {
    const double* row = X + b * S;
    double acc[KB];
#pragma unroll
    for (int n = 0; n < KB; ++n) acc[n] = 0.0;
    for (int64_t x = lane; x < S; x += 32) {
      const double v = __ldcs(row + x);
#pragma unroll
      for (int n = 0; n < KB; ++n)
        if (n < K) acc[n] = fma(v, __ldg(F + x * K + n), acc[n]);
    }
#pragma unroll
    for (int n = 0; n < KB; ++n)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc[n] += __shfl_xor_sync(0xffffffffu, acc[n], o);
    if (lane == 0) {
#pragma unroll
      for (int n = 0; n < KB; ++n)
        if (n < K) out[b * K + n] = acc[n];
    }
  }
}

// Bulk-copy versions of the two skinny kernels above (same per-output fma chains in ascending x,
// so bit-identical): X reaches shared memory by 1-D bulk async copies (cp.async.bulk, SASS
// UBLKCP) completing on an mbarrier, instead of per-thread loads -- every CTA keeps one or two
// whole chunks of X in flight with one issuing thread.  tools/probe_skinny.cu on the compact
// Laplacian's 1.95 GB first-level shapes (L2 flushed): k-contiguous 428 -> 329 us (4.9 -> 6.4
// TB/s), m-contiguous 531 -> 336 us (4.0 -> 6.3 TB/s).  Per-CTA multi-stage rings measured
// slower for the m-contiguous shape (NS = 2..4 with 1-2 CTAs per SM: 3.1-5.5 TB/s); four CTAs
// per SM with one chunk each are the fastest.
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar,
                                         uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
      ::"r"(dst), "l"(src), "r"(bytes), "r"(bar), "l"(pol)
      : "memory");
}

//   k-contiguous (R == 1): a chunk = SKB_CH consecutive rows of S doubles, one contiguous run
//     (SKB_CH even and X 16-byte aligned, so every full chunk is a legal bulk copy); an
//     SKB_NS-deep ring per CTA; thread = row; a ragged last chunk by plain loads.
constexpr int SKB_CH = 256, SKB_NS = 2;
template <int KB>
__global__ void __launch_bounds__(SKB_CH)
    ttm_skinny_kc_bulk_kernel(const double* __restrict__ X, int64_t B, int S, const double* __restrict__ F,
                              int K, double* __restrict__ out) {
  extern __shared__ __align__(16) double skb[];   // [SKB_NS][SKB_CH * S] | factor [S * K] | barriers
  double* fs = skb + (int64_t)SKB_NS * SKB_CH * S;
  uint64_t* full = reinterpret_cast<uint64_t*>(fs + ((S * K + 1) & ~1));
  const int tid = threadIdx.x;
  const int64_t nch = (B + SKB_CH - 1) / SKB_CH, nfull = B / SKB_CH;
  const uint32_t bytes = static_cast<uint32_t>(SKB_CH) * S * 8;
  if (tid == 0) {
    for (int s = 0; s < SKB_NS; ++s) mbar_init(smem_u32(&full[s]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  pdl_wait();
  uint64_t pol = 0;
  if (tid == 0) {
    pol = l2_policy_x();
    for (int s = 0; s < SKB_NS; ++s) {
      const int64_t c = blockIdx.x + static_cast<int64_t>(s) * gridDim.x;
      if (c < nfull) {
        mbar_expect_tx(smem_u32(&full[s]), bytes);
        bulk_g2s(smem_u32(skb + static_cast<int64_t>(s) * SKB_CH * S), X + c * SKB_CH * S, bytes,
                 smem_u32(&full[s]), pol);
      }
    }
  }
  for (int e = tid; e < S * K; e += SKB_CH) fs[e] = F[e];
  __syncthreads();
  uint32_t phase = 0;   // per-stage parity (a plain-load chunk leaves its stage's barrier as it is)
  int it = 0;
  for (int64_t c = blockIdx.x; c < nch; c += gridDim.x, ++it) {
    const int st = it % SKB_NS;
    double* stage = skb + static_cast<int64_t>(st) * SKB_CH * S;
    const int nr = static_cast<int>(B - c * SKB_CH < SKB_CH ? B - c * SKB_CH : SKB_CH);
    if (c < nfull) {
      mbar_wait(smem_u32(&full[st]), (phase >> st) & 1u);
      phase ^= 1u << st;
    } else {
      for (int e = tid; e < nr * S; e += SKB_CH) stage[e] = __ldcs(X + c * SKB_CH * S + e);
      __syncthreads();
    }
    if (tid < nr) {
      const double* row = stage + tid * S;   // odd S: conflict-free 8-byte reads across the warp
      double acc[KB];
#pragma unroll
      for (int n = 0; n < KB; ++n) acc[n] = 0.0;
      for (int x = 0; x < S; ++x) {
        const double v = row[x];
#pragma unroll
        for (int n = 0; n < KB; ++n)
          if (n < K) acc[n] = fma(v, fs[x * K + n], acc[n]);
      }
      double* o = out + (c * SKB_CH + tid) * K;
#pragma unroll
      for (int n = 0; n < KB; ++n)
        if (n < K) o[n] = acc[n];
    }
    __syncthreads();   // every thread is done with the stage before it is refilled
    if (tid == 0) {
      const int64_t cn = c + static_cast<int64_t>(SKB_NS) * gridDim.x;
      if (cn < nfull) {
        mbar_expect_tx(smem_u32(&full[st]), bytes);
        bulk_g2s(smem_u32(stage), X + cn * SKB_CH * S, bytes, smem_u32(&full[st]), pol);
      }
    }
  }
}

//   m-contiguous (R >= SMB_CR): a unit = (b, SMB_CR consecutive r, SMB_XG consecutive x): SMB_XG
//     row segments X[b][x][r0 .. r0 + SMB_CR), each copied from the 16-byte boundary at or below
//     its start (odd R: every other x row is 8 bytes off), pitch SMB_CR + 2; a CTA runs the x
//     groups of its r block in order, so each thread's SMB_CR / 256 accumulator sets persist
//     across units; blocks whose rounded copies would leave X (the ragged last r block of a
//     batch, the very end of X) go by plain loads.
constexpr int SMB_CR = 1024, SMB_XG = 5, SMB_THREADS = 256;
template <int KB>
__global__ void __launch_bounds__(SMB_THREADS)
    ttm_skinny_mc_bulk_kernel(const double* __restrict__ X, int64_t B, int S, int64_t R,
                              const double* __restrict__ F, int K, double* __restrict__ out) {
  extern __shared__ __align__(16) double smb[];   // [SMB_XG][SMB_CR + 2] | factor [S * K] | barrier
  constexpr int P = SMB_CR + 2, RT = SMB_CR / SMB_THREADS;
  double* fs = smb + SMB_XG * P;
  uint64_t* full = reinterpret_cast<uint64_t*>(fs + ((S * K + 1) & ~1));
  const int tid = threadIdx.x;
  const int ng = (S + SMB_XG - 1) / SMB_XG;
  const int64_t nrb = (R + SMB_CR - 1) / SMB_CR, nch = B * nrb;
  const double* Xend = X + B * S * R;
  auto bulk_ok = [&](int64_t b, int64_t r0) {
    return r0 + SMB_CR <= R && X + ((b * S + S - 1) * R + r0 + SMB_CR + 2) <= Xend;
  };
  auto seg_off = [](const double* p) { return static_cast<int>((reinterpret_cast<uintptr_t>(p) >> 3) & 1); };
  if (tid == 0) {
    mbar_init(smem_u32(&full[0]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  pdl_wait();
  for (int e = tid; e < S * K; e += SMB_THREADS) fs[e] = F[e];
  const uint64_t pol = l2_policy_x();
  uint32_t phase = 0;
  double acc[RT][KB];
  for (int64_t c = blockIdx.x; c < nch; c += gridDim.x) {
    const int64_t b = c / nrb, r0 = (c - b * nrb) * SMB_CR;
    const int nr = static_cast<int>(R - r0 < SMB_CR ? R - r0 : SMB_CR);
    const bool bulk = bulk_ok(b, r0);
#pragma unroll
    for (int j = 0; j < RT; ++j)
#pragma unroll
      for (int n = 0; n < KB; ++n) acc[j][n] = 0.0;
    for (int g = 0; g < ng; ++g) {
      const int xa = g * SMB_XG, xb = xa + SMB_XG < S ? xa + SMB_XG : S;
      const double* row0 = X + (b * S + xa) * R + r0;
      __syncthreads();   // the previous unit's readers are done (and the factor is staged)
      if (bulk) {
        if (tid == 0) {
          uint32_t tot = 0;
          for (int x = xa; x < xb; ++x)
            tot += static_cast<uint32_t>(((SMB_CR + seg_off(row0 + (x - xa) * R)) * 8 + 15) & ~15);
          mbar_expect_tx(smem_u32(&full[0]), tot);
          for (int x = xa; x < xb; ++x) {
            const double* src = row0 + (x - xa) * R;
            const int off = seg_off(src);
            bulk_g2s(smem_u32(smb + (x - xa) * P), src - off,
                     static_cast<uint32_t>(((SMB_CR + off) * 8 + 15) & ~15), smem_u32(&full[0]), pol);
          }
        }
        mbar_wait(smem_u32(&full[0]), phase);
        phase ^= 1u;
      } else {
        for (int x = xa; x < xb; ++x) {
          const double* src = row0 + (x - xa) * R;
          const int off = seg_off(src);
          for (int t = tid; t < nr; t += SMB_THREADS) smb[(x - xa) * P + off + t] = __ldcs(src + t);
        }
        __syncthreads();
      }
      for (int x = xa; x < xb; ++x) {
        const double* srow = smb + (x - xa) * P + seg_off(row0 + (x - xa) * R);
        double f[KB];
#pragma unroll
        for (int n = 0; n < KB; ++n) f[n] = n < K ? fs[x * K + n] : 0.0;
#pragma unroll
        for (int j = 0; j < RT; ++j) {
          const double v = srow[tid + SMB_THREADS * j];
#pragma unroll
          for (int n = 0; n < KB; ++n)
            if (n < K) acc[j][n] = fma(v, f[n], acc[j][n]);
        }
      }
    }
#pragma unroll
    for (int j = 0; j < RT; ++j) {
      const int r = tid + SMB_THREADS * j;
      if (r < nr) {
        double* o = out + (b * R + r0 + r) * K;
#pragma unroll
        for (int n = 0; n < KB; ++n)
          if (n < K) o[n] = acc[j][n];
      }
    }
  }
}

bool skinny_bulk_on() {
  static const bool off = getenv("CPPP_NO_SKINNY_BULK") != nullptr;   // A/B: the register-load kernels
  return !off;
}

template <int KB>
cudaError_t run_skinny(const double* X, int64_t B, int64_t S, int64_t R, const double* F, int K,
                       double* out, cudaStream_t st) {
  const bool al16 = (reinterpret_cast<uintptr_t>(X) & 15) == 0;
  if (R > 1 && al16 && skinny_bulk_on() && R >= SMB_CR && S * K <= 1024 && S < (1 << 30)) {
    const size_t smem = sizeof(double) * (SMB_XG * (SMB_CR + 2) + ((S * K + 1) & ~1)) + 16;
    static bool attr = false;
    if (!attr) {
      cudaError_t e = cudaFuncSetAttribute(ttm_skinny_mc_bulk_kernel<KB>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, 56 * 1024);
      if (e != cudaSuccess) return e;
      attr = true;
    }
    int64_t blocks = B * ((R + SMB_CR - 1) / SMB_CR);
    if (blocks > 148 * 4) blocks = 148 * 4;
    cudaError_t e = launch_pdl(ttm_skinny_mc_bulk_kernel<KB>, dim3((unsigned)blocks), dim3(SMB_THREADS), smem,
                               st, X, B, (int)S, R, F, K, out);
    note_launch();
    return e;
  }
  if (R > 1) {
    int64_t blocks = (B * R + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    cudaError_t e = launch_pdl(ttm_skinny_mc_kernel<KB>, dim3((unsigned)blocks), dim3(256), 0, st, X, B, S, R,
                               F, K, out);
    note_launch();
    return e;
  }
  const size_t smem = sizeof(double) * (static_cast<size_t>(SK_ROWS) * S + S * K);
  if (smem > 200 * 1024) {
    int64_t blocks = (B * 32 + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    cudaError_t e = launch_pdl(ttm_skinny_rows_kernel<KB>, dim3((unsigned)blocks), dim3(256), 0, st, X, B, S, F,
                               K, out);
    note_launch();
    return e;
  }
  const size_t smem_b = sizeof(double) * (static_cast<size_t>(SKB_NS) * SKB_CH * S + ((S * K + 1) & ~1)) + 16 * SKB_NS;
  if (al16 && skinny_bulk_on() && smem_b <= 110 * 1024) {   // two CTAs per SM
    static bool attr_b = false;
    if (!attr_b) {
      cudaError_t e = cudaFuncSetAttribute(ttm_skinny_kc_bulk_kernel<KB>,
                                           cudaFuncAttributeMaxDynamicSharedMemorySize, 110 * 1024);
      if (e != cudaSuccess) return e;
      attr_b = true;
    }
    int64_t blocks = (B + SKB_CH - 1) / SKB_CH;
    if (blocks > 148 * 2) blocks = 148 * 2;
    cudaError_t e = launch_pdl(ttm_skinny_kc_bulk_kernel<KB>, dim3((unsigned)blocks), dim3(SKB_CH), smem_b, st, X,
                               B, (int)S, F, K, out);
    note_launch();
    return e;
  }
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(ttm_skinny_kc_kernel<KB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         200 * 1024);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  int64_t blocks = (B + SK_ROWS - 1) / SK_ROWS;
  if (blocks > 148 * 8) blocks = 148 * 8;
  cudaError_t e = launch_pdl(ttm_skinny_kc_kernel<KB>, dim3((unsigned)blocks), dim3(SK_ROWS), smem, st, X, B,
                             (int)S, F, K, out);
  note_launch();
  return e;
}

// ---------------------------------------------------------------- host side
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                  const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                  const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn get_encode() {
  static EncodeTiledFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeTiledFn>(p);
  });
  return fn;
}

bool make_map(CUtensorMap* m, const void* ptr, int rank, const cuuint64_t* dims,
              const cuuint64_t* strides_bytes, const cuuint32_t* box) {
  EncodeTiledFn enc = get_encode();
  if (!enc) return false;
  cuuint32_t es[5] = {1, 1, 1, 1, 1};
  CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, rank, const_cast<void*>(ptr), dims,
                   strides_bytes, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

bool getenv_no_box8() {   // CPPP_NO_BOX8: the per-16-row boxes (A/B)
  static const bool v = getenv("CPPP_NO_BOX8") != nullptr;
  return v;
}

template <int NT, bool MC, bool BATCH>
cudaError_t run_dmma_b(const double* X, int64_t B, int64_t S, int64_t R, const double* Fp, int K,
                     double* out, unsigned long long* counter, unsigned int* tickets, double* part,
                     cudaStream_t st, TtmOpts topt) {
  using C = Cfg<NT>;
  static bool attr_done = false;
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(ttm_dmma_kernel<NT, MC, BATCH>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         C::smem(C::MAX_STAGES));
    if (e != cudaSuccess) return e;
    attr_done = true;
  }
  CUtensorMap tmX, tmF;
  // m-contiguous with several batches and R % 16 == 0: tiles run over the flattened (b, r) rows
  // (16-row boxes never straddle a batch), so no batch leaves a partial tile (C2's middle mode:
  // R = 400 = 3 x 128 + 16 wasted 22% of the tiles' rows)
  const int64_t Rflat = (MC && B > 1 && R % 16 == 0) ? R : 0;
  const int box8 = (MC && R % 16 == 0 && R >= BM && !getenv_no_box8()) ? 1 : 0;
  const int64_t Mrows = MC ? (Rflat ? B * R : R) : B;
  if (!MC) {
    cuuint64_t dims[2] = {(cuuint64_t)S, (cuuint64_t)B};
    cuuint64_t str[1] = {(cuuint64_t)S * 8};
    cuuint32_t box[2] = {16, BM};
    if (!make_map(&tmX, X, 2, dims, str, box)) return cudaErrorInvalidValue;
  } else {
    cuuint64_t dims[3] = {(cuuint64_t)R, (cuuint64_t)S, (cuuint64_t)B};
    cuuint64_t str[2] = {(cuuint64_t)R * 8, (cuuint64_t)(S * R) * 8};
    cuuint32_t box[3] = {16, 16, 1};
    if (!make_map(&tmX, X, 3, dims, str, box)) return cudaErrorInvalidValue;
  }
  CUtensorMap tmX4 = tmX;
  if (box8) {
    // [B][S][R] viewed as [B][R/16][S][16] (r = 16 r_hi + r_lo): one box = 8 r_hi x 16 x x 16 r_lo,
    // landing in shared memory exactly as the eight 16 x 16 boxes of the 3-D map
    cuuint64_t dims[4] = {16, (cuuint64_t)S, (cuuint64_t)(R / 16), (cuuint64_t)B};
    cuuint64_t str[3] = {(cuuint64_t)R * 8, 128, (cuuint64_t)(S * R) * 8};
    cuuint32_t box[4] = {16, 16, 8, 1};
    if (!make_map(&tmX4, X, 4, dims, str, box)) return cudaErrorInvalidValue;
  }
  {
    // the padded factor [S][BNP] viewed as [BNP/16][S][16]: one box = every 16-column strip of
    // a 16-deep k slice, landing as the strips' 16 x 16 boxes one after another.  In place
    // (direct_factor) the row stride is K: columns >= K of a strip hold the next row's head,
    // which only feeds output columns the epilogue drops
    const int64_t ld = topt.direct_factor ? K : C::BNP;
    cuuint64_t dims[3] = {16, (cuuint64_t)S, (cuuint64_t)(C::BNP / 16)};
    cuuint64_t str[2] = {(cuuint64_t)ld * 8, 128};
    cuuint32_t box[3] = {16, 16, (cuuint32_t)(C::BNP / 16)};
    if (!make_map(&tmF, Fp, 3, dims, str, box)) return cudaErrorInvalidValue;
  }
  // the ring spans several tiles when S is short (C4: s = 20 -> 2 slices per tile), so the
  // producer keeps loading the next tiles while the consumers finish this one
  static const int stages_env = [] {   // CPPP_TTM_STAGES: ring depth override (A/B)
    const char* e = getenv("CPPP_TTM_STAGES");
    return e ? atoi(e) : 0;
  }();
  int stages = stages_env >= 2 && stages_env <= C::MAX_STAGES ? stages_env : C::MAX_STAGES;
  if (topt.max_stages >= 2 && topt.max_stages < stages) stages = topt.max_stages;
  const int smem = C::smem(stages);
  const int64_t mtiles = (Mrows + BM - 1) / BM;
  const int64_t ntiles = mtiles * ((MC && !Rflat) ? B : 1);
  int occ = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, ttm_dmma_kernel<NT, MC, BATCH>, NTHREADS, smem);
  if (occ < 1) occ = 1;
  int sms = 148;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  // `reserve` SMs get no CTA: the latency-bound kernels of other streams run there meanwhile
  // (a persistent CTA holds its SM until the GEMM ends)
  const int64_t full_grid = std::max<int64_t>(1, static_cast<int64_t>(sms) * occ - topt.reserve_sms);
  int64_t grid = full_grid;
  if (grid > ntiles) grid = ntiles;
  const int nk = static_cast<int>((S + BK - 1) / BK);
  const int64_t slot = static_cast<int64_t>(NT) * 2 * NWARP * 32;   // doubles per parked chunk
  int64_t nsplit = 0, skG = 0;
  int ks = 1;
  const double eff1 = [&] {
    const double w = static_cast<double>(ntiles) / full_grid;
    return w / std::ceil(w);
  }();
  if (eff1 < 0.9 && nk >= 32 && ntiles <= TTM_TICKETS) {
    // few tiles or a badly filled last wave, and a long reduction (the multi-mode first level):
    // split every tile into ks k chunks, the smallest ks whose units fill their last wave to
    // >= 90% (else the fullest)
    int best = 1;
    double best_eff = eff1;
    for (int k = 2; k <= 32 && k <= nk / 8 && ntiles * k * slot <= TTM_PART; ++k) {
      const double waves = static_cast<double>(ntiles * k) / full_grid;
      const double eff = waves / std::ceil(waves);
      if (eff > best_eff + 1e-9) {
        best = k;
        best_eff = eff;
      }
      if (eff >= 0.9) break;
    }
    ks = best;
    // stream-K instead when the uniform split still leaves its last wave < 95% full: every
    // CTA gets the same number of k slices (C3: ks = 7 left 553 units 3.7 waves deep, SMs
    // ending between 279 and 380 us; stream-K 343-349 us).  C4's ks = 7 fills 99.3% and
    // stays (stream-K measured 2.6% slower there)
    // A static partition cannot absorb a CTA that waits for an SM (the side-stream Γ
    // factorization is resident on some SM when the GEMM starts), so stream-K leaves two SMs
    // free unless the caller already reserved some (C3 1029 -> 1048 sweeps/s)
    static const bool no_sk = getenv("CPPP_NO_STREAMK") != nullptr;   // A/B
    const int64_t G = std::max<int64_t>(1, full_grid - (topt.reserve_sms > 0 ? 0 : 2));
    const int64_t T = ntiles * nk, per = T / G;
    const int ksmax = per > 0 ? static_cast<int>((nk + per - 1) / per) + 1 : 0;
    if (!no_sk && ks > 1 && best_eff < 0.95 && per >= 8 && ntiles * ksmax * slot <= TTM_PART) {
      skG = G;
      ks = ksmax;
      nsplit = ntiles;
      grid = G;
    } else if (ks > 1) {
      nsplit = ntiles;
      grid = full_grid < ntiles * ks ? full_grid : ntiles * ks;
    } else {
      ks = 1;
    }
  }
  if (ks == 1) {
    // a last wave at most half full is split into k halves (one wave of half-tiles).  (Stream-K
    // over the last wave's k slices -- every SM ending within a few slices of the others -- was
    // slower: the partial-tile combines land on the critical path, C2's GEMM 395 -> 404 us.)
    const int64_t tail = ntiles % grid;
    if (ntiles > grid && tail > 0 && 2 * tail <= grid && tail * 2 * slot <= TTM_PART && nk >= 4) {
      nsplit = tail;
      ks = 2;
    }
  }
  const int64_t nfull = skG ? 0 : ntiles - nsplit;
  static const bool dbg = getenv("CPPP_DEBUG_TTM") != nullptr;
  if (dbg)
    fprintf(stderr, "ttm B %lld S %lld R %lld K %d: tiles %lld grid %lld split %lld x %d%s\n",
            (long long)B, (long long)S, (long long)R, K, (long long)ntiles, (long long)grid,
            (long long)nsplit, ks, skG ? " (stream-K)" : "");
  cudaError_t e = launch_pdl(ttm_dmma_kernel<NT, MC, BATCH>, dim3((unsigned)grid), dim3(NTHREADS), smem, st,
                             tmX, tmF, tmX4, out, Mrows, mtiles, nfull, nsplit, ks, (int)S, K, stages,
                             Rflat, counter, tickets, part, box8, R, skG);
  note_launch();
  return e;
}

// units of fewer than 8 k stages (S <= 112, whole tiles) take the batched scheduler when there
// are many of them (>= 8 per SM; a small GEMM would leave CTAs idle: C1's 13 tiles)
template <int NT, bool MC>
cudaError_t run_dmma(const double* X, int64_t B, int64_t S, int64_t R, const double* Fp, int K,
                     double* out, unsigned long long* counter, unsigned int* tickets, double* part,
                     cudaStream_t st, TtmOpts topt) {
  const int64_t tiles_est = MC ? B * ((R + BM - 1) / BM) : (B + BM - 1) / BM;
  if ((S + BK - 1) / BK < 8 && tiles_est >= 148 * 8)
    return run_dmma_b<NT, MC, true>(X, B, S, R, Fp, K, out, counter, tickets, part, st, topt);
  return run_dmma_b<NT, MC, false>(X, B, S, R, Fp, K, out, counter, tickets, part, st, topt);
}

template <bool MC, int NT = 1>
cudaError_t dispatch_nt(int nt, const double* X, int64_t B, int64_t S, int64_t R, const double* Fp,
                        int K, double* out, unsigned long long* counter, unsigned int* tickets,
                        double* part, cudaStream_t st, TtmOpts topt) {
  if constexpr (NT > 16) {
    return cudaErrorInvalidValue;
  } else {
    if (nt == NT) return run_dmma<NT, MC>(X, B, S, R, Fp, K, out, counter, tickets, part, st, topt);
    return dispatch_nt<MC, NT + 1>(nt, X, B, S, R, Fp, K, out, counter, tickets, part, st, topt);
  }
}

template <int NT>
cudaError_t run_fused(const double* X, int64_t B, int64_t S, int64_t R, const double* Fp, int K,
                      unsigned long long* counter, const FusedArgs& fa, cudaStream_t st) {
  using C = Cfg<NT>;
  // the fast-leaf reduction buffer and the run's loop-leaf slice live beside the stage ring
  const int red_bytes = NWARP * C::BN * 8 + BM * (C::BN + 1) * 8;
  int stages = C::MAX_STAGES;
  while (stages > 2 && C::smem(stages) + red_bytes > 220 * 1024) --stages;
  static bool attr_done = false;
  if (!attr_done) {
    cudaError_t e = cudaFuncSetAttribute(ttm_fused_kernel<NT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         220 * 1024);
    if (e != cudaSuccess) return e;
    attr_done = true;
  }
  CUtensorMap tmX4, tmF;
  {
    cuuint64_t dims[4] = {16, (cuuint64_t)S, (cuuint64_t)(R / 16), (cuuint64_t)B};
    cuuint64_t str[3] = {(cuuint64_t)R * 8, 128, (cuuint64_t)(S * R) * 8};
    cuuint32_t box[4] = {16, 16, 8, 1};
    if (!make_map(&tmX4, X, 4, dims, str, box)) return cudaErrorInvalidValue;
  }
  {
    cuuint64_t dims[3] = {16, (cuuint64_t)S, (cuuint64_t)(C::BNP / 16)};
    cuuint64_t str[2] = {(cuuint64_t)C::BNP * 8, 128};
    cuuint32_t box[3] = {16, 16, (cuuint32_t)(C::BNP / 16)};
    if (!make_map(&tmF, Fp, 3, dims, str, box)) return cudaErrorInvalidValue;
  }
  const int smem = C::smem(stages) + red_bytes;
  int sms = 148;
  {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const long long nunits = fa.n_o * fa.nh * fa.nP;
  const long long grid = nunits < sms ? nunits : sms;
  static const bool dbg = getenv("CPPP_DEBUG_TTM") != nullptr;
  if (dbg)
    fprintf(stderr, "ttm fused B %lld S %lld R %lld K %d: units %lld (run %lld) grid %lld stages %d\n",
            (long long)B, (long long)S, (long long)R, K, nunits, (long long)fa.run, grid, stages);
  cudaError_t e = launch_pdl(ttm_fused_kernel<NT>, dim3((unsigned)grid), dim3(NTHREADS), smem, st, tmF, tmX4,
                             R / BM, (int)S, K, stages, counter, fa);
  note_launch();
  return e;
}

template <int NT = 1>
cudaError_t dispatch_fused(int nt, const double* X, int64_t B, int64_t S, int64_t R, const double* Fp,
                           int K, unsigned long long* counter, const FusedArgs& fa, cudaStream_t st) {
  if constexpr (NT > 16) {
    return cudaErrorInvalidValue;
  } else {
    if (nt == NT) return run_fused<NT>(X, B, S, R, Fp, K, counter, fa, st);
    return dispatch_fused<NT + 1>(nt, X, B, S, R, Fp, K, counter, fa, st);
  }
}

__global__ void sum_parts_kernel(const double* __restrict__ part, int np, int64_t n, double* __restrict__ out) {
  pdl_wait();
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    double s = __ldcs(part + e);
    for (int q = 1; q < np; ++q) s += __ldcs(part + q * n + e);
    out[e] = s;
  }
}

}  // namespace

bool ttm_fused_ok(int64_t B, int64_t S, int64_t R, int K, int64_t sf) {
  return ttm_dmma_supported(B, S, R, K) && sf % BM == 0 && R % BM == 0;
}

cudaError_t launch_ttm_fused(const double* X, int64_t B, int64_t S, int64_t R, int K, const double* Fpad,
                             const TtmFused& f, cudaStream_t st) {
  double* ctl = const_cast<double*>(Fpad);
  unsigned long long* counter = reinterpret_cast<unsigned long long*>(ctl);
  FusedArgs fa;
  fa.o_str = f.o_str;
  fa.l_str = f.l_str;
  fa.n_o = f.n_o;
  fa.n_l = f.n_l;
  fa.sf = f.sf;
  fa.nh = f.sf / BM;
  fa.nP = f.nP;
  fa.run = (f.n_l + f.nP - 1) / f.nP;
  fa.Af = f.Af;
  fa.Al = f.Al;
  fa.fast = f.fast;
  fa.fl_o = f.fl_o;
  fa.fl_l = f.fl_l;
  fa.loop = f.loop;
  if (fa.run >= 65536) return cudaErrorInvalidValue;
  return dispatch_fused(static_cast<int>((K + 7) / 8), X, B, S, R, ctl + TTM_CTL + TTM_PART, K, counter, fa, st);
}

cudaError_t launch_sum_parts(const double* part, int np, int64_t n, double* out, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  int64_t blocks = (n + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  cudaError_t e = launch_pdl(sum_parts_kernel, dim3((unsigned)blocks), dim3(256), 0, st, part, np, n, out);
  note_launch();
  return e;
}

bool ttm_dmma_supported(int64_t B, int64_t S, int64_t R, int K) {
  if (K < 1 || K > 128) return false;
  if (S % 2 != 0) return false;                 // TMA: row strides multiple of 16 bytes
  if (R > 1 && R % 2 != 0) return false;
  if (S >= (1ll << 31) || B >= (1ll << 31) || R >= (1ll << 31)) return false;
  // (shape only: the workspace plan must not depend on the machine; a missing tensor-map encoder
  // makes the launch fail -- make_map -- rather than silently change the plan)
  return true;
}

bool ttm_skinny_ok(int64_t S, int64_t R, int K) {
  (void)S;
  (void)R;
  return K <= 16;
}

cudaError_t launch_ttm_simt(const double* X, int64_t B, int64_t S, int64_t R, const double* F,
                            int K, double* out, cudaStream_t st) {
  const int64_t total = B * R * K;
  if (total == 0) return cudaSuccess;
  static const bool no_skinny = getenv("CPPP_NO_SKINNY") != nullptr;   // A/B: the generic kernel
  if (!no_skinny && ttm_skinny_ok(S, R, K)) {
    if (K <= 2) return run_skinny<2>(X, B, S, R, F, K, out, st);
    if (K <= 4) return run_skinny<4>(X, B, S, R, F, K, out, st);
    if (K <= 8) return run_skinny<8>(X, B, S, R, F, K, out, st);
    return run_skinny<16>(X, B, S, R, F, K, out, st);
  }
  int64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 64) blocks = 148 * 64;
  ttm_simt_kernel<<<(unsigned)blocks, 256, 0, st>>>(X, B, S, R, F, K, out);
  note_launch();
  return cudaGetLastError();
}

bool ttm_uses_dmma(int64_t B, int64_t S, int64_t R, int K, bool force_simt) {
  return !force_simt && ttm_dmma_supported(B, S, R, K);
}


bool ttm_direct_ok(const double* F, int K) {
  return F != nullptr && K % 2 == 0 && (reinterpret_cast<uintptr_t>(F) & 15) == 0;
}

// padded factor width for K: 16-column TMA boxes
int ttm_ld(int K) { return ((((K + 7) / 8) * 8 + 15) / 16) * 16; }


cudaError_t ttm_prepare(int64_t S, const double* F, int K, double* Fpad, cudaStream_t st) {
  return launch_pad_rows(F, S, K, Fpad + TTM_CTL + TTM_PART, ttm_ld(K), st);
}

// Khatri-Rao product of the factors of consecutive modes m_0 < ... < m_{h-1} (row-major over
// (x_0, ..., x_{h-1}), last fastest; product in ascending j), written straight into the padded
// factor area (ld = ttm_ld(K), zero columns past K): the multi-mode first level of the
// dimension tree contracts X_(m_0..m_{h-1}) with it in one GEMM (P:78-80 with the contracted
// modes of a half taken together; the MTTKRP definition).
__global__ void krp_kernel(KrpArgs a, double* __restrict__ out) {
  pdl_wait();
  const int64_t total = a.rows * a.ld;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = e / a.ld;
    const int k = static_cast<int>(e - row * a.ld);
    if (k >= a.K) {
      out[e] = 0.0;
      continue;
    }
    int64_t x[CPPP_MAX_ORDER_];
    int64_t r = row;
    for (int j = a.nm - 1; j >= 0; --j) {
      x[j] = r % a.dims[j];
      r /= a.dims[j];
    }
    double v = 1.0;
    for (int j = 0; j < a.nm; ++j) v *= __ldg(a.F[j] + x[j] * a.K + k);
    out[e] = v;
  }
}

cudaError_t ttm_prepare_krp(const KrpArgs& args, double* Fpad, cudaStream_t st) {
  KrpArgs a = args;
  a.ld = ttm_ld(a.K);
  a.rows = 1;
  for (int j = 0; j < a.nm; ++j) a.rows *= a.dims[j];
  const int64_t total = a.rows * a.ld;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  cudaError_t e = launch_pdl(krp_kernel, dim3((unsigned)blocks), dim3(256), 0, st, a,
                             Fpad + TTM_CTL + TTM_PART);
  note_launch();
  return e;
}

// Kronecker product of factor matrices (Tucker's multi-mode contraction):
// out[(x_0 .. x_{h-1})][(z_0 .. z_{h-1})] = Π_j F_j[x_j][z_j], both multi-indices row-major
__global__ void kron_kernel(KronArgs a, double* __restrict__ out) {
  pdl_wait();
  const int64_t total = a.rows * a.ld;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = e / a.ld;
    int col = static_cast<int>(e - row * a.ld);
    if (col >= a.cols) {
      out[e] = 0.0;
      continue;
    }
    int64_t x[CPPP_MAX_ORDER_];
    int z[CPPP_MAX_ORDER_];
    int64_t r = row;
    for (int j = a.nm - 1; j >= 0; --j) {
      x[j] = r % a.dims[j];
      r /= a.dims[j];
      z[j] = col % a.ranks[j];
      col /= a.ranks[j];
    }
    double v = 1.0;
    for (int j = 0; j < a.nm; ++j) v *= __ldg(a.F[j] + x[j] * a.ranks[j] + z[j]);
    out[e] = v;
  }
}

cudaError_t ttm_prepare_kron(const KronArgs& args, double* Fpad, cudaStream_t st) {
  KronArgs a = args;
  a.rows = 1;
  a.cols = 1;
  for (int j = 0; j < a.nm; ++j) {
    a.rows *= a.dims[j];
    a.cols *= a.ranks[j];
  }
  a.ld = ttm_ld(a.cols);
  const int64_t total = a.rows * a.ld;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  cudaError_t e = launch_pdl(kron_kernel, dim3((unsigned)blocks), dim3(256), 0, st, a,
                             Fpad + TTM_CTL + TTM_PART);
  note_launch();
  return e;
}

size_t ttm_scratch_doubles(int64_t S) { return TTM_CTL + TTM_PART + static_cast<size_t>(S) * 128; }

cudaError_t launch_ttm_padded(const double* X, int64_t B, int64_t S, int64_t R, int K, double* out,
                              const double* Fpad, cudaStream_t st) {
  return launch_ttm_core(X, B, S, R, nullptr, K, out, Fpad, false, st);
}

cudaError_t launch_ttm_core(const double* X, int64_t B, int64_t S, int64_t R, const double* F,
                            int K, double* out, const double* Fpad, bool force_simt,
                            cudaStream_t st, TtmOpts topt) {
  if (B * R * K == 0) return cudaSuccess;
  if (!ttm_uses_dmma(B, S, R, K, force_simt)) return launch_ttm_simt(X, B, S, R, F, K, out, st);
  double* ctl = const_cast<double*>(Fpad);
  unsigned long long* counter = reinterpret_cast<unsigned long long*>(ctl);
  unsigned int* tickets = reinterpret_cast<unsigned int*>(ctl + 8);
  double* part = ctl + TTM_CTL;
  const double* Fp = topt.direct_factor ? F : ctl + TTM_CTL + TTM_PART;
  const int nt = (K + 7) / 8;
  if (R == 1)
    return dispatch_nt<false>(nt, X, B, S, R, Fp, K, out, counter, tickets, part, st, topt);
  return dispatch_nt<true>(nt, X, B, S, R, Fp, K, out, counter, tickets, part, st, topt);
}

cudaError_t launch_ttm(const double* X, int64_t B, int64_t S, int64_t R, const double* F, int K,
                       double* out, double* Fpad, bool force_simt, cudaStream_t st) {
  if (B * R * K == 0) return cudaSuccess;
  if (ttm_uses_dmma(B, S, R, K, force_simt)) {
    cudaError_t e = ttm_prepare(S, F, K, Fpad, st);
    if (e != cudaSuccess) return e;
  }
  return launch_ttm_core(X, B, S, R, F, K, out, Fpad, force_simt, st);
}

}  // namespace cppp
