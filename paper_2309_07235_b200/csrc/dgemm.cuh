// Knob-driven fp64 GEMM for sm_100a:  C (+)= (+/-) A[MxK] * B[KxN]
//
// Replaces the reference's matmul_tiled (kernels.cpp:91-111) and serves the
// LU trailing update (kernels.cpp:205-216) and the Cholesky update
// (kernels.cpp:273-286, right-looking form, B given as N x K = "NT").
//
// Schedule (per CTA, mirrors the reference's (yo, xo) outer tile loops):
//   * one CTA owns one output REGION of reg_y x reg_x elements — the knob
//     (fy, fx) of the reference loop nest; sub-atom regions (< 8) are packed
//     into the 8x8 DMMA atom by the host launcher;
//   * the region is swept in BM x BN tile steps; each step is a full-K
//     reduction (the reference's k loop) in BK=16 chunks;
//   * warp 'NCW' is a TMA producer (one elected lane): each stage is one A box
//     [BM x 16] and the B box(es), 128B-swizzled, completion on a full
//     mbarrier; consumer warps release a stage through an empty mbarrier;
//   * consumer warps own WTM x WTN warp tiles of 8x8x4 DMMA atoms with
//     register accumulators (fp64 has no TMEM/UMMA path on sm_100a).
//
// Bank-conflict-free fragment loads: the k index a lane feeds in DMMA step s
// is K(s,t) = 8(s>>1) + 2t + (s&1) (so A/B^T pairs are one LDS.128) and the
// A (and B^T) fragment row g maps to tile row (g>>1) + 4(g&1) inside each
// 8-row group; with the 128B swizzle every quarter-warp hits 8 distinct
// 16-byte chunks.  Any permutation of the k order is legal: each output
// element still receives every product exactly once, accumulated by DMMA.
#pragma once
#include <climits>
#include <cstdint>

#include "tt_ptx.cuh"

namespace tt {

constexpr int kBK = 16;

struct GemmArgs {
  double* c;       // output view origin: element (0,0) of the M x N view
  long long ldc;
  int M, N, K;
  int a_r0, a_c0;  // A view origin inside the A tensor map (row, col)
  int b_r0, b_c0;  // NN: (k-row, n-col) of B; NT: (n-row, k-col) of B^T
  int reg_y, reg_x;
  int nreg_x;
  int klo;         // 1: the A (and B^T) k origin was moved one column left to an even,
                   //    16-byte-aligned TMA coordinate; k' = 0 is masked (K' = K + 1)
  int alpha_neg;   // 1: accumulate -A*B
  int beta;        // 1: accumulators start from C (C += ...), 0: from zero
  int lower;       // 1: only write view elements with i + diag_off >= j
  int diag_off;
  int c_tma;       // beta=1 only: the producer TMA-prefetches each tile's C block
                   // (box BM x (BN+2) from an even column, `c_sh` = view column
                   // shift of the map) so the accumulator init never waits on
                   // global-memory latency
  int c_sh;
};

template <int BM, int BN, bool BT>
struct GemmShape {
  // Warp tiles up to 32 x 64 (64 fp64 accumulators per lane).  A DMMA warp
  // carries a fixed issue stall after every DMMA, so one consumer warp per SM
  // sub-partition cannot keep the fp64 tensor pipe busy next to its fragment
  // loads (72% pipe-active with 4 warps of 32 x 64, profiles/ncu_r02_3mm_xl.txt):
  // tiles of >= 128 x 64 run 8 consumer warps (two per sub-partition) —
  // 4 x 2 warps of 32 x 64 (128 x 128), 4 x 2 of 32 x 32 (128 x 64),
  // 2 x 4 of 32 x 32 (64 x 128) — and 64 x 64 runs 2 x 2 of 32 x 32.
  static constexpr int WTM = BM < 32 ? BM : 32;
  static constexpr int WGM = BM / WTM;
  static constexpr int WGN = (BM * BN >= 128 * 64) ? 8 / WGM
                             : (BM == 64 && BN == 64) ? 2
                             : (BN < 64 ? 1 : BN / 64);
  static constexpr int WTN = BN / WGN;
  static constexpr int MF = WTM / 8;
  static constexpr int NF = WTN / 8;
  static constexpr int NCW = WGM * WGN;
  // 8 consumer warps: no separate producer warp (ptxas budgets registers
  // per 4-warp group: a 9th warp would cap every thread at 168 registers);
  // consumer warp 0's lane 0 issues the TMA loads in line, STAGES-1 ahead.
  // These variants have no C prefetch (beta = 1 loads C directly).
  static constexpr bool INLINE_TMA = NCW == 8;
  static constexpr int THREADS = (NCW + (INLINE_TMA ? 0 : 1)) * 32;
  static_assert(NCW <= 8, "at most 8 consumer warps");
  static constexpr int STAGES = (BM + BN) >= 256 ? 5 : (BM + BN) >= 192 ? 4 : 6;
  static constexpr int A_BYTES = BM * kBK * 8;
  static constexpr int B_COLS = BT ? BN : (BN < 16 ? 16 : BN);  // NN boxes are 16 wide
  static constexpr int B_BYTES = B_COLS * kBK * 8;
  static constexpr int NBOX_B = BT ? 1 : B_COLS / 16;
  // NN tiles whose first B column is odd start their boxes one column left
  // (TMA boxes must start 16-byte aligned) and need one extra box when BN >= 16.
  static constexpr int B_ALLOC = BT ? B_BYTES : B_BYTES + (BN >= 16 ? kBK * 128 : 0);
  static constexpr int STAGE_BYTES = A_BYTES + B_ALLOC;
  static constexpr int C_LD = BN + 2;  // doubles per row of the C prefetch box
  static constexpr int C_BYTES = BM * C_LD * 8;
  static constexpr int SMEM = STAGES * STAGE_BYTES + C_BYTES + 2 * STAGES * 8 + 16 + 1024;
  // without the C prefetch buffer (beta = 0, or c_tma off): the barriers
  // move to its place, the kernel never touches sC
  static constexpr int SMEM_NOC = STAGES * STAGE_BYTES + 2 * STAGES * 8 + 16 + 1024;
  static constexpr int SMEM_OPT = SMEM <= 227 * 1024 ? SMEM : SMEM_NOC;
};

// Byte offset of (row, 16B-chunk) in a tile of 128-byte rows written by TMA
// with CU_TENSOR_MAP_SWIZZLE_128B (tile base 1024-byte aligned).
__device__ __forceinline__ int swz(int row, int chunk) {
  return row * 128 + ((chunk ^ (row & 7)) << 4);
}

template <int BM, int BN, bool BT>
__global__ void __launch_bounds__(GemmShape<BM, BN, BT>::THREADS, 1)
    dgemm_kernel(const __grid_constant__ CUtensorMap tmA,
                 const __grid_constant__ CUtensorMap tmB,
                 const __grid_constant__ CUtensorMap tmC, const GemmArgs p) {
  using S = GemmShape<BM, BN, BT>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~static_cast<uintptr_t>(1023));
  const bool c_tma = !S::INLINE_TMA && p.beta && p.c_tma;
  double* sC = reinterpret_cast<double*>(smem + S::STAGES * S::STAGE_BYTES);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S::STAGES * S::STAGE_BYTES +
                                               (c_tma ? S::C_BYTES : 0));
  uint64_t* empty = full + S::STAGES;
  uint64_t* cfull = empty + S::STAGES;
  uint64_t* cempty = cfull + 1;

  const int rid = blockIdx.x;
  const int ry = rid / p.nreg_x;
  const int rx = rid - ry * p.nreg_x;
  const int y0 = ry * p.reg_y, x0 = rx * p.reg_x;
  const int y1 = min(y0 + p.reg_y, p.M), x1 = min(x0 + p.reg_x, p.N);
  if (p.lower && (y1 - 1 + p.diag_off < x0)) return;  // region strictly above the diagonal
  const int nty = (y1 - y0 + BM - 1) / BM;
  const int ntx = (x1 - x0 + BN - 1) / BN;
  const int kend = p.K + p.klo;  // k' range [klo, kend) is the operand's K
  const int nk = (kend + kBK - 1) / kBK;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
#pragma unroll
    for (int s = 0; s < S::STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], S::NCW);
    }
    mbar_init(cfull, 1);
    mbar_init(cempty, S::NCW);
    fence_mbar_init();
  }
  __syncthreads();

  if (!S::INLINE_TMA && warp == S::NCW) {  // ---------------- TMA producer ----------------
    if (lane == 0) {
      prefetch_tmap(&tmA);
      prefetch_tmap(&tmB);
      if (c_tma) prefetch_tmap(&tmC);
      int stage = 0;
      uint32_t phase = 0;
      uint32_t cphase = 0;
      for (int ty = 0; ty < nty; ++ty) {
        const int ty0 = y0 + ty * BM;
        const int ty1 = min(ty0 + BM, y1);
        for (int tx = 0; tx < ntx; ++tx) {
          const int tx0 = x0 + tx * BN;
          if (p.lower && (ty1 - 1 + p.diag_off < tx0)) continue;
          if (c_tma) {  // C block of this tile, once the consumers read the last one
            mbar_wait(cempty, cphase ^ 1);
            mbar_arrive_expect_tx(cfull, S::C_BYTES);
            const int cc0 = p.c_sh + tx0;
            tma_load_2d(sC, &tmC, cfull, cc0 & ~1, ty0);
            cphase ^= 1;
          }
          const int bs = BT ? 0 : ((p.b_c0 + tx0) & 1);  // NN column shift of this tile
          const int nbox = S::NBOX_B + ((bs && BN >= 16) ? 1 : 0);
          const uint32_t tx_bytes = S::A_BYTES + (BT ? S::B_BYTES : nbox * (kBK * 128));
          for (int kc = 0; kc < nk; ++kc) {
            mbar_wait(&empty[stage], phase ^ 1);
            uint8_t* sa = smem + stage * S::STAGE_BYTES;
            uint8_t* sb = sa + S::A_BYTES;
            mbar_arrive_expect_tx(&full[stage], tx_bytes);
            tma_load_2d(sa, &tmA, &full[stage], p.a_c0 + kc * kBK, p.a_r0 + ty0);
            if (BT) {
              tma_load_2d(sb, &tmB, &full[stage], p.b_c0 + kc * kBK, p.b_r0 + tx0);
            } else {
              for (int j = 0; j < nbox; ++j)
                tma_load_2d(sb + j * (kBK * 128), &tmB, &full[stage], p.b_c0 + tx0 - bs + 16 * j,
                            p.b_r0 + kc * kBK);
            }
            if (++stage == S::STAGES) {
              stage = 0;
              phase ^= 1;
            }
          }
        }
      }
    }
    return;
  }

  // ---------------- DMMA consumers ----------------
  constexpr int MF = S::MF, NF = S::NF;
  const int wm = warp / S::WGN, wn = warp - (warp / S::WGN) * S::WGN;
  const int g = lane >> 2, t = lane & 3;
  const int rperm = (g >> 1) + 4 * (g & 1);
  const double sgn = p.alpha_neg ? -1.0 : 1.0;
  int stage = 0;
  uint32_t phase = 0;
  uint32_t cphase = 0;

  // in-line producer (INLINE_TMA; never with the C prefetch): the chunk
  // stream of the tile loop below, issued STAGES-1 chunks ahead; issuing
  // chunk g+STAGES-1 reuses chunk g-1's slot (every warp released it)
  int q_t = 0, q_kc = 0, q_stage = 0;
  uint32_t q_phase = 0;
  auto issue_next = [&]() {
    for (; q_t < nty * ntx; ++q_t, q_kc = 0) {
      const int ty = q_t / ntx, tx = q_t - (q_t / ntx) * ntx;
      const int ty0 = y0 + ty * BM, tx0 = x0 + tx * BN;
      if (p.lower && (min(ty0 + BM, y1) - 1 + p.diag_off < tx0)) continue;
      const int bs = BT ? 0 : ((p.b_c0 + tx0) & 1);
      const int nbox = S::NBOX_B + ((bs && BN >= 16) ? 1 : 0);
      const uint32_t tx_bytes = S::A_BYTES + (BT ? S::B_BYTES : nbox * (kBK * 128));
      mbar_wait(&empty[q_stage], q_phase ^ 1);
      uint8_t* sa = smem + q_stage * S::STAGE_BYTES;
      uint8_t* sb = sa + S::A_BYTES;
      mbar_arrive_expect_tx(&full[q_stage], tx_bytes);
      tma_load_2d(sa, &tmA, &full[q_stage], p.a_c0 + q_kc * kBK, p.a_r0 + ty0);
      if (BT) {
        tma_load_2d(sb, &tmB, &full[q_stage], p.b_c0 + q_kc * kBK, p.b_r0 + tx0);
      } else {
        for (int j = 0; j < nbox; ++j)
          tma_load_2d(sb + j * (kBK * 128), &tmB, &full[q_stage], p.b_c0 + tx0 - bs + 16 * j,
                      p.b_r0 + q_kc * kBK);
      }
      if (++q_stage == S::STAGES) {
        q_stage = 0;
        q_phase ^= 1;
      }
      if (++q_kc == nk) {
        q_kc = 0;
        ++q_t;
      }
      return;
    }
  };
  const bool producer_lane = S::INLINE_TMA && warp == 0 && lane == 0;
  if (producer_lane) {
    prefetch_tmap(&tmA);
    prefetch_tmap(&tmB);
    for (int i = 0; i + 1 < S::STAGES; ++i) issue_next();
  }

  for (int ty = 0; ty < nty; ++ty) {
    const int ty0 = y0 + ty * BM;
    const int ty1 = min(ty0 + BM, y1);
    for (int tx = 0; tx < ntx; ++tx) {
      const int tx0 = x0 + tx * BN;
      if (p.lower && (ty1 - 1 + p.diag_off < tx0)) continue;
      const int bs = BT ? 0 : ((p.b_c0 + tx0) & 1);

      double acc[MF][NF][2];
#pragma unroll
      for (int mf = 0; mf < MF; ++mf)
#pragma unroll
        for (int nf = 0; nf < NF; ++nf) {
          acc[mf][nf][0] = 0.0;
          acc[mf][nf][1] = 0.0;
        }
      if (c_tma) {
        mbar_wait(cfull, cphase);
        cphase ^= 1;
        const int cs = (p.c_sh + tx0) & 1;
#pragma unroll
        for (int mf = 0; mf < MF; ++mf) {
          const int rl = wm * S::WTM + mf * 8 + rperm;
#pragma unroll
          for (int nf = 0; nf < NF; ++nf)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int cl = wn * S::WTN + nf * 8 + (BT ? t + 4 * h : 2 * t + h);
              acc[mf][nf][h] = sC[rl * S::C_LD + cl + cs];
            }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(cempty);
      } else if (p.beta) {
#pragma unroll
        for (int mf = 0; mf < MF; ++mf) {
          const int r = ty0 + wm * S::WTM + mf * 8 + rperm;
          if (r < ty1) {
            const double* crow = p.c + static_cast<long long>(r) * p.ldc;
#pragma unroll
            for (int nf = 0; nf < NF; ++nf)
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int cc = tx0 + wn * S::WTN + nf * 8 + (BT ? t + 4 * h : 2 * t + h);
                if (cc < x1) acc[mf][nf][h] = crow[cc];
              }
          }
        }
      }

      for (int kc = 0; kc < nk; ++kc) {
        mbar_wait(&full[stage], phase);
        if (producer_lane) issue_next();
        const uint8_t* sa = smem + stage * S::STAGE_BYTES;
        const uint8_t* sb = sa + S::A_BYTES;
        // chunk-local valid k' window [klo_c, kvalid): masks the aligned-origin
        // column (first chunk) and the K tail (last chunk)
        const int klo_c = kc == 0 ? p.klo : 0;
        const int kvalid = kend - kc * kBK;
        const bool tail = kvalid < kBK || klo_c > 0;

        // Two k-pairs per chunk: pair sp feeds DMMA steps s = 2sp, 2sp+1 with
        // k = 8sp + 2t + h.  Large warp tiles keep the pair loop rolled so
        // only one pair of operand fragments is live next to the accumulators.
#pragma unroll(S::MF * S::NF >= 32 ? 1 : 2)
        for (int sp = 0; sp < 2; ++sp) {
          double a[MF][2];
#pragma unroll
          for (int mf = 0; mf < MF; ++mf) {
            const int row = wm * S::WTM + mf * 8 + rperm;
            const double2 v = *reinterpret_cast<const double2*>(sa + swz(row, sp * 4 + t));
            a[mf][0] = v.x * sgn;
            a[mf][1] = v.y * sgn;
          }
          double b[2][NF];
          if (BT) {
#pragma unroll
            for (int nf = 0; nf < NF; ++nf) {
              const int row = wn * S::WTN + nf * 8 + rperm;
              const double2 v = *reinterpret_cast<const double2*>(sb + swz(row, sp * 4 + t));
              b[0][nf] = v.x;
              b[1][nf] = v.y;
            }
          } else {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int krow = 8 * sp + 2 * t + h;
#pragma unroll
              for (int nf = 0; nf < NF; ++nf) {
                const int cn = wn * S::WTN + nf * 8 + g + bs;
                const int cc = cn & 15;
                b[h][nf] = *reinterpret_cast<const double*>(
                    sb + (cn >> 4) * (kBK * 128) + swz(krow, cc >> 1) + (cc & 1) * 8);
              }
            }
          }
          if (tail) {  // zero the k >= K lanes of both operands
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int kk = 8 * sp + 2 * t + h;
              if (kk >= kvalid || kk < klo_c) {
#pragma unroll
                for (int mf = 0; mf < MF; ++mf) a[mf][h] = 0.0;
#pragma unroll
                for (int nf = 0; nf < NF; ++nf) b[h][nf] = 0.0;
              }
            }
          }
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int mf = 0; mf < MF; ++mf)
#pragma unroll
              for (int nf = 0; nf < NF; ++nf)
                dmma_8x8x4(acc[mf][nf][0], acc[mf][nf][1], a[mf][h], b[h][nf]);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stage]);
        if (++stage == S::STAGES) {
          stage = 0;
          phase ^= 1;
        }
      }

      // epilogue: predicated stores inside the region / view / triangle
#pragma unroll
      for (int mf = 0; mf < MF; ++mf) {
        const int r = ty0 + wm * S::WTM + mf * 8 + rperm;
        if (r < ty1) {
          double* crow = p.c + static_cast<long long>(r) * p.ldc;
#pragma unroll
          for (int nf = 0; nf < NF; ++nf)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const int cc = tx0 + wn * S::WTN + nf * 8 + (BT ? t + 4 * h : 2 * t + h);
              if (cc < x1 && (!p.lower || r + p.diag_off >= cc)) crow[cc] = acc[mf][nf][h];
            }
        }
      }
    }
  }
}

}  // namespace tt
