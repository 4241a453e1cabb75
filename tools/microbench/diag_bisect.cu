#include <cstdio>
#include <vector>
#include "../../paper_2309_07235_b200/csrc/dag_factor.cu"
namespace tt { namespace dag { namespace {
template <bool CHOL>
__device__ __forceinline__ void tf_full(double* __restrict__ dk, long long ld, int T, int gcol,
                                            int* info, double* pbuf, double* rk,
                                            unsigned long long* ph, double* solve) {
  // pbuf parity block: [0,64) pivot row (LU), [64,128) column k, [128] 1/pivot, [129] l_kk
  // rk[c]: 1/pivot of column c (LU) or 1/l_cc (Cholesky); rk[64 + c]: l_cc
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i0 = 8 * w;
  const bool wide = T > 32;
  double x[8][2];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int i = i0 + q;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = lane + 32 * h;
      x[q][h] = (i < T && c < T && (!CHOL || c <= i))
                    ? __ldcg(dk + static_cast<long long>(i) * ld + c) : 0.0;
    }
  }
  // publish step 0: column 0 (+ row 0 for LU) and the pivot's reciprocal
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < 8; ++q) pbuf[64 + i0 + q] = x[q][0];
  }
  if (w == 0) {
    if (!CHOL) {
      pbuf[lane] = x[0][0];
      pbuf[lane + 32] = x[0][1];
    }
    if (lane == 0) {
      const double d = x[0][0];
      if (!CHOL) {
        if (fabs(d) < 1e-300) atomicMin(info, gcol);  // kernels.cpp:187-190
        rk[0] = pbuf[128] = rcp_nr(d);
      } else {
        if (d <= 0.0) atomicMin(info, gcol);  // kernels.cpp:297-302 (NaN passes)
        const double l0 = sqrt(d);
        rk[64] = l0;
        rk[0] = pbuf[128] = rcp_nr(l0);
      }
    }
  }
  __syncthreads();
  if (ph && threadIdx.x == 0) ph[0] = globaltimer();
  for (int k = 0; k < T; ++k) {
    const double* cb = pbuf + (k & 1) * kPB;
    double* nb = pbuf + ((k + 1) & 1) * kPB;
    const int k1 = k + 1;
    if (i0 + 7 > k && i0 < T) {  // warp-uniform: this warp still has live rows > k
      // x_ij -= a_ik * (u_kj / pivot): the reciprocal is folded into the
      // operand row (Cholesky: u_kj = a_jk, scaled by 1/l_kk^2), so a step
      // is one DFMA per element; the multipliers are formed at the end.
      const double r = cb[128];
      const double rs = CHOL ? r * r : r;
      double a[8];
#pragma unroll
      for (int q = 0; q < 8; q += 2) {
        const double2 v = *reinterpret_cast<const double2*>(cb + 64 + i0 + q);
        a[q] = v.x;
        a[q + 1] = v.y;
      }
      if (i0 <= k) {  // the warp holding row k: rows <= k are final
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (i0 + q <= k) a[q] = 0.0;
      }
      const double* src = CHOL ? cb + 64 : cb;
      const double u0 = lane > k ? src[lane] * rs : 0.0;
      if (wide) {
        const double u1 = lane + 32 > k ? src[lane + 32] * rs : 0.0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          x[q][0] = fma(-a[q], u0, x[q][0]);
          x[q][1] = fma(-a[q], u1, x[q][1]);
        }
      } else {
#pragma unroll
        for (int q = 0; q < 8; ++q) x[q][0] = fma(-a[q], u0, x[q][0]);
      }
      if (k1 < T) {
        // next pivot row k+1 (LU) and its reciprocal: the owner warp (a
        // uniform jump on q1 = (k+1) % 8 instead of a select chain)
        if ((k1 >> 3) == w) {
          double v0, v1;
          switch (k1 & 7) {
#define TT_ROW(Q)     \
  case Q:             \
    v0 = x[Q][0];     \
    v1 = x[Q][1];     \
    break;
            TT_ROW(0) TT_ROW(1) TT_ROW(2) TT_ROW(3) TT_ROW(4) TT_ROW(5) TT_ROW(6) default: TT_ROW(7)
#undef TT_ROW
          }
          if (lane == (k1 & 31)) {
            const double d = k1 >= 32 ? v1 : v0;
            if (!CHOL) {
              rk[k1] = nb[128] = rcp_nr(d);
              if (fabs(d) < 1e-300) atomicMin(info, gcol + k1);  // kernels.cpp:187-190
            } else {
              const double l1 = sqrt(d);
              rk[64 + k1] = l1;
              rk[k1] = nb[128] = rcp_nr(l1);
              if (d <= 0.0) atomicMin(info, gcol + k1);  // kernels.cpp:297-302
            }
          }
          if (!CHOL) {
            nb[lane] = v0;
            nb[lane + 32] = v1;
          }
        }
        // column k+1 of my rows (the lane holding it)
        if (lane == (k1 & 31)) {
          if (k1 >= 32) {
#pragma unroll
            for (int q = 0; q < 8; q += 2)
              *reinterpret_cast<double2*>(nb + 64 + i0 + q) = make_double2(x[q][1], x[q + 1][1]);
          } else {
#pragma unroll
            for (int q = 0; q < 8; q += 2)
              *reinterpret_cast<double2*>(nb + 64 + i0 + q) = make_double2(x[q][0], x[q + 1][0]);
          }
        }
      }
    }
    __syncthreads();
  }
  if (ph && threadIdx.x == 0) ph[1] = globaltimer();
  // multipliers below the diagonal (and l_cc on it for Cholesky), then store
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int i = i0 + q;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = lane + 32 * h;
      double v = x[q][h];
      if (c < i) v *= rk[c];
      if (CHOL && c == i) v = rk[64 + c];
      if (i < T && c < T && (!CHOL || c <= i)) dk[static_cast<long long>(i) * ld + c] = v;
    }
  }
  // per-column reciprocals of the diagonal (1/u_cc, Cholesky 1/l_cc) for the
  // TRSM tasks' 8x8 block inverses
  if (threadIdx.x < 64) solve[threadIdx.x] = rk[threadIdx.x];
}


template <bool CHOL>
__device__ __forceinline__ void tf_no_zeroing(double* __restrict__ dk, long long ld, int T, int gcol,
                                            int* info, double* pbuf, double* rk,
                                            unsigned long long* ph, double* solve) {
  // pbuf parity block: [0,64) pivot row (LU), [64,128) column k, [128] 1/pivot, [129] l_kk
  // rk[c]: 1/pivot of column c (LU) or 1/l_cc (Cholesky); rk[64 + c]: l_cc
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i0 = 8 * w;
  const bool wide = T > 32;
  double x[8][2];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int i = i0 + q;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = lane + 32 * h;
      x[q][h] = (i < T && c < T && (!CHOL || c <= i))
                    ? __ldcg(dk + static_cast<long long>(i) * ld + c) : 0.0;
    }
  }
  // publish step 0: column 0 (+ row 0 for LU) and the pivot's reciprocal
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < 8; ++q) pbuf[64 + i0 + q] = x[q][0];
  }
  if (w == 0) {
    if (!CHOL) {
      pbuf[lane] = x[0][0];
      pbuf[lane + 32] = x[0][1];
    }
    if (lane == 0) {
      const double d = x[0][0];
      if (!CHOL) {
        if (fabs(d) < 1e-300) atomicMin(info, gcol);  // kernels.cpp:187-190
        rk[0] = pbuf[128] = rcp_nr(d);
      } else {
        if (d <= 0.0) atomicMin(info, gcol);  // kernels.cpp:297-302 (NaN passes)
        const double l0 = sqrt(d);
        rk[64] = l0;
        rk[0] = pbuf[128] = rcp_nr(l0);
      }
    }
  }
  __syncthreads();
  if (ph && threadIdx.x == 0) ph[0] = globaltimer();
  for (int k = 0; k < T; ++k) {
    const double* cb = pbuf + (k & 1) * kPB;
    double* nb = pbuf + ((k + 1) & 1) * kPB;
    const int k1 = k + 1;
    if (i0 + 7 > k && i0 < T) {  // warp-uniform: this warp still has live rows > k
      // x_ij -= a_ik * (u_kj / pivot): the reciprocal is folded into the
      // operand row (Cholesky: u_kj = a_jk, scaled by 1/l_kk^2), so a step
      // is one DFMA per element; the multipliers are formed at the end.
      const double r = cb[128];
      const double rs = CHOL ? r * r : r;
      double a[8];
#pragma unroll
      for (int q = 0; q < 8; q += 2) {
        const double2 v = *reinterpret_cast<const double2*>(cb + 64 + i0 + q);
        a[q] = v.x;
        a[q + 1] = v.y;
      }

      const double* src = CHOL ? cb + 64 : cb;
      const double u0 = lane > k ? src[lane] * rs : 0.0;
      if (wide) {
        const double u1 = lane + 32 > k ? src[lane + 32] * rs : 0.0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          x[q][0] = fma(-a[q], u0, x[q][0]);
          x[q][1] = fma(-a[q], u1, x[q][1]);
        }
      } else {
#pragma unroll
        for (int q = 0; q < 8; ++q) x[q][0] = fma(-a[q], u0, x[q][0]);
      }
      if (k1 < T) {
        // next pivot row k+1 (LU) and its reciprocal: the owner warp (a
        // uniform jump on q1 = (k+1) % 8 instead of a select chain)
        if ((k1 >> 3) == w) {
          double v0, v1;
          switch (k1 & 7) {
#define TT_ROW(Q)     \
  case Q:             \
    v0 = x[Q][0];     \
    v1 = x[Q][1];     \
    break;
            TT_ROW(0) TT_ROW(1) TT_ROW(2) TT_ROW(3) TT_ROW(4) TT_ROW(5) TT_ROW(6) default: TT_ROW(7)
#undef TT_ROW
          }
          if (lane == (k1 & 31)) {
            const double d = k1 >= 32 ? v1 : v0;
            if (!CHOL) {
              rk[k1] = nb[128] = rcp_nr(d);
              if (fabs(d) < 1e-300) atomicMin(info, gcol + k1);  // kernels.cpp:187-190
            } else {
              const double l1 = sqrt(d);
              rk[64 + k1] = l1;
              rk[k1] = nb[128] = rcp_nr(l1);
              if (d <= 0.0) atomicMin(info, gcol + k1);  // kernels.cpp:297-302
            }
          }
          if (!CHOL) {
            nb[lane] = v0;
            nb[lane + 32] = v1;
          }
        }
        // column k+1 of my rows (the lane holding it)
        if (lane == (k1 & 31)) {
          if (k1 >= 32) {
#pragma unroll
            for (int q = 0; q < 8; q += 2)
              *reinterpret_cast<double2*>(nb + 64 + i0 + q) = make_double2(x[q][1], x[q + 1][1]);
          } else {
#pragma unroll
            for (int q = 0; q < 8; q += 2)
              *reinterpret_cast<double2*>(nb + 64 + i0 + q) = make_double2(x[q][0], x[q + 1][0]);
          }
        }
      }
    }
    __syncthreads();
  }
  if (ph && threadIdx.x == 0) ph[1] = globaltimer();
  // multipliers below the diagonal (and l_cc on it for Cholesky), then store
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int i = i0 + q;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = lane + 32 * h;
      double v = x[q][h];
      if (c < i) v *= rk[c];
      if (CHOL && c == i) v = rk[64 + c];
      if (i < T && c < T && (!CHOL || c <= i)) dk[static_cast<long long>(i) * ld + c] = v;
    }
  }
  // per-column reciprocals of the diagonal (1/u_cc, Cholesky 1/l_cc) for the
  // TRSM tasks' 8x8 block inverses
  if (threadIdx.x < 64) solve[threadIdx.x] = rk[threadIdx.x];
}


template <bool CHOL>
__device__ __forceinline__ void tf_no_atomic(double* __restrict__ dk, long long ld, int T, int gcol,
                                            int* info, double* pbuf, double* rk,
                                            unsigned long long* ph, double* solve) {
  // pbuf parity block: [0,64) pivot row (LU), [64,128) column k, [128] 1/pivot, [129] l_kk
  // rk[c]: 1/pivot of column c (LU) or 1/l_cc (Cholesky); rk[64 + c]: l_cc
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i0 = 8 * w;
  const bool wide = T > 32;
  double x[8][2];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int i = i0 + q;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = lane + 32 * h;
      x[q][h] = (i < T && c < T && (!CHOL || c <= i))
                    ? __ldcg(dk + static_cast<long long>(i) * ld + c) : 0.0;
    }
  }
  // publish step 0: column 0 (+ row 0 for LU) and the pivot's reciprocal
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < 8; ++q) pbuf[64 + i0 + q] = x[q][0];
  }
  if (w == 0) {
    if (!CHOL) {
      pbuf[lane] = x[0][0];
      pbuf[lane + 32] = x[0][1];
    }
    if (lane == 0) {
      const double d = x[0][0];
      if (!CHOL) {
        if (fabs(d) < 1e-300) atomicMin(info, gcol);  // kernels.cpp:187-190
        rk[0] = pbuf[128] = rcp_nr(d);
      } else {
        if (d <= 0.0) atomicMin(info, gcol);  // kernels.cpp:297-302 (NaN passes)
        const double l0 = sqrt(d);
        rk[64] = l0;
        rk[0] = pbuf[128] = rcp_nr(l0);
      }
    }
  }
  __syncthreads();
  if (ph && threadIdx.x == 0) ph[0] = globaltimer();
  for (int k = 0; k < T; ++k) {
    const double* cb = pbuf + (k & 1) * kPB;
    double* nb = pbuf + ((k + 1) & 1) * kPB;
    const int k1 = k + 1;
    if (i0 + 7 > k && i0 < T) {  // warp-uniform: this warp still has live rows > k
      // x_ij -= a_ik * (u_kj / pivot): the reciprocal is folded into the
      // operand row (Cholesky: u_kj = a_jk, scaled by 1/l_kk^2), so a step
      // is one DFMA per element; the multipliers are formed at the end.
      const double r = cb[128];
      const double rs = CHOL ? r * r : r;
      double a[8];
#pragma unroll
      for (int q = 0; q < 8; q += 2) {
        const double2 v = *reinterpret_cast<const double2*>(cb + 64 + i0 + q);
        a[q] = v.x;
        a[q + 1] = v.y;
      }
      if (i0 <= k) {  // the warp holding row k: rows <= k are final
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (i0 + q <= k) a[q] = 0.0;
      }
      const double* src = CHOL ? cb + 64 : cb;
      const double u0 = lane > k ? src[lane] * rs : 0.0;
      if (wide) {
        const double u1 = lane + 32 > k ? src[lane + 32] * rs : 0.0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          x[q][0] = fma(-a[q], u0, x[q][0]);
          x[q][1] = fma(-a[q], u1, x[q][1]);
        }
      } else {
#pragma unroll
        for (int q = 0; q < 8; ++q) x[q][0] = fma(-a[q], u0, x[q][0]);
      }
      if (k1 < T) {
        // next pivot row k+1 (LU) and its reciprocal: the owner warp (a
        // uniform jump on q1 = (k+1) % 8 instead of a select chain)
        if ((k1 >> 3) == w) {
          double v0, v1;
          switch (k1 & 7) {
#define TT_ROW(Q)     \
  case Q:             \
    v0 = x[Q][0];     \
    v1 = x[Q][1];     \
    break;
            TT_ROW(0) TT_ROW(1) TT_ROW(2) TT_ROW(3) TT_ROW(4) TT_ROW(5) TT_ROW(6) default: TT_ROW(7)
#undef TT_ROW
          }
          if (lane == (k1 & 31)) {
            const double d = k1 >= 32 ? v1 : v0;
            if (!CHOL) {
              rk[k1] = nb[128] = rcp_nr(d);
                // kernels.cpp:187-190
            } else {
              const double l1 = sqrt(d);
              rk[64 + k1] = l1;
              rk[k1] = nb[128] = rcp_nr(l1);
                // kernels.cpp:297-302
            }
          }
          if (!CHOL) {
            nb[lane] = v0;
            nb[lane + 32] = v1;
          }
        }
        // column k+1 of my rows (the lane holding it)
        if (lane == (k1 & 31)) {
          if (k1 >= 32) {
#pragma unroll
            for (int q = 0; q < 8; q += 2)
              *reinterpret_cast<double2*>(nb + 64 + i0 + q) = make_double2(x[q][1], x[q + 1][1]);
          } else {
#pragma unroll
            for (int q = 0; q < 8; q += 2)
              *reinterpret_cast<double2*>(nb + 64 + i0 + q) = make_double2(x[q][0], x[q + 1][0]);
          }
        }
      }
    }
    __syncthreads();
  }
  if (ph && threadIdx.x == 0) ph[1] = globaltimer();
  // multipliers below the diagonal (and l_cc on it for Cholesky), then store
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int i = i0 + q;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = lane + 32 * h;
      double v = x[q][h];
      if (c < i) v *= rk[c];
      if (CHOL && c == i) v = rk[64 + c];
      if (i < T && c < T && (!CHOL || c <= i)) dk[static_cast<long long>(i) * ld + c] = v;
    }
  }
  // per-column reciprocals of the diagonal (1/u_cc, Cholesky 1/l_cc) for the
  // TRSM tasks' 8x8 block inverses
  if (threadIdx.x < 64) solve[threadIdx.x] = rk[threadIdx.x];
}


template <bool CHOL>
__device__ __forceinline__ void tf_no_wide(double* __restrict__ dk, long long ld, int T, int gcol,
                                            int* info, double* pbuf, double* rk,
                                            unsigned long long* ph, double* solve) {
  // pbuf parity block: [0,64) pivot row (LU), [64,128) column k, [128] 1/pivot, [129] l_kk
  // rk[c]: 1/pivot of column c (LU) or 1/l_cc (Cholesky); rk[64 + c]: l_cc
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i0 = 8 * w;
  const bool wide = T > 32;
  double x[8][2];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int i = i0 + q;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = lane + 32 * h;
      x[q][h] = (i < T && c < T && (!CHOL || c <= i))
                    ? __ldcg(dk + static_cast<long long>(i) * ld + c) : 0.0;
    }
  }
  // publish step 0: column 0 (+ row 0 for LU) and the pivot's reciprocal
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < 8; ++q) pbuf[64 + i0 + q] = x[q][0];
  }
  if (w == 0) {
    if (!CHOL) {
      pbuf[lane] = x[0][0];
      pbuf[lane + 32] = x[0][1];
    }
    if (lane == 0) {
      const double d = x[0][0];
      if (!CHOL) {
        if (fabs(d) < 1e-300) atomicMin(info, gcol);  // kernels.cpp:187-190
        rk[0] = pbuf[128] = rcp_nr(d);
      } else {
        if (d <= 0.0) atomicMin(info, gcol);  // kernels.cpp:297-302 (NaN passes)
        const double l0 = sqrt(d);
        rk[64] = l0;
        rk[0] = pbuf[128] = rcp_nr(l0);
      }
    }
  }
  __syncthreads();
  if (ph && threadIdx.x == 0) ph[0] = globaltimer();
  for (int k = 0; k < T; ++k) {
    const double* cb = pbuf + (k & 1) * kPB;
    double* nb = pbuf + ((k + 1) & 1) * kPB;
    const int k1 = k + 1;
    if (i0 + 7 > k && i0 < T) {  // warp-uniform: this warp still has live rows > k
      // x_ij -= a_ik * (u_kj / pivot): the reciprocal is folded into the
      // operand row (Cholesky: u_kj = a_jk, scaled by 1/l_kk^2), so a step
      // is one DFMA per element; the multipliers are formed at the end.
      const double r = cb[128];
      const double rs = CHOL ? r * r : r;
      double a[8];
#pragma unroll
      for (int q = 0; q < 8; q += 2) {
        const double2 v = *reinterpret_cast<const double2*>(cb + 64 + i0 + q);
        a[q] = v.x;
        a[q + 1] = v.y;
      }
      if (i0 <= k) {  // the warp holding row k: rows <= k are final
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (i0 + q <= k) a[q] = 0.0;
      }
      const double* src = CHOL ? cb + 64 : cb;
      const double u0 = lane > k ? src[lane] * rs : 0.0;
      if (false) {
        const double u1 = lane + 32 > k ? src[lane + 32] * rs : 0.0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          x[q][0] = fma(-a[q], u0, x[q][0]);
          x[q][1] = fma(-a[q], u1, x[q][1]);
        }
      } else {
#pragma unroll
        for (int q = 0; q < 8; ++q) x[q][0] = fma(-a[q], u0, x[q][0]);
      }
      if (k1 < T) {
        // next pivot row k+1 (LU) and its reciprocal: the owner warp (a
        // uniform jump on q1 = (k+1) % 8 instead of a select chain)
        if ((k1 >> 3) == w) {
          double v0, v1;
          switch (k1 & 7) {
#define TT_ROW(Q)     \
  case Q:             \
    v0 = x[Q][0];     \
    v1 = x[Q][1];     \
    break;
            TT_ROW(0) TT_ROW(1) TT_ROW(2) TT_ROW(3) TT_ROW(4) TT_ROW(5) TT_ROW(6) default: TT_ROW(7)
#undef TT_ROW
          }
          if (lane == (k1 & 31)) {
            const double d = k1 >= 32 ? v1 : v0;
            if (!CHOL) {
              rk[k1] = nb[128] = rcp_nr(d);
              if (fabs(d) < 1e-300) atomicMin(info, gcol + k1);  // kernels.cpp:187-190
            } else {
              const double l1 = sqrt(d);
              rk[64 + k1] = l1;
              rk[k1] = nb[128] = rcp_nr(l1);
              if (d <= 0.0) atomicMin(info, gcol + k1);  // kernels.cpp:297-302
            }
          }
          if (!CHOL) {
            nb[lane] = v0;
            nb[lane + 32] = v1;
          }
        }
        // column k+1 of my rows (the lane holding it)
        if (lane == (k1 & 31)) {
          if (k1 >= 32) {
#pragma unroll
            for (int q = 0; q < 8; q += 2)
              *reinterpret_cast<double2*>(nb + 64 + i0 + q) = make_double2(x[q][1], x[q + 1][1]);
          } else {
#pragma unroll
            for (int q = 0; q < 8; q += 2)
              *reinterpret_cast<double2*>(nb + 64 + i0 + q) = make_double2(x[q][0], x[q + 1][0]);
          }
        }
      }
    }
    __syncthreads();
  }
  if (ph && threadIdx.x == 0) ph[1] = globaltimer();
  // multipliers below the diagonal (and l_cc on it for Cholesky), then store
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int i = i0 + q;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = lane + 32 * h;
      double v = x[q][h];
      if (c < i) v *= rk[c];
      if (CHOL && c == i) v = rk[64 + c];
      if (i < T && c < T && (!CHOL || c <= i)) dk[static_cast<long long>(i) * ld + c] = v;
    }
  }
  // per-column reciprocals of the diagonal (1/u_cc, Cholesky 1/l_cc) for the
  // TRSM tasks' 8x8 block inverses
  if (threadIdx.x < 64) solve[threadIdx.x] = rk[threadIdx.x];
}


template <bool CHOL>
__device__ __forceinline__ void tf_no_fixup(double* __restrict__ dk, long long ld, int T, int gcol,
                                            int* info, double* pbuf, double* rk,
                                            unsigned long long* ph, double* solve) {
  // pbuf parity block: [0,64) pivot row (LU), [64,128) column k, [128] 1/pivot, [129] l_kk
  // rk[c]: 1/pivot of column c (LU) or 1/l_cc (Cholesky); rk[64 + c]: l_cc
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int i0 = 8 * w;
  const bool wide = T > 32;
  double x[8][2];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int i = i0 + q;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = lane + 32 * h;
      x[q][h] = (i < T && c < T && (!CHOL || c <= i))
                    ? __ldcg(dk + static_cast<long long>(i) * ld + c) : 0.0;
    }
  }
  // publish step 0: column 0 (+ row 0 for LU) and the pivot's reciprocal
  if (lane == 0) {
#pragma unroll
    for (int q = 0; q < 8; ++q) pbuf[64 + i0 + q] = x[q][0];
  }
  if (w == 0) {
    if (!CHOL) {
      pbuf[lane] = x[0][0];
      pbuf[lane + 32] = x[0][1];
    }
    if (lane == 0) {
      const double d = x[0][0];
      if (!CHOL) {
        if (fabs(d) < 1e-300) atomicMin(info, gcol);  // kernels.cpp:187-190
        rk[0] = pbuf[128] = rcp_nr(d);
      } else {
        if (d <= 0.0) atomicMin(info, gcol);  // kernels.cpp:297-302 (NaN passes)
        const double l0 = sqrt(d);
        rk[64] = l0;
        rk[0] = pbuf[128] = rcp_nr(l0);
      }
    }
  }
  __syncthreads();
  if (ph && threadIdx.x == 0) ph[0] = globaltimer();
  for (int k = 0; k < T; ++k) {
    const double* cb = pbuf + (k & 1) * kPB;
    double* nb = pbuf + ((k + 1) & 1) * kPB;
    const int k1 = k + 1;
    if (i0 + 7 > k && i0 < T) {  // warp-uniform: this warp still has live rows > k
      // x_ij -= a_ik * (u_kj / pivot): the reciprocal is folded into the
      // operand row (Cholesky: u_kj = a_jk, scaled by 1/l_kk^2), so a step
      // is one DFMA per element; the multipliers are formed at the end.
      const double r = cb[128];
      const double rs = CHOL ? r * r : r;
      double a[8];
#pragma unroll
      for (int q = 0; q < 8; q += 2) {
        const double2 v = *reinterpret_cast<const double2*>(cb + 64 + i0 + q);
        a[q] = v.x;
        a[q + 1] = v.y;
      }
      if (i0 <= k) {  // the warp holding row k: rows <= k are final
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (i0 + q <= k) a[q] = 0.0;
      }
      const double* src = CHOL ? cb + 64 : cb;
      const double u0 = lane > k ? src[lane] * rs : 0.0;
      if (wide) {
        const double u1 = lane + 32 > k ? src[lane + 32] * rs : 0.0;
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          x[q][0] = fma(-a[q], u0, x[q][0]);
          x[q][1] = fma(-a[q], u1, x[q][1]);
        }
      } else {
#pragma unroll
        for (int q = 0; q < 8; ++q) x[q][0] = fma(-a[q], u0, x[q][0]);
      }
      if (k1 < T) {
        // next pivot row k+1 (LU) and its reciprocal: the owner warp (a
        // uniform jump on q1 = (k+1) % 8 instead of a select chain)
        if ((k1 >> 3) == w) {
          double v0, v1;
          switch (k1 & 7) {
#define TT_ROW(Q)     \
  case Q:             \
    v0 = x[Q][0];     \
    v1 = x[Q][1];     \
    break;
            TT_ROW(0) TT_ROW(1) TT_ROW(2) TT_ROW(3) TT_ROW(4) TT_ROW(5) TT_ROW(6) default: TT_ROW(7)
#undef TT_ROW
          }
          if (lane == (k1 & 31)) {
            const double d = k1 >= 32 ? v1 : v0;
            if (!CHOL) {
              rk[k1] = nb[128] = rcp_nr(d);
              if (fabs(d) < 1e-300) atomicMin(info, gcol + k1);  // kernels.cpp:187-190
            } else {
              const double l1 = sqrt(d);
              rk[64 + k1] = l1;
              rk[k1] = nb[128] = rcp_nr(l1);
              if (d <= 0.0) atomicMin(info, gcol + k1);  // kernels.cpp:297-302
            }
          }
          if (!CHOL) {
            nb[lane] = v0;
            nb[lane + 32] = v1;
          }
        }
        // column k+1 of my rows (the lane holding it)
        if (lane == (k1 & 31)) {
          if (k1 >= 32) {
#pragma unroll
            for (int q = 0; q < 8; q += 2)
              *reinterpret_cast<double2*>(nb + 64 + i0 + q) = make_double2(x[q][1], x[q + 1][1]);
          } else {
#pragma unroll
            for (int q = 0; q < 8; q += 2)
              *reinterpret_cast<double2*>(nb + 64 + i0 + q) = make_double2(x[q][0], x[q + 1][0]);
          }
        }
      }
    }
    __syncthreads();
  }
  if (ph && threadIdx.x == 0) ph[1] = globaltimer();
  // multipliers below the diagonal (and l_cc on it for Cholesky), then store
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int i = i0 + q;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int c = lane + 32 * h;
      double v = x[q][h];
      
      if (CHOL && c == i) v = rk[64 + c];
      if (i < T && c < T && (!CHOL || c <= i)) dk[static_cast<long long>(i) * ld + c] = v;
    }
  }
  // per-column reciprocals of the diagonal (1/u_cc, Cholesky 1/l_cc) for the
  // TRSM tasks' 8x8 block inverses
  if (threadIdx.x < 64) solve[threadIdx.x] = rk[threadIdx.x];
}


} } }
__global__ void __launch_bounds__(256, 1) k_full(double* a, long long ld, int T, int* info, long long* cyc) {
  __shared__ __align__(16) double pbuf[2 * 132]; __shared__ double rk[128]; __shared__ double slv[64];
  __syncthreads(); long long t0 = clock64();
  tt::dag::tf_full<false>(a, ld, T, 0, info, pbuf, rk, nullptr, slv);
  __syncthreads(); long long t1 = clock64(); if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void __launch_bounds__(256, 1) k_no_zeroing(double* a, long long ld, int T, int* info, long long* cyc) {
  __shared__ __align__(16) double pbuf[2 * 132]; __shared__ double rk[128]; __shared__ double slv[64];
  __syncthreads(); long long t0 = clock64();
  tt::dag::tf_no_zeroing<false>(a, ld, T, 0, info, pbuf, rk, nullptr, slv);
  __syncthreads(); long long t1 = clock64(); if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void __launch_bounds__(256, 1) k_no_atomic(double* a, long long ld, int T, int* info, long long* cyc) {
  __shared__ __align__(16) double pbuf[2 * 132]; __shared__ double rk[128]; __shared__ double slv[64];
  __syncthreads(); long long t0 = clock64();
  tt::dag::tf_no_atomic<false>(a, ld, T, 0, info, pbuf, rk, nullptr, slv);
  __syncthreads(); long long t1 = clock64(); if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void __launch_bounds__(256, 1) k_no_wide(double* a, long long ld, int T, int* info, long long* cyc) {
  __shared__ __align__(16) double pbuf[2 * 132]; __shared__ double rk[128]; __shared__ double slv[64];
  __syncthreads(); long long t0 = clock64();
  tt::dag::tf_no_wide<false>(a, ld, T, 0, info, pbuf, rk, nullptr, slv);
  __syncthreads(); long long t1 = clock64(); if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
__global__ void __launch_bounds__(256, 1) k_no_fixup(double* a, long long ld, int T, int* info, long long* cyc) {
  __shared__ __align__(16) double pbuf[2 * 132]; __shared__ double rk[128]; __shared__ double slv[64];
  __syncthreads(); long long t0 = clock64();
  tt::dag::tf_no_fixup<false>(a, ld, T, 0, info, pbuf, rk, nullptr, slv);
  __syncthreads(); long long t1 = clock64(); if (threadIdx.x == 0) cyc[0] = t1 - t0;
}
int main() {
  const int n = 64; std::vector<double> h(n * n);
  for (int i = 0; i < n; ++i) for (int j = 0; j < n; ++j) h[i * n + j] = (i == j ? 100.0 : 0.0) + 1.0 / (1 + i + j);
  double* d; int* info; long long* cyc; cudaMalloc(&d, n * n * 8); cudaMalloc(&info, 4); cudaMallocManaged(&cyc, 8);
  for (int T : {16, 50}) {
    for (int r = 0; r < 2; ++r) { cudaMemcpy(d, h.data(), n*n*8, cudaMemcpyHostToDevice); cudaMemset(info, 0x7f, 4); k_full<<<1,256>>>(d, n, T, info, cyc); cudaDeviceSynchronize(); }
    printf("T=%d %-12s %.1f cycles/pivot\n", T, "full", (double)cyc[0] / T);
    for (int r = 0; r < 2; ++r) { cudaMemcpy(d, h.data(), n*n*8, cudaMemcpyHostToDevice); cudaMemset(info, 0x7f, 4); k_no_zeroing<<<1,256>>>(d, n, T, info, cyc); cudaDeviceSynchronize(); }
    printf("T=%d %-12s %.1f cycles/pivot\n", T, "no_zeroing", (double)cyc[0] / T);
    for (int r = 0; r < 2; ++r) { cudaMemcpy(d, h.data(), n*n*8, cudaMemcpyHostToDevice); cudaMemset(info, 0x7f, 4); k_no_atomic<<<1,256>>>(d, n, T, info, cyc); cudaDeviceSynchronize(); }
    printf("T=%d %-12s %.1f cycles/pivot\n", T, "no_atomic", (double)cyc[0] / T);
    for (int r = 0; r < 2; ++r) { cudaMemcpy(d, h.data(), n*n*8, cudaMemcpyHostToDevice); cudaMemset(info, 0x7f, 4); k_no_wide<<<1,256>>>(d, n, T, info, cyc); cudaDeviceSynchronize(); }
    printf("T=%d %-12s %.1f cycles/pivot\n", T, "no_wide", (double)cyc[0] / T);
    for (int r = 0; r < 2; ++r) { cudaMemcpy(d, h.data(), n*n*8, cudaMemcpyHostToDevice); cudaMemset(info, 0x7f, 4); k_no_fixup<<<1,256>>>(d, n, T, info, cyc); cudaDeviceSynchronize(); }
    printf("T=%d %-12s %.1f cycles/pivot\n", T, "no_fixup", (double)cyc[0] / T);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
