// potrf_variants.cuh -- POTRF variants for tools/micro/potrf_lab.cu
#pragma once
template <int V> constexpr int variant_n() { return 16; }
template <int V> constexpr int variant_ld() { return LD; }

// V2: three-row uniform lookahead.  Every lane carries, identically, the pivot and the entries
// of rows c+1..c+3 that the next three columns need; the rank-1 update reaches entries c+1..c+3
// through registers (uniform multipliers l1..l3), entries c+4.. through the column in shared
// memory, APPLIED ONE ITERATION LATER; the row entering the window is shuffled from its lane one
// iteration before its first use.  So the chain per column is rsqrt + mul + fma, and every
// shared-memory / shuffle latency has a whole column of slack.
__device__ __forceinline__ void potrf_v2(const double* A, double* D, double* lbuf, double eps, double& carry) {
  constexpr int NB = 16;
  const int r = threadIdx.x & 31;
  const bool inv = r >= NB;
  double row[NB];
  double dg = 1.0;
#pragma unroll
  for (int c = 0; c < NB; ++c) {
    const double v = A[c * LD + ((c <= r && !inv) ? r : 0)] + eps * carry;
    row[c] = inv ? (c == r - NB ? 1.0 : 0.0) : v;
    if (c == r) dg = v;
  }
  double p = __shfl_sync(kFull, row[0], 0);
  double a1 = __shfl_sync(kFull, row[0], 1), b11 = __shfl_sync(kFull, row[1], 1);
  double a2 = __shfl_sync(kFull, row[0], 2), b21 = __shfl_sync(kFull, row[1], 2), b22 = __shfl_sync(kFull, row[2], 2);
  double a3 = __shfl_sync(kFull, row[0], 3), b31 = __shfl_sync(kFull, row[1], 3), b32 = __shfl_sync(kFull, row[2], 3),
         b33 = __shfl_sync(kFull, row[3], 3);
  double rs = rsqrt_nr(p);
  double2 pend[NB / 2];
  double lrc_prev = 0.0;
#pragma unroll
  for (int h = 0; h < NB / 2; ++h) pend[h] = make_double2(0.0, 0.0);
#pragma unroll
  for (int c = 0; c < NB; ++c) {
    const double l1 = a1 * rs, l2 = a2 * rs, l3 = a3 * rs;
    const double pn = fma(-l1, l1, b11);
    const double rsn = rsqrt_nr(pn);
    const double lrc = row[c] * rs;
    // column c-1 through shared memory (loaded an iteration ago): entries c+3..
    if (c >= 1) {
#pragma unroll
      for (int h = 0; h < NB / 2; ++h) {
        if (2 * h >= c + 3) row[2 * h] = fma(-lrc_prev, pend[h].x, row[2 * h]);
        if (2 * h + 1 >= c + 3) row[2 * h + 1] = fma(-lrc_prev, pend[h].y, row[2 * h + 1]);
      }
    }
    // column c through registers: entries c+1..c+3, and the lane's own diagonal entry
    if (c + 1 < NB) row[c + 1 < NB ? c + 1 : 0] = fma(-lrc, l1, row[c + 1 < NB ? c + 1 : 0]);
    if (c + 2 < NB) row[c + 2 < NB ? c + 2 : 0] = fma(-lrc, l2, row[c + 2 < NB ? c + 2 : 0]);
    if (c + 3 < NB) row[c + 3 < NB ? c + 3 : 0] = fma(-lrc, l3, row[c + 3 < NB ? c + 3 : 0]);
    dg = fma(-lrc, lrc, dg);
    // row c+4 enters the window
    double e0 = 0.0, e1 = 0.0, e2 = 0.0, e3 = 0.0;
    if (c + 4 < NB) {
      e0 = shfl_early(row[c + 1 < NB ? c + 1 : 0], c + 4);
      e1 = shfl_early(row[c + 2 < NB ? c + 2 : 0], c + 4);
      e2 = shfl_early(row[c + 3 < NB ? c + 3 : 0], c + 4);
      e3 = shfl_early(dg, c + 4);
    }
    row[c] = lrc;
    double* dc = D + c * LD;
    *(inv ? lbuf + (r - NB) : dc + r) = lrc;
    __syncwarp();
#pragma unroll
    for (int h = 0; h < NB / 2; ++h)
      if (2 * h + 1 >= c + 4) pend[h] = reinterpret_cast<const double2*>(dc)[h];
    lrc_prev = lrc;
    // the window moves one row
    a1 = fma(-l2, l1, b21);
    b11 = fma(-l2, l2, b22);
    a2 = fma(-l3, l1, b31);
    b21 = fma(-l3, l2, b32);
    b22 = fma(-l3, l3, b33);
    a3 = e0; b31 = e1; b32 = e2; b33 = e3;
    p = pn;
    rs = rsn;
  }
  carry = row[15];
}

template <int V>
__device__ __forceinline__ void run_variant(const double* A, double* D, double* lbuf, double eps, double& carry) {
  if (V == 0) potrf_v0(A, D, lbuf, eps, carry);
  else potrf_v2(A, D, lbuf, eps, carry);
}
