// band_cta.cuh -- one thread block factors one band matrix.
//
// Right-looking blocked band Cholesky (the reference's sliding window of
// blocked.py:1-7, :297-315, re-derived for one CTA).  Step k owns columns
// [j0, j0+nb), j0 = k*NB:
//   1. POTRF of the nb x nb diagonal block        (blocked.py:259-269 factor_diag)
//   2. TRSM of the m x nb panel below it, m = min(kd, n-j0-nb); the out-of-band
//      triangle (blocked.py:136-167 WorkArray) is exact zeros in registers
//                                                  (blocked.py:271-276 solve_panel)
//   3. SYRK/GEMM of the m x m trailing triangle    (blocked.py:278-284 update_*)
//
// B200 mapping:
//   * The active window (kd+NB columns x (kd+1) entries) lives in shared memory as
//     a ring of column slots; every column is loaded from HBM once (cp.async, a
//     step ahead of first use) and written back once, right after its panel step.
//   * POTRF runs in warp 0 with the pivot chain computed REDUNDANTLY in every
//     lane (p_{c+1} = A'(c+1,c+1) - (A'(c+1,c) rsqrt(p_c))^2 from two values
//     broadcast one step ahead), so one column costs rsqrt + mul + fma on the
//     critical path instead of rsqrt + shuffle + mul + fma.
//   * Lookahead: the update of step k is split; the part that touches the next
//     panel's columns runs first, then warp 0 factors the next diagonal block
//     while warps 1-7 finish the rest of step k's update.
//   * The trailing update runs on the FP64 tensor path (mma.sync m8n8k4 f64 ->
//     DMMA), 16x16 warp tiles, operands from a dense panel copy P whose leading
//     dimension is 4 (mod 16) doubles (conflict-free fragment loads).
#pragma once
#include <type_traits>
#include <cstdint>
#include <cuda_runtime.h>

namespace bcg {

constexpr int kCtaThreads = 256;
static_assert(kCtaThreads - 64 == 192, "cta_panel_doubles sizes the far partials for 192 threads");
constexpr int kCtaWarps = kCtaThreads / 32;
constexpr unsigned kFull = 0xffffffffu;
// the thread that issues and waits on the window's bulk copies: lane 0 of the last warp,
// so the POTRF warp (warp 0) never blocks on copy-engine bookkeeping
constexpr int kCopyThread = kCtaThreads - 32;

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem) : "memory");
}
// 8-byte cp.async; ok = false writes zeros (src-size 0, src not read)
__device__ __forceinline__ void cp_async8_zfill(double* smem, const double* gmem, bool ok) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(ok ? 8 : 0) : "memory");
}
// arrive on an mbarrier once every prior cp.async of this thread has landed (counted
// against the barrier's expected arrivals)
__device__ __forceinline__ void cp_async_mbar_arrive(unsigned long long* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"((unsigned)__cvta_generic_to_shared(bar))
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait_group() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

// ---- bulk async copies (TMA bulk path, SASS UBLKCP) + mbarriers -------------------
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned phase) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}
// global -> shared, completion counted on `bar` (bytes % 16 == 0, both addresses 16-aligned)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
// plain (count) arrival, release semantics at CTA scope
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// named barrier over `count` threads (warps of the pipelined factorization)
__device__ __forceinline__ void named_bar(int id, int count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}
// shared -> global (bulk group)
__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, unsigned bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
// make this thread's generic-proxy shared-memory writes visible to the async proxy
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void fence_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

// ---- optional trace (bcg_set_trace): phase stamps, %globaltimer ns -------------
// [0] = steps recorded, then kTracePhases stamps per step (block 0 / matrix 0 only
// for this kernel; the pivot CTA for the multi-CTA kernel).
constexpr int kTracePhases = 8;
__device__ unsigned long long* g_trace = nullptr;
__device__ unsigned long long g_trace_cap = 0;

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%clock64;" : "=l"(t));  // SM cycles: phases of one CTA
  return t;
}
__device__ __forceinline__ void trace_stamp_to(unsigned long long* tr, int j, int phase) {
  if (tr) {
    const unsigned long long idx = 1 + (unsigned long long)j * kTracePhases + phase;
    if (idx < g_trace_cap) tr[idx] = gtime();
    if (phase == 0) tr[0] = j + 1;  // (steps are stamped in increasing order: no read-back)
  }
}

// Re-broadcast a value the compiler cannot prove warp-uniform (read from shared memory)
// from lane 0: branches on the result are then known not to split the warp, which keeps
// ptxas from wrapping every later shuffle / __syncwarp in collective divergence handling.
__device__ __forceinline__ int warp_uniform(int v) { return __shfl_sync(0xffffffffu, v, 0); }

// 64-bit broadcast from `src` issued where written: volatile asm keeps the compiler from
// sinking the shuffle down to its first use, so its latency overlaps the rest of a
// POTRF column instead of sitting on the pivot chain.
__device__ __forceinline__ double shfl_early(double v, int src) {
  unsigned lo, hi;
  asm volatile("mov.b64 {%0, %1}, %2;" : "=r"(lo), "=r"(hi) : "d"(v));
  asm volatile("shfl.sync.idx.b32 %0, %0, %1, 0x1f, 0xffffffff;" : "+r"(lo) : "r"(src));
  asm volatile("shfl.sync.idx.b32 %0, %0, %1, 0x1f, 0xffffffff;" : "+r"(hi) : "r"(src));
  double r;
  asm volatile("mov.b64 %0, {%1, %2};" : "=d"(r) : "r"(lo), "r"(hi));
  return r;
}

// Column permutation of the tile GEMM's B operand / C fragment: lane (gr, gc) loads B column
// kPerm(gr) and owns C columns kPerm(2gc), kPerm(2gc+1).  With column strides = 4 (mod 16)
// doubles (window lds - 1 = 100 for kd = 100, P's pld, D's kLDD) every fragment access of a
// half-warp -- B loads and the C loads/stores in the band window or P -- hits 16 distinct
// bank pairs (the identity order makes the C accesses 2-way conflicted).
__device__ __forceinline__ int kperm(int x) { return (0x57463120u >> (4 * x)) & 7; }  // 0,2,1,3,6,4,7,5

// d -= a b (negated A operand; not volatile, so the scheduler may interleave chains)
__device__ __forceinline__ void dmma884n(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(-a), "d"(b));
}
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// Branch-free full-precision 1/sqrt(p) for finite p > 0: MUFU.RSQ64H seed + two
// Newton steps (relative error ~2^-44 after the first, rounding-limited after the
// second).  No special-case branch, so the compiler can interleave it with the
// surrounding work; non-positive / NaN pivots are caught by the caller's check.
__device__ __forceinline__ double rsqrt_nr(double p) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(p));
  double h = p * y;
  double e = fma(-h, y, 1.0);
  y = fma(y * 0.5, e, y);
  h = p * y;
  e = fma(-h, y, 1.0);
  y = fma(y * 0.5, e, y);
  return y;
}

// Branch-free 1/d for finite d > 0: MUFU.RCP64H seed + two Newton steps.
__device__ __forceinline__ double rcp_nr(double d) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(d));
  double e = fma(-d, y, 1.0);
  y = fma(y, e, y);
  e = fma(-d, y, 1.0);
  return fma(y, e, y);
}

struct CtaGeom {
  int n, kd, ldab;  // matrix geometry
  int lds, nslot;   // shared window: nslot column slots of lds doubles
  int pld;          // leading dimension of the dense panel P (>= kd rounded up to 16, = 4 mod 16)
};

// The dense panel buffer P (nb_block x pld).
__host__ __device__ inline size_t cta_panel_doubles(int nb_block, const CtaGeom& g) {
  return (size_t)nb_block * g.pld;
}

// Forward-sweep scratch of the fused factor + forward solve (dpbsv): the accumulator ring
// (rows j0 .. j0 + kd + 15, a multiple of 16) + two 16-vectors (v = b + acc, y).
__host__ __device__ inline int cta_fwd_ring(int kd) { return (kd + 16 + 15) / 16 * 16; }
__host__ __device__ inline size_t cta_fwd_doubles(int kd) { return (size_t)cta_fwd_ring(kd) + 32; }

// Shared-memory footprint (bytes) of one CTA for block size NB.
__host__ __device__ inline size_t cta_smem_bytes(int nb_block, const CtaGeom& g) {
  // D: two L11 / L11^-1 buffers (the pipelined factorization alternates them by step)
  size_t d = (size_t)g.nslot * g.lds + cta_panel_doubles(nb_block, g) + 2 * (size_t)nb_block * (nb_block + 4) +
             nb_block + cta_fwd_doubles(g.kd);
  return d * sizeof(double) + 64;
}

// Compile-time geometry for one band width (the bench configuration): kd, ldab = lds =
// kd + 1, the ring and panel strides exactly as make_geom() (bandchol_b200.cu) picks them,
// so index arithmetic folds to constants and frees registers in the hot loops; n stays
// runtime.  KD = 0 selects the runtime CtaGeom.
template <int KD>
struct GeomFixed {
  int n;
  static constexpr int kd = KD, ldab = KD + 1, lds = KD + 1;
  static constexpr int ns0 = KD + 16;
  static constexpr int nslot = (ns0 & 1) ? ns0 + 1 : ns0;
  static constexpr int pld = KD + ((4 - KD % 16) + 16) % 16;
  __host__ __device__ GeomFixed(const CtaGeom& x) : n(x.n) {}
  // true when the runtime geometry the host chose is exactly this one
  __host__ __device__ static bool matches(const CtaGeom& x) {
    return x.kd == kd && x.ldab == ldab && x.lds == lds && x.nslot == nslot && x.pld == pld;
  }
};
template <int KD>
struct GeomOf { using type = GeomFixed<KD>; };
template <>
struct GeomOf<0> { using type = CtaGeom; };

template <int NB, int KD = 0>
struct CtaBand {
  static_assert(NB == 16, "block size: lanes 16-31 of the POTRF warp invert L11");
  const typename GeomOf<KD>::type g;
  double* __restrict__ ab;   // this matrix in global memory
  double* win;               // shared ring of column slots
  double* P;                 // NB x pld dense panel, P[c*pld + r] = L(j0+nb+r, j0+c)
  static constexpr int kLDD = NB + 4;  // D stride (= 4 mod 16: conflict-free DMMA fragments)
  double* D;                 // L11, D[c*kLDD + r] = L(r, c); then L11^-1, D[i*kLDD + j] = Linv(i, j)
  double* lbuf;              // NB doubles: sink for the inverse lanes' column stores
  unsigned long long* bars;  // mbarrier [0]: window loads
  unsigned long long* sig;   // pipelined factorization: [0] panel ready, [1] column 0 updated, [2 + (k&1)] update done, [4] y_k ready
  unsigned phase = 0;        // parity of the next wait on bars[0] (uniform register)
  bool pending = false;      // a load_cols is in flight
  bool fast = false;         // every column chunk meets the bulk-copy alignment rules
  // Warp roles by SM sub-partition (set_roles): the POTRF warp pw and a light warp share
  // SMSP 0 with the other CTA's pivot; the six warps on SMSPs 1-3 run every DMMA.
  int pw = 0;                // the POTRF warp
  int wk = -1;               // this warp's worker index 0..5 (-1: pivot or light warp)
  unsigned long long* tr = nullptr;  // trace buffer (block 0 only), see bcg_set_trace
  // fused forward sweep (dpbsv, pipelined factorization only): the light warp solves
  // L y = b block by block right behind the panel, from the panel still in shared memory
  const double* fb = nullptr;  // this matrix's right-hand side (nullptr: factorization only)
  double* fy = nullptr;        // y out (n doubles)
  double* fws = nullptr;       // shared scratch: accumulator ring, then v[16], y[16]

  // Roles from the hardware warp slot (%warpid & 3 = SMSP): the second CTA on an SM is
  // rotated by one sub-partition (tools/micro/warpid.cu), so warp index alone cannot tell.
  // s_sp: kCtaWarps ints of shared scratch.  Call by all threads, before any role is used.
  __device__ void set_roles(int* s_sp) {
    const int warp = threadIdx.x >> 5;
    unsigned hw;
    asm volatile("mov.u32 %0, %%warpid;" : "=r"(hw));
    if ((threadIdx.x & 31) == 0) s_sp[warp] = (int)(hw & 3);
    __syncthreads();
    int n0 = 0, first0 = -1;
    for (int w = 0; w < kCtaWarps; ++w)
      if (s_sp[w] == 0) { ++n0; if (first0 < 0) first0 = w; }
    const bool hwmap = n0 == 2;  // else: fall back to warp index mod 4
    pw = hwmap ? first0 : 0;
    int idx = 0, mine = -1;
    for (int w = 0; w < kCtaWarps; ++w) {
      if ((hwmap ? s_sp[w] : (w & 3)) == 0) continue;
      if (w == warp) mine = idx;
      ++idx;
    }
    wk = warp_uniform(mine);
    __syncthreads();
  }

  __device__ __forceinline__ void trace_stamp(int j, int ph) const {
#ifdef BCG_TRACE
    if (tr && (threadIdx.x & 31) == 0) trace_stamp_to(tr, j, ph);
#else
    (void)j;
    (void)ph;
#endif
  }

  // ---- ring addressing: slot(j) = j mod nslot without a division on hot paths ----
  __device__ __forceinline__ int slot_from(int s0, int j0, int j) const {
    int s = s0 + (j - j0);
    return s >= g.nslot ? s - g.nslot : s;  // valid for j0 <= j < j0 + nslot
  }
  __device__ __forceinline__ int col_len(int j) const { return min(g.kd, g.n - 1 - j) + 1; }

  // ---- column streaming between HBM and the ring -----------------------------------
  // Whole columns (ldab doubles, padding included, so the write-back restores the
  // padding bytes unchanged) move as bulk async copies in contiguous chunks; a column
  // whose chunk would break the 16-byte rules of cp.async.bulk goes element-wise.
  // Plan for columns [jlo, jhi) placed at ring slot (jlo % nslot) onward: up to two
  // contiguous pieces (ring wrap), each trimmed to an aligned bulk range.
  struct Piece { int j, cnt, slot; };
  __device__ __forceinline__ int pieces(int jlo, int jhi, Piece* pc) const {
    const int s0 = jlo % g.nslot;
    const int c1 = min(jhi - jlo, g.nslot - s0);
    pc[0] = {jlo, c1, s0};
    if (c1 < jhi - jlo) { pc[1] = {jlo + c1, jhi - jlo - c1, 0}; return 2; }
    return 1;
  }
  // bulk sub-range [b0, b0+bc) of a piece; columns outside it go element-wise
  __device__ __forceinline__ void bulk_range(const Piece& p, const double* gbase, int& b0, int& bc) const {
    auto aligned = [&](int c) {
      return !(((uintptr_t)(gbase + (int64_t)(p.j + c) * g.ldab)) & 15) &&
             !(((uintptr_t)(win + (size_t)(p.slot + c) * g.lds)) & 15);
    };
    b0 = aligned(0) ? 0 : 1;  // odd start with odd ldab: the next column is aligned on both sides
    if (b0 >= p.cnt || !aligned(b0)) {
      b0 = 0;
      bc = 0;
      return;
    }
    bc = p.cnt - b0;
    if (((size_t)bc * g.ldab * sizeof(double)) % 16) bc -= 1;
  }
  __device__ void elem_copy_col(int j, int slot, bool to_smem) {
    double* sp = win + (size_t)slot * g.lds;
    double* gp = ab + (int64_t)j * g.ldab;
    for (int o = threadIdx.x; o < g.ldab; o += kCtaThreads) {
      if (to_smem) cp_async8(sp + o, gp + o);
      else gp[o] = sp[o];
    }
  }

  // The fast path holds when the matrix base is 16-byte aligned and every chunk the
  // kernel moves starts on an even column with an even count or ldab is even
  // (decided once per matrix by the host-chosen geometry, see init_fast()).
  __device__ void init_fast() {
    fast = !(((uintptr_t)ab) & 15) && !(((uintptr_t)win) & 15) && ((g.ldab % 2 == 0) || (g.nslot % 2 == 0 && g.kd % 2 == 0));
    // with odd ldab the chunks start at j0 + NB + kd (even) and the tail count n - jlo must be even
    if (fast && g.ldab % 2 == 1) fast = ((g.n - min(g.n, g.kd + NB)) % 2 == 0) && (min(g.n, g.kd + NB) % 2 == 0);
  }

  // async load of columns [jlo, jhi); complete with wait_cols()
  // sj: ring slot of column jlo when the caller knows it (saves a division), else -1
  __device__ void load_cols(int jlo, int jhi, int sj = -1) {
    if (sj < 0) sj = jlo % g.nslot;
    if (fast) {
      if (threadIdx.x == kCopyThread) {
        bulk_wait_read0();  // the write-back that read these slots is done reading
        const unsigned col = (unsigned)g.ldab * sizeof(double);
        mbar_expect_tx(bars, (unsigned)(jhi - jlo) * col);
        const int s0 = sj;
        const int c1 = min(jhi - jlo, g.nslot - s0);
        bulk_g2s(win + (size_t)s0 * g.lds, ab + (int64_t)jlo * g.ldab, c1 * col, bars);
        if (c1 < jhi - jlo) bulk_g2s(win, ab + (int64_t)(jlo + c1) * g.ldab, (jhi - jlo - c1) * col, bars);
      }
      pending = true;
      return;
    }
    if (threadIdx.x == kCopyThread) bulk_wait_read0();  // the write-back that read these slots is done reading
    __syncthreads();
    Piece pc[2];
    const int np = pieces(jlo, jhi, pc);
    unsigned bytes = 0;
    for (int q = 0; q < np; ++q) {
      int b0, bc;
      bulk_range(pc[q], ab, b0, bc);
      bytes += (unsigned)bc * g.ldab * sizeof(double);
      for (int c = 0; c < pc[q].cnt; ++c)
        if (c < b0 || c >= b0 + bc) elem_copy_col(pc[q].j + c, pc[q].slot + c, true);
    }
    if (threadIdx.x == kCopyThread) {
      mbar_expect_tx(bars, bytes);
      for (int q = 0; q < np; ++q) {
        int b0, bc;
        bulk_range(pc[q], ab, b0, bc);
        if (bc > 0)
          bulk_g2s(win + (size_t)(pc[q].slot + b0) * g.lds, ab + (int64_t)(pc[q].j + b0) * g.ldab,
                   (unsigned)bc * g.ldab * sizeof(double), bars);
      }
    }
    cp_async_commit();
    pending = true;
  }
  // all threads: the last load_cols has landed and is visible
  __device__ __forceinline__ void wait_cols() {
    if (!fast) cp_async_wait_all();
    mbar_wait(bars, phase);
    phase ^= 1u;
    pending = false;
    __syncthreads();
  }

  // Panel columns [j0, j0+nb) back to HBM (final L).  Call after a barrier that
  // follows fence_async_smem() by every writer; the bulk part is issued by thread 0.
  __device__ void store_cols(int j0, int nb, int sj = -1) {  // sj: ring slot of column j0
    if (fast) {
      if (threadIdx.x == kCopyThread) {
        const unsigned col = (unsigned)g.ldab * sizeof(double);
        const int s0 = sj >= 0 ? sj : j0 % g.nslot;
        const int c1 = min(nb, g.nslot - s0);
        bulk_s2g(ab + (int64_t)j0 * g.ldab, win + (size_t)s0 * g.lds, c1 * col);
        if (c1 < nb) bulk_s2g(ab + (int64_t)(j0 + c1) * g.ldab, win, (nb - c1) * col);
        bulk_commit();
      }
      return;
    }
    Piece pc[2];
    const int np = pieces(j0, j0 + nb, pc);
    for (int q = 0; q < np; ++q) {
      int b0, bc;
      bulk_range(pc[q], ab, b0, bc);
      for (int c = 0; c < pc[q].cnt; ++c)
        if (c < b0 || c >= b0 + bc) elem_copy_col(pc[q].j + c, pc[q].slot + c, false);
      if (threadIdx.x == kCopyThread && bc > 0)
        bulk_s2g(ab + (int64_t)(pc[q].j + b0) * g.ldab, win + (size_t)(pc[q].slot + b0) * g.lds,
                 (unsigned)bc * g.ldab * sizeof(double));
    }
    if (threadIdx.x == kCopyThread) bulk_commit();
  }

  // Warp pw: Cholesky of the nb x nb diagonal block at column j0.
  // Lane r holds row r.  Returns the local failing column or -1 (uniform).
  //
  // Straight-line for every block: a short last block (nb < NB) is padded with identity
  // rows, so the column loop has no per-column masks.  Column c of D doubles as the
  // broadcast buffer of the rank-1 update (distinct per column, so one __syncwarp per
  // column suffices), lanes NB..31 build L11^-1 along the way, and failure is found
  // once at the end: after a non-positive / NaN pivot every later pivot of the block is
  // NaN, so the first failing column is the first lane whose L(r, r) is not > 0.
  __device__ int potrf_diag(int s0, int j0, int nb) {
    const int r = threadIdx.x & 31;
    double row[NB];
    const int sw = g.nslot - s0;  // columns before the ring wraps
    // lanes NB..2NB-1 start from e_(r-NB): the column step below is then, for them,
    // forward substitution L11 x = e_(r-NB), so they finish holding column r-NB of L11^-1
    // (the panel TRSM is a product with it) at no extra instruction cost
    const bool inv = r >= NB;
    const double e = 1.0;
    if (nb == NB && g.kd >= NB - 1) {
      // whole block inside the band: entries above the diagonal are don't-care, so the
      // loads only need an in-bounds offset
#pragma unroll
      for (int c = 0; c < NB; ++c) {
        const int sl = c < sw ? s0 + c : s0 + c - g.nslot;
        const double v = win[sl * g.lds + ((c <= r && !inv) ? r - c : 0)];
        row[c] = inv ? (c == r - NB ? e : 0.0) : v;
      }
    } else {
#pragma unroll
      for (int c = 0; c < NB; ++c) {
        const int sl = c < sw ? s0 + c : s0 + c - g.nslot;
        const bool in = r < nb && c <= r && r - c <= g.kd;
        const double v = win[sl * g.lds + (in ? r - c : 0)];
        row[c] = in ? v : ((inv ? c == r - NB : (r >= nb && c == r)) ? e : 0.0);
      }
    }
    // chain state, identical in every lane: p = pivot of column c, (alpha, beta) =
    // (A'(c+1,c), A'(c+1,c+1)) through column c-1, broadcast by lane c+1 a step early.
    double p = __shfl_sync(kFull, row[0], 0);
    double alpha = __shfl_sync(kFull, row[0], 1);
    double beta = __shfl_sync(kFull, row[1], 1);
    double rs = rsqrt_nr(p);
    // Software-pipelined: the next column's 1/sqrt and chain broadcasts are issued
    // before this column's rank-1 update, so their latency hides under it.
#pragma unroll
    for (int c = 0; c < NB; ++c) {
      // L(r, c) for r >= c (for r == c this is p * rs: lane c's own entry equals p
      // bit for bit); lanes r < c compute don't-care values that are never read
      const double lrc = row[c] * rs;
      const double l1 = alpha * rs;                     // L(c+1, c)
      const double pn = fma(-l1, l1, beta);             // pivot of column c+1
      const double rsn = rsqrt_nr(pn);
      // entry (r, c+1) first, with L(c+1,c) = l1 from registers: the next column's
      // L(r, c+1) never waits on the shared-memory broadcast below
      if (c + 1 < NB) row[c + 1 < NB ? c + 1 : 0] = fma(-lrc, l1, row[c + 1 < NB ? c + 1 : 0]);
      double alpha_n = 0.0, beta_n = 0.0;
      if (c + 2 < NB) {
        // lane c+2's entries (c+2, c+1), (c+2, c+2) after this column
        const double bn = fma(-lrc, lrc, row[c + 2 < NB ? c + 2 : 0]);
        alpha_n = shfl_early(row[c + 1 < NB ? c + 1 : 0], c + 2);
        beta_n = shfl_early(bn, c + 2);
      }
      row[c] = lrc;
      double* dc = D + c * kLDD;  // column c of L11 (rows < c: don't-care)
      *(inv ? lbuf + (r - NB) : dc + r) = lrc;  // lanes >= NB: scratch, no branch
      __syncwarp();
      // rank-1 update of the rest of the row; entries right of the diagonal become
      // garbage that is never read (only c2 <= r is used or stored)
#pragma unroll
      for (int h = 0; h < NB / 2; ++h) {  // two broadcast values per 128-bit load
        if (2 * h + 1 >= c + 2) {
          const double2 l2 = reinterpret_cast<const double2*>(dc)[h];
          if (2 * h >= c + 2) row[2 * h] = fma(-lrc, l2.x, row[2 * h]);
          row[2 * h + 1] = fma(-lrc, l2.y, row[2 * h + 1]);
        }
      }
      p = pn;
      rs = rsn;
      alpha = alpha_n;
      beta = beta_n;
    }
    const double dgl = (r < nb) ? D[r * kLDD + r] : 1.0;
    const unsigned bad = __ballot_sync(kFull, !(dgl > 0.0));
    if (bad) return __ffs(bad) - 1;
    // the factored block back to its window slots (the lookahead leaves warp 0 slack)
#pragma unroll
    for (int c = 0; c < NB; ++c) {
      const int sl = c < sw ? s0 + c : s0 + c - g.nslot;
      if (c <= r && r < nb && r - c <= g.kd) win[sl * g.lds + (r - c)] = row[c];
    }
    // D <- L11^-1, row-major (D[i*kLDD + j] = Linv(i, j)), once every lane is done
    // reading L11 from it
    __syncwarp();
    if (inv) {
#pragma unroll
      for (int i = 0; i < NB; ++i) D[i * kLDD + (r - NB)] = row[i];
    }
    return -1;
  }

  // Panel TRSM as a product: X = A L11^-T for the m panel rows, 16-row tiles over the
  // warps, DMMA m8n8k4 with A from the window (entries outside the band read as 0) and
  // B(k, c) = Linv(c, k) from D.  X goes to the dense panel P and back to the window.
  // Tiles t = wid, wid + nw, ... (the calling warp is worker wid of nw).
  __device__ void trsm_panel(int s0, int j0, int nb, int m, int wid, int nw) {
    const int lane = threadIdx.x & 31;
    const int gr = lane >> 2, gc = lane & 3;
    const int sw = g.nslot - s0;
    const int T = (m + 15) >> 4;
    for (int t = wid; t < T; t += nw) {
      const bool tail = 16 * t + 8 >= m;  // rows 16t+8.. are all past m
      double acc[2][NB / 8][2];
#pragma unroll
      for (int u = 0; u < 2; ++u)
#pragma unroll
        for (int v = 0; v < NB / 8; ++v) acc[u][v][0] = acc[u][v][1] = 0.0;
#pragma unroll
      for (int kk = 0; kk < NB / 4; ++kk) {
        const int k = 4 * kk + gc;
        const int sl = k < sw ? s0 + k : s0 + k - g.nslot;
        double a[2], bf[NB / 8];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int off = nb + 16 * t + 8 * u + gr - k;
          const bool in = k < nb && off <= g.kd;
          const double v = win[sl * g.lds + (in ? off : 0)];
          a[u] = in ? v : 0.0;
        }
#pragma unroll
        for (int v = 0; v < NB / 8; ++v) bf[v] = D[(8 * v + kperm(gr)) * kLDD + k];  // (kperm: conflict-free C)
#pragma unroll
        for (int u = 0; u < 2; ++u)
#pragma unroll
          for (int v = 0; v < NB / 8; ++v)  // L11^-T is upper triangular: k > 8v+7 adds zeros
            if ((u == 0 || !tail) && kk <= 2 * v + 1) dmma884(acc[u][v][0], acc[u][v][1], a[u], bf[v]);
      }
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int r = 16 * t + 8 * u + gr;
        if (r >= m) continue;
#pragma unroll
        for (int v = 0; v < NB / 8; ++v)
#pragma unroll
          for (int e = 0; e < 2; ++e) {
            const int c = 8 * v + kperm(2 * gc + e);
            const int off = nb + r - c;
            const int sl = c < sw ? s0 + c : s0 + c - g.nslot;
            P[c * g.pld + r] = acc[u][v][e];
            if (c < nb && off <= g.kd) win[sl * g.lds + off] = acc[u][v][e];
          }
      }
    }
  }

  // Trailing update of 16x16 tiles, C(i,j) -= sum_c P(i,c) P(j,c), i,j < m, lower only.
  // Tiles are numbered column by column ((0,0), (1,0), ..., (T-1,0), (1,1), ...); the
  // calling warp (rank wid of nw workers) takes tiles first + wid, first + wid + nw, ...
  // below `last`.
  // One 16x16 tile C(i0.., q0..) -= P(i0..) P(q0..)^T.  DIAG: a diagonal tile (the 8x8
  // block above the diagonal is skipped, the two diagonal 8x8 blocks are masked to q <= i);
  // ROWS: 0 every row < m, 1 rows i0+8.. partly past m (masked), 2 rows i0+8.. all past m
  // (their two 8x8 blocks skipped).  Straight-line per kind, so every accumulator chain
  // of the tile is in flight at once.
  template <bool DIAG, int ROWS>
  __device__ __forceinline__ void tile_update(const int (&cb)[2][2], int i0, int q0, int m) {
    const int lane = threadIdx.x & 31;
    const int gr = lane >> 2, gc = lane & 3;
    constexpr bool kU1 = ROWS != 2;   // rows i0+8.. computed
    constexpr bool kV1 = !DIAG;       // block (0,1) computed
    auto ok = [&](int u, int v, int e) {
      const int i = i0 + u * 8 + gr, q = q0 + v * 8 + kperm(2 * gc + e);
      bool r = true;
      if (DIAG && u == v) r = q <= i;
      if (ROWS != 0 && (u == 1 || ROWS == 2)) r = r && i < m;
      return r;
    };
    double acc[2][2][2];
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int v = 0; v < 2; ++v)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          if ((u == 1 && !kU1) || (u == 0 && v == 1 && !kV1)) { acc[u][v][e] = 0.0; continue; }
          const int i = i0 + u * 8 + gr;
          acc[u][v][e] = ok(u, v, e) ? win[cb[v][e] + i] : 0.0;
        }
#pragma unroll
    for (int k0 = 0; k0 < NB; k0 += 4) {
      const double* pk = P + (k0 + gc) * g.pld;
      const double a0 = pk[i0 + gr], a1 = kU1 ? pk[i0 + 8 + gr] : 0.0;
      const double b0 = pk[q0 + kperm(gr)], b1 = pk[q0 + 8 + kperm(gr)];
      dmma884n(acc[0][0][0], acc[0][0][1], a0, b0);
      if (kU1) dmma884n(acc[1][0][0], acc[1][0][1], a1, b0);
      if (kV1) dmma884n(acc[0][1][0], acc[0][1][1], a0, b1);
      if (kU1) dmma884n(acc[1][1][0], acc[1][1][1], a1, b1);
    }
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int v = 0; v < 2; ++v)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          if ((u == 1 && !kU1) || (u == 0 && v == 1 && !kV1)) continue;
          const int i = i0 + u * 8 + gr;
          if (ok(u, v, e)) win[cb[v][e] + i] = acc[u][v][e];
        }
  }

  // Trailing update of 16x16 tiles, C(i,j) -= sum_c P(i,c) P(j,c), i,j < m, lower only.
  // Tiles are numbered column by column ((0,0), (1,0), ..., (T-1,0), (1,1), ...); the
  // calling warp (rank wid of nw workers) takes tiles first + wid, first + wid + nw, ...
  // below `last`.
  __device__ void update_tiles(int s0, int j0, int nb, int m, int first, int last, int wid, int nw) {
    const int lane = threadIdx.x & 31;
    const int gc = lane & 3;
    const int base = j0 + nb;
    const int T = (m + 15) >> 4;
    int tj = 0, ti = first + wid, left = last - first - wid;
    while (tj < T && ti >= T) { ti += tj + 1 - T; ++tj; }
    while (tj < T && left > 0) {
      const int i0 = ti * 16, q0 = tj * 16;
      // this lane's 4 columns of the tile, as window offsets minus the row
      int cb[2][2];
#pragma unroll
      for (int v = 0; v < 2; ++v)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int q = q0 + v * 8 + kperm(2 * gc + e);
          cb[v][e] = slot_from(s0, j0, base + (q < m ? q : 0)) * g.lds - q;
        }
      const int rows = i0 + 16 <= m ? 0 : (i0 + 8 < m ? 1 : 2);
      if (ti != tj) {
        if (rows == 0) tile_update<false, 0>(cb, i0, q0, m);
        else if (rows == 1) tile_update<false, 1>(cb, i0, q0, m);
        else tile_update<false, 2>(cb, i0, q0, m);
      } else {
        if (rows == 0) tile_update<true, 0>(cb, i0, q0, m);
        else if (rows == 1) tile_update<true, 1>(cb, i0, q0, m);
        else tile_update<true, 2>(cb, i0, q0, m);
      }
      ti += nw;
      left -= nw;
      while (tj < T && ti >= T) { ti += tj + 1 - T; ++tj; }
    }
  }

  // ---- pipelined factorization (kd >= 32) -------------------------------------------
  // Three warp roles, no CTA-wide barrier inside the column loop:
  //   pivot (SMSP 0): SYRK of tile (0,0) of update(k-1) -> POTRF(k) (+ L11^-1) -> TRSM of
  //                   panel tile 0 -> signal sig[0] ("panel k ready")
  //   workers (6, SMSPs 1-3): TRSM of panel tiles 1.. -> column 0 of update(k) (signal
  //                   sig[1]) -> the rest of update(k) (signal sig[2 + (k&1)])
  //   light (SMSP 0): write-back of panel k, prefetch of the columns update(k+1) needs
  // The pivot's chain per step is SYRK + POTRF + one 16x16 TRSM; it waits on update(k-2)
  // (finished a whole step earlier) and on column 0 of update(k-1) (one tile per worker,
  // done while the pivot runs its POTRF), so it normally never stalls.  Every mbarrier is
  // at most one phase ahead of its waiters (W is double-buffered by step parity).
  static constexpr int kWorkers = kCtaWarps - 2;
  static constexpr int kBarA = 2, kBarB = 3;  // named barriers (1 is the backward sweep's)

  // light warp: panel write-back (lane 0 issues bulk copies; element-wise when not fast)
  __device__ void light_store(int j0, int nb, int sj) {
    const int lane = threadIdx.x & 31;
    if (fast) {
      if (lane == 0) {
        const unsigned col = (unsigned)g.ldab * sizeof(double);
        const int c1 = min(nb, g.nslot - sj);
        bulk_s2g(ab + (int64_t)j0 * g.ldab, win + (size_t)sj * g.lds, c1 * col);
        if (c1 < nb) bulk_s2g(ab + (int64_t)(j0 + c1) * g.ldab, win, (nb - c1) * col);
        bulk_commit();
      }
      return;
    }
    for (int c = 0; c < nb; ++c) {
      const int sl = slot_from(sj, j0, j0 + c);
      for (int o = lane; o < g.ldab; o += 32) ab[(int64_t)(j0 + c) * g.ldab + o] = win[sl * g.lds + o];
    }
    __syncwarp();
  }
  // light warp: columns [jlo, jhi) into the ring from slot sj on;
  // completes one phase of bars[0]
  __device__ void light_load(int jlo, int jhi, int sj) {
    const int lane = threadIdx.x & 31;
    if (fast) {
      if (lane == 0) {
        bulk_wait_read0();  // the write-back that read these slots is done reading
        const unsigned col = (unsigned)g.ldab * sizeof(double);
        mbar_expect_tx(bars, (unsigned)(jhi - jlo) * col);
        const int c1 = min(jhi - jlo, g.nslot - sj);
        bulk_g2s(win + (size_t)sj * g.lds, ab + (int64_t)jlo * g.ldab, c1 * col, bars);
        if (c1 < jhi - jlo) bulk_g2s(win, ab + (int64_t)(jlo + c1) * g.ldab, (jhi - jlo - c1) * col, bars);
      }
    } else {
      for (int j = jlo; j < jhi; ++j) {
        const int sl = slot_from(sj, jlo, j);
        for (int o = lane; o < g.ldab; o += 32) win[sl * g.lds + o] = ab[(int64_t)j * g.ldab + o];
      }
    }
    __syncwarp();
    if (!fast && lane == 0) mbar_arrive(bars);  // plain arrival: completes the phase
  }

  __device__ void pivot_loop(int nblk, volatile int* s_fail) {
    const int n = g.n, kd = g.kd, lane = threadIdx.x & 31;
    double* const Dbase = D;
    int s0 = 0, sp = 0, mp = 0;
    for (int k = 0; k < nblk; ++k) {
      const int j0 = k * NB, nb = min(NB, n - j0);
      const int m = min(kd, n - j0 - nb);
      trace_stamp(k, 0);
      if (k >= 2) mbar_wait(sig + 2 + (k & 1), ((k - 2) >> 1) & 1);  // update(k-2) complete
      trace_stamp(k, 1);
      if (k >= 1) {
        // tile (0,0) of update(k-1) (this block), from P rows 0..15 = X0(k-1)
        update_tiles(sp, j0 - NB, NB, mp, 0, 1, 0, 1);
        __syncwarp();
      }
      trace_stamp(k, 2);
      D = Dbase + (k & 1) * NB * kLDD;
      const int f = potrf_diag(s0, j0, nb);
      trace_stamp(k, 3);
      // column 0 of update(k-1) done: A(k+1, k) is final and P rows 0..15 are free.  Also
      // waited when there is no TRSM (last block, failure): it proves every worker and the
      // light warp consumed sig[0] phase k-1, so sig[0] never runs two phases ahead
      if (k >= 1) mbar_wait(sig + 1, (k - 1) & 1);
      trace_stamp(k, 4);
      if (f >= 0) {
        if (lane == 0) *s_fail = j0 + f;
        __syncwarp();
        if (lane == 0) mbar_arrive(sig);
        break;
      }
      if (m > 0) trsm_panel(s0, j0, nb, m, 0, 1 << 20);
      fence_async_smem();  // L11 and X0 in the window -> the light warp's bulk write-back
      __syncwarp();
      if (lane == 0) mbar_arrive(sig);
      trace_stamp(k, 5);
      sp = s0;
      mp = m;
      s0 += NB;
      if (s0 >= g.nslot) s0 -= g.nslot;
    }
    D = Dbase;
  }

  __device__ void worker_loop(int nblk, volatile int* s_fail) {
    const int n = g.n, kd = g.kd, lane = threadIdx.x & 31;
    double* const Dbase = D;
    unsigned lph = phase;  // parity of the next window-load completion
    int s0 = 0, ring0 = 0;
    for (int k = 0; k < nblk; ++k) {
      const int j0 = k * NB, nb = min(NB, n - j0);
      const int m = min(kd, n - j0 - nb);
      mbar_wait(sig, k & 1);  // panel k: L11^-1(k) in D, X0 in P rows 0..15
      if (*s_fail >= 0) break;
      const int tw = 2 * nblk + 2 + k;  // worker 0's trace row (after the backward sweep's)
      if (wk == 0) { trace_stamp(k, 6); trace_stamp(tw, 0); }
      if (wk == 0) trace_stamp(tw, 1);
      named_bar(kBarA, 32 * kWorkers);  // update(k-1) done by every worker
      if (wk == 0) trace_stamp(tw, 2);
      D = Dbase + (k & 1) * NB * kLDD;
      if (m > NB) trsm_panel(s0, j0, nb, m, 1 + wk, kWorkers);
      fence_async_smem();
      if (wk == 0) trace_stamp(tw, 3);
      // tile column 0 of update(k) (the next panel): tile (t, 0) needs only this warp's own
      // TRSM tile X_t and the pivot's X_0, so it runs before barrier B
      const int T = (m + 15) >> 4;
      __syncwarp();
      update_tiles(s0, j0, nb, m, 1, T, wk, kWorkers);
      __syncwarp();
      if (lane == 0) mbar_arrive(sig + 1);
      if (wk == 0) trace_stamp(tw, 4);
      named_bar(kBarB, 32 * (kWorkers + 1));  // panel k complete (+ the light warp)
      // the columns update(k) brings into the window (prefetched at step k-1): only the last
      // tile columns of the rest below touch them -- TRSM(k) and tile column 0 do not -- so
      // the copy has had those phases to land
      if (k >= 1 && k * NB + kd < n) {
        mbar_wait(bars, lph);
        lph ^= 1u;
      }
      if (wk == 0) trace_stamp(tw, 5);
      // the rest, starting with the workers that had no column-0 tile
      const int first = (T - 1) % kWorkers;
      update_tiles(s0, j0, nb, m, T, 1 << 20, (wk + kWorkers - first) % kWorkers, kWorkers);
      if (fb) {
        // fused forward sweep: acc[rows below] -= X(k) y_k for panel rows 16.. (the light warp
        // did y_k and rows 0..15 right after barrier B: long done, the wait is a formality)
        mbar_wait(sig + 4, k & 1);
        forward_tail(m, ring0, wk);
        ring0 += NB;
        if (ring0 >= cta_fwd_ring(kd)) ring0 = 0;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(sig + 2 + (k & 1));
      if (wk == 0) { trace_stamp(k, 7); trace_stamp(tw, 6); }
      s0 += NB;
      if (s0 >= g.nslot) s0 -= g.nslot;
    }
    D = Dbase;
  }

  // Fused forward sweep, light warp, step k, after barrier B (panel k complete: L11^-1(k) in
  // D[k & 1], the panel X(k) dense in P) -- the block form of core.py:216-240's forward loop:
  //   forward_head (light warp): y_k = L11^-1 (b_k + acc_k), acc[rows j0+16..j0+31] -= X0(k) y_k.
  //                 D[k & 1] and P rows 0..15 stay valid until the pivot's POTRF(k+2) / TRSM(k+1),
  //                 ordered after this warp's sig[1] arrival of step k.
  //   forward_tail (workers, after their share of update(k)): acc[rows below] -= X(k) y_k for
  //                 panel rows 16.., which the workers overwrite in TRSM(k+1), after their barrier A.
  // The light warp's share is kept minimal: measured, anything it runs on the pivots' SM
  // sub-partition lengthens both CTAs' POTRF chains.
  __device__ __forceinline__ void forward_head(int j0, int nb, int m, int ring0, const double* Dk, double& bnext) {
    const int lane = threadIdx.x & 31, i = lane & 15;
    const int nxf = cta_fwd_ring(g.kd);
    double* sv = fws + nxf;
    double* sy = sv + 16;
    const double bcur = bnext;
    {
      const int jn = j0 + NB + i;  // next step's rows, a step ahead of their use
      bnext = (lane < 16 && jn < g.n) ? fb[jn] : 0.0;
    }
    if (lane < 16) {
      const double a = fws[ring0 + i];
      fws[ring0 + i] = 0.0;  // the slot's next row starts from zero
      sv[i] = i < nb ? bcur + a : 0.0;
    }
    __syncwarp();
    double y = 0.0;
    {
      const double* dr = Dk + i * kLDD;  // row i of L11^-1 (zeros right of the diagonal)
      double a4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int kk = 0; kk < 16; kk += 2) {
        const double2 d2 = *reinterpret_cast<const double2*>(dr + kk);
        const double2 v2 = *reinterpret_cast<const double2*>(sv + kk);
        a4[kk & 3] = fma(d2.x, v2.x, a4[kk & 3]);
        a4[(kk + 1) & 3] = fma(d2.y, v2.y, a4[(kk + 1) & 3]);
      }
      y = (a4[0] + a4[1]) + (a4[2] + a4[3]);
    }
    if (lane < 16) {
      sy[i] = y;
      if (i < nb) fy[j0 + i] = y;
    }
    __syncwarp();
    // panel rows 0..15 (lanes 16-31 mirror lanes 0-15 and do not store)
    if (m > 0) {
      double a4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int c = 0; c < 16; ++c) a4[c & 3] = fma(P[c * g.pld + i], sy[c], a4[c & 3]);
      int rs = ring0 + NB + i;
      if (rs >= nxf) rs -= nxf;
      if (lane < 16 && i < m) fws[rs] -= (a4[0] + a4[1]) + (a4[2] + a4[3]);
    }
    __syncwarp();
  }

  // worker wid, at the end of its share of update(k): rows 16 + 32 wid + lane of the panel
  // (row r is always updated by the same thread within a step; steps are ordered by the
  // workers' barrier A)
  __device__ __forceinline__ void forward_tail(int m, int ring0, int wid) {
    const int lane = threadIdx.x & 31;
    const int r = NB + 32 * wid + lane;
    if (32 * wid + NB >= m) return;  // (warp-uniform)
    const int nxf = cta_fwd_ring(g.kd);
    const double* sy = fws + nxf + 16;
    const double* pr = P + (r < m ? r : 0);
    double l[16];
#pragma unroll
    for (int c = 0; c < 16; ++c) l[c] = pr[c * g.pld];
    double a4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
    for (int c = 0; c < 16; c += 2) {
      const double2 y2 = *reinterpret_cast<const double2*>(sy + c);
      a4[c & 3] = fma(l[c], y2.x, a4[c & 3]);
      a4[(c + 1) & 3] = fma(l[c + 1], y2.y, a4[(c + 1) & 3]);
    }
    int rs = ring0 + NB + r;
    if (rs >= nxf) rs -= nxf;
    if (r < m) fws[rs] -= (a4[0] + a4[1]) + (a4[2] + a4[3]);
  }

  __device__ int light_loop(int nblk, volatile int* s_fail) {
    const int n = g.n, kd = g.kd;
    int s0 = 0, nload = 0, ring0 = 0;
    double bnext = 0.0;
    if (fb) {
      const int lane = threadIdx.x & 31;
      bnext = (lane < 16 && lane < n) ? fb[lane] : 0.0;
    }
    for (int k = 0; k < nblk; ++k) {
      const int j0 = k * NB, nb = min(NB, n - j0);
      const int m = min(kd, n - j0 - nb);
      mbar_wait(sig, k & 1);
      if (*s_fail >= 0) break;
      named_bar(kBarB, 32 * (kWorkers + 1));  // panel k complete
      // write-back and prefetch first (the forward step does not read the window), so the
      // columns update(k+1) needs are in flight while it runs
      light_store(j0, nb, s0);
      const int jlo = j0 + NB + kd;
      if (jlo < n) {
        light_load(jlo, min(n, jlo + NB), slot_from(s0, j0, jlo));
        ++nload;
      }
      if (fb) {
#ifdef BCG_TRACE
        const unsigned long long tf0 = gtime();
#endif
        forward_head(j0, nb, m, ring0, D + (k & 1) * NB * kLDD, bnext);
        if ((threadIdx.x & 31) == 0) mbar_arrive(sig + 4);  // y_k is in shared memory: the workers' forward_tail
#ifdef BCG_TRACE
        if (tr && (threadIdx.x & 31) == 0) {  // duration of the forward step (worker-0 trace row, slot 7)
          const unsigned long long idx = 1 + (unsigned long long)(2 * nblk + 2 + k) * kTracePhases + 7;
          if (idx < g_trace_cap) tr[idx] = gtime() - tf0;
        }
#endif
        ring0 += NB;
        if (ring0 >= cta_fwd_ring(kd)) ring0 = 0;
      }
      __syncwarp();
      // After barrier B (the workers arrive before it), so sig[0] never runs two phases ahead
      // of this warp; after the forward step, so P(k) and D[k & 1] may be overwritten: the
      // pivot awaits this arrival before TRSM(k+1), and the workers' TRSM(k+1) follows the
      // pivot's next signal.
      if ((threadIdx.x & 31) == 0) mbar_arrive(sig + 1);
      s0 += NB;
      if (s0 >= g.nslot) s0 -= g.nslot;
    }
    return nload;
  }

  __device__ int factor_la() {
    const int n = g.n, kd = g.kd;
    __shared__ int s_fail, s_nload;
    const int warp = warp_uniform(threadIdx.x >> 5);
    init_fast();
    for (int idx = threadIdx.x; idx < NB * g.pld; idx += kCtaThreads) P[idx] = 0.0;
    if (fb)
      for (int idx = threadIdx.x; idx < (int)cta_fwd_doubles(kd); idx += kCtaThreads) fws[idx] = 0.0;
    if (threadIdx.x == 0) {
      // sig[1] (column 0 done) also counts the light warp's arrival right after it consumed
      // sig[0]: the workers arrive before barrier B, so without it the pivot could complete
      // sig[0] twice before the light warp waited once
      for (int i = 0; i < 4; ++i) mbar_init(sig + i, i == 0 ? 1 : (i == 1 ? kWorkers + 1 : kWorkers));
      mbar_init(sig + 4, 1);  // y_k ready (fused forward sweep)
      s_fail = -1;
      s_nload = 0;
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    load_cols(0, min(n, kd + NB));
    wait_cols();  // (CTA barrier: also publishes the mbarrier init)
    const int nblk = (n + NB - 1) / NB;
    if (warp == pw) {
      pivot_loop(nblk, &s_fail);
    } else if (wk >= 0) {
      worker_loop(nblk, &s_fail);
    } else {
      const int nload = light_loop(nblk, &s_fail);
      if ((threadIdx.x & 31) == 0) {
        s_nload = nload;
        if (nload > 0) mbar_wait(bars, phase ^ ((unsigned)(nload - 1) & 1u));  // the last prefetch landed
        bulk_wait0();  // write-backs complete
        fence_async_global();
      }
    }
    __syncthreads();
    phase ^= (unsigned)s_nload & 1u;
    const int fail = s_fail;
    if (threadIdx.x == 0)
      for (int i = 0; i < 5; ++i) asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(sig + i)) : "memory");
    __syncthreads();
    return fail < 0 ? -1 : fail;
  }

  // Whole factorization: the pipelined kernel for kd >= 32, else the lock-step loop below.
  // Returns -1 or the failing column.
  __device__ int factor() {
    if (g.kd >= 32) return factor_la();
    const int n = g.n, kd = g.kd;
    __shared__ int s_fail;
    const int warp = threadIdx.x >> 5;
    init_fast();
    // zero the panel buffer once (rows past m are read, never used, by the tile GEMM)
    for (int idx = threadIdx.x; idx < NB * g.pld; idx += kCtaThreads) P[idx] = 0.0;
    load_cols(0, min(n, kd + NB));
    wait_cols();
    // Loop rotated so that one call site factors every diagonal block.  Iteration k:
    //   warp pw:           tile (0,0) of update(k-1) -> POTRF(k) (+ L11^-1)
    //   6 other warps:     the rest of update(k-1)            (warp pw+4 idles: it shares
    //                                                          the POTRF's sub-partition)
    //   barrier, TRSM(k) as a DMMA product (all warps), barrier,
    //   write-back of panel k, prefetch of the columns step k+1 brings into the window.
    // The per-step chain is POTRF -> TRSM -> one tile update; everything else overlaps.
    int jp = -NB, sp = 0, nbp = 0, mp = 0;  // previous step
    int j0 = 0, s0 = 0;
    for (;;) {
      const int nb = min(NB, n - j0);
      const int step = j0 / NB;
      if (kd < NB && pending) wait_cols();  // the last prefetch overlaps this panel
      // warp_uniform(): tell ptxas the branch cannot split a warp, so the POTRF's
      // shuffles compile to plain SHFL instead of collective divergence handling
      const int wu = warp_uniform(warp);
      if (wu == pw) {
        // the previous step's update of this block (tile (0,0)), then POTRF: no CTA
        // barrier between the TRSM that fed it and this POTRF
        if (jp >= 0) {
          update_tiles(sp, jp, nbp, mp, 0, 1, 0, 1);
          __syncwarp();
        }
        trace_stamp(step, 3);
        const int f = potrf_diag(s0, j0, nb);
        if ((threadIdx.x & 31) == 0) s_fail = f;
        trace_stamp(step, 4);
      } else if (wk >= 0 && jp >= 0) {
        // the rest of the previous step's update, on the other three SM sub-partitions
        update_tiles(sp, jp, nbp, mp, 1, 1 << 20, wk, kCtaWarps - 2);
        if (wk == 0) trace_stamp(step, 5);
      }
      __syncthreads();
      if (threadIdx.x < 32) trace_stamp(step, 6);
      const int fl = warp_uniform(s_fail);
      if (fl >= 0) {
        drain();
        return j0 + fl;
      }
      const int m = min(kd, n - j0 - nb);
      if (threadIdx.x < 32) trace_stamp(step, 0);
      // TRSM on the six warps off the POTRF warps' sub-partition: a DMMA queued on that
      // SMSP stalls the other CTA's pivot chain for hundreds of cycles
      // (tools/micro/pipe_mix.cu: a dependent DFMA 8.7 -> 73 cycles with one DMMA warp there)
      if (wk >= 0) trsm_panel(s0, j0, nb, m, wk, kCtaWarps - 2);
      if (threadIdx.x < 32) trace_stamp(step, 7);
      fence_async_smem();  // panel writes -> visible to the bulk write-back
      if (pending) wait_cols();  // columns prefetched by the previous step
      else __syncthreads();
      if (threadIdx.x < 32) trace_stamp(step, 1);
      store_cols(j0, nb);
      // prefetch the columns step k+1 brings into the window (into the slots just
      // written back, once the write-back has read them)
      const int jlo = j0 + NB + kd;
      if (jlo < n) load_cols(jlo, min(n, jlo + NB));
      if (threadIdx.x < 32) trace_stamp(step, 2);
      if (j0 + nb >= n) break;
      jp = j0; sp = s0; nbp = nb; mp = m;
      j0 += nb;
      s0 += nb;
      if (s0 >= g.nslot) s0 -= g.nslot;
    }
    drain();
    return -1;
  }

  // finish every async copy of this matrix (loads landed, write-backs complete)
  __device__ void drain() {
    if (pending) wait_cols();
    if (threadIdx.x == kCopyThread) {
      bulk_wait0();
      fence_async_global();
    }
    __syncthreads();
  }
};

}  // namespace bcg
