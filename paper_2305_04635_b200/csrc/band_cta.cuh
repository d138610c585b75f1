// band_cta.cuh -- one thread block factors (and optionally solves) one band matrix.
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
//     critical path instead of rsqrt + shuffle + mul + fma.  The forward sweep of
//     the solve rides along in the same loop.
//   * Lookahead: the update of step k is split; the part that touches the next
//     panel's columns runs first, then warp 0 factors the next diagonal block
//     while warps 1-7 finish the rest of step k's update.
//   * The trailing update runs on the FP64 tensor path (mma.sync m8n8k4 f64 ->
//     DMMA), 16x16 warp tiles, operands from a dense panel copy P whose leading
//     dimension is 4 (mod 16) doubles (conflict-free fragment loads).
//   * Backward sweep (fused solve): L is streamed back through the same ring with a
//     cp.async pipeline several blocks deep.
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
    if (phase == 0 && (unsigned long long)j + 1 > tr[0]) tr[0] = j + 1;
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
  int nx;           // ring of rhs / solution entries (bw): nx slots (= nslot in the fused kernel)
};

// The panel buffer P; the backward sweep reuses it for two L11^-1 blocks.
__host__ __device__ inline size_t cta_panel_doubles(int nb_block, const CtaGeom& g, bool solve) {
  // backward sweep scratch: 3 x (M_b, G_b) + far partials + c + 2 t, of which the two D
  // buffers that follow P in shared memory hold 2 * nb_block * (nb_block + 4) doubles
  const size_t p = (size_t)nb_block * g.pld;
  const size_t need = 6 * (size_t)nb_block * (nb_block + 4) + 192 + 4 * (size_t)nb_block;
  const size_t inv = need - 2 * (size_t)nb_block * (nb_block + 4);
  return (solve && inv > p) ? inv : p;
}

// Column-block buffers of the streamed sweeps (at most 7, at least 5: host geometry).
template <class G>
__host__ __device__ inline int cta_sweep_buffers(int nb_block, const G& g) {
  const int n = g.nslot / nb_block;
  return n < 7 ? n : 7;
}

// Shared-memory footprint (bytes) of one CTA for block size NB.
__host__ __device__ inline size_t cta_smem_bytes(int nb_block, const CtaGeom& g, bool solve) {
  // D: two L11 / L11^-1 buffers (the pipelined factorization alternates them by step)
  size_t d = (size_t)g.nslot * g.lds + cta_panel_doubles(nb_block, g, solve) + 2 * (size_t)nb_block * (nb_block + 4) +
             nb_block;
  if (solve) d += (size_t)g.nx + (size_t)cta_sweep_buffers(nb_block, g) * nb_block;  // rhs ring + staged y
  return d * sizeof(double) + 64;
}

// Compile-time geometry for one band width (the bench configuration): kd, ldab = lds =
// kd + 1, the ring and panel strides exactly as make_geom() (bandchol_b200.cu) picks them,
// so index arithmetic folds to constants and frees registers in the hot loops; n stays
// runtime.  KD = 0 selects the runtime CtaGeom.
template <int KD, bool kSolve>
struct GeomFixed {
  int n;
  static constexpr int kd = KD, ldab = KD + 1, lds = KD + 1;
  static constexpr int ns0 = (kSolve && KD + 16 < 5 * 16) ? 5 * 16 : KD + 16;
  static constexpr int nslot = (ns0 & 1) ? ns0 + 1 : ns0, nx = nslot;
  static constexpr int pld = KD + ((4 - KD % 16) + 16) % 16;
  __host__ __device__ GeomFixed(const CtaGeom& x) : n(x.n) {}
  // true when the runtime geometry the host chose is exactly this one
  __host__ __device__ static bool matches(const CtaGeom& x) {
    return x.kd == kd && x.ldab == ldab && x.lds == lds && x.nslot == nslot && x.nx == nx && x.pld == pld;
  }
};
template <int KD, bool kSolve>
struct GeomOf { using type = GeomFixed<KD, kSolve>; };
template <bool kSolve>
struct GeomOf<0, kSolve> { using type = CtaGeom; };

template <int NB, bool kSolve, int KD = 0>
struct CtaBand {
  static_assert(NB == 16, "block size: lanes 16-31 of the POTRF warp invert L11");
  const typename GeomOf<KD, kSolve>::type g;
  double* __restrict__ ab;   // this matrix in global memory
  double* __restrict__ rhs;  // its right-hand side (kSolve)
  double* win;               // shared ring of column slots
  double* P;                 // NB x pld dense panel, P[c*pld + r] = L(j0+nb+r, j0+c)
  static constexpr int kLDD = NB + 4;  // D stride (= 4 mod 16: conflict-free DMMA fragments)
  double* D;                 // L11, D[c*kLDD + r] = L(r, c); then L11^-1, D[i*kLDD + j] = Linv(i, j)
  double* Dinv;              // 3 x NB doubles of sweep scratch (aliases the second D buffer,
                             // free outside the factorization)
  double* lbuf;              // NB doubles: sink for the inverse lanes' column stores
  double* bw;                // ring of rhs / solution entries, slot(i) like columns
  double* yb;                // backward sweep: nbuf x NB staged y entries; factor: y of the last two blocks
  unsigned long long* bars;  // mbarriers: [0] window loads, [1 + k] backward buffer k
  unsigned long long* sig;   // pipelined factorization: [0] panel ready, [1] column 0 updated, [2 + (k&1)] update done
  unsigned* bphase;          // smem: parity of the next wait on bars[1 + k]
  unsigned phase = 0;        // parity of the next wait on bars[0] (uniform register)
  bool pending = false;      // a load_cols is in flight
  bool fast = false;         // every column chunk meets the bulk-copy alignment rules
  // Warp roles by SM sub-partition (set_roles): the POTRF warp pw and a light warp share
  // SMSP 0 with the other CTA's pivot; the six warps on SMSPs 1-3 run every DMMA.
  int pw = 0;                // the POTRF warp
  int wk = -1;               // this warp's worker index 0..5 (-1: pivot or light warp)
  unsigned long long* tr = nullptr;  // trace buffer (block 0 only), see bcg_set_trace

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

  // async load of columns [jlo, jhi) (and their rhs entries); complete with wait_cols()
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
      if (kSolve) {
        for (int j = jlo + threadIdx.x; j < jhi; j += kCtaThreads) {
          int sl = sj + (j - jlo);
          if (sl >= g.nslot) sl -= g.nslot;
          cp_async8(bw + sl, rhs + j);
        }
        cp_async_commit();
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
    if (kSolve)
      for (int j = jlo + threadIdx.x; j < jhi; j += kCtaThreads) cp_async8(bw + (j % g.nslot), rhs + j);
    cp_async_commit();
    pending = true;
  }
  // all threads: the last load_cols has landed and is visible
  __device__ __forceinline__ void wait_cols() {
    if (kSolve || !fast) cp_async_wait_all();
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

  // Warp pw: Cholesky of the nb x nb diagonal block at column j0 (+ forward sweep).
  // Lane r holds row r.  Returns the local failing column or -1 (uniform).
  //
  // Straight-line for every block: a short last block (nb < NB) is padded with identity
  // rows, so the column loop has no per-column masks.  Column c of D doubles as the
  // broadcast buffer of the rank-1 update (distinct per column, so one __syncwarp per
  // column suffices), lanes NB..31 build L11^-1 along the way, and failure is found
  // once at the end: after a non-positive / NaN pivot every later pivot of the block is
  // NaN, so the first failing column is the first lane whose L(r, r) is not > 0.
  template <bool kFwd>
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
    double s = 0.0;
    if (kFwd && r < nb) s = bw[slot_from(s0, j0, j0 + r)];
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
      if (kFwd) {
        const double yc = __shfl_sync(kFull, s, c) * rs;
        s = (r == c) ? yc : ((r > c) ? fma(-lrc, yc, s) : s);
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
    if (kFwd && r < nb) {
      bw[slot_from(s0, j0, j0 + r)] = s;
      rhs[j0 + r] = s;
      yb[((j0 / NB) & 1) * NB + r] = s;  // y of this block for update_rhs (ring slot is reused)
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

  // Forward-sweep update of the trailing rhs entries: b_i -= sum_c P(i,c) y_c.
  // Rows [lo, min(hi, m)) by threads tid, tid + nt, ...
  __device__ void update_rhs(int s0, int j0, int nb, int m, int lo, int hi, int tid, int nt) {
    const int base = j0 + nb;
    hi = min(hi, m);
    for (int i = lo + tid; i < hi; i += nt) {
      double s = 0.0;
#pragma unroll
      for (int c = 0; c < NB; ++c)
        if (c < nb) s = fma(P[c * g.pld + i], yb[((j0 / NB) & 1) * NB + c], s);
      bw[slot_from(s0, j0, base + i)] -= s;
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
        // tile (0,0) of update(k-1) (this block) and its rhs rows, from P rows 0..15 = X0(k-1)
        update_tiles(sp, j0 - NB, NB, mp, 0, 1, 0, 1);
        __syncwarp();
      }
      trace_stamp(k, 2);
      D = Dbase + (k & 1) * NB * kLDD;
      const int f = potrf_diag<false>(s0, j0, nb);
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
    int s0 = 0;
    for (int k = 0; k < nblk; ++k) {
      const int j0 = k * NB, nb = min(NB, n - j0);
      const int m = min(kd, n - j0 - nb);
      mbar_wait(sig, k & 1);  // panel k: L11^-1(k) in D, X0 in P rows 0..15
      if (*s_fail >= 0) break;
      const int tw = 2 * nblk + 2 + k;  // worker 0's trace row (after the backward sweep's)
      if (wk == 0) { trace_stamp(k, 6); trace_stamp(tw, 0); }
      if (k >= 1 && k * NB + kd < n) {  // the columns update(k) brings in (prefetched at k-1)
        mbar_wait(bars, lph);
        lph ^= 1u;
      }
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
      if (wk == 0) trace_stamp(tw, 5);
      // the rest, starting with the workers that had no column-0 tile
      const int first = (T - 1) % kWorkers;
      update_tiles(s0, j0, nb, m, T, 1 << 20, (wk + kWorkers - first) % kWorkers, kWorkers);
      __syncwarp();
      if (lane == 0) mbar_arrive(sig + 2 + (k & 1));
      if (wk == 0) { trace_stamp(k, 7); trace_stamp(tw, 6); }
      s0 += NB;
      if (s0 >= g.nslot) s0 -= g.nslot;
    }
    D = Dbase;
  }

  __device__ int light_loop(int nblk, volatile int* s_fail) {
    const int n = g.n, kd = g.kd;
    int s0 = 0, nload = 0;
    for (int k = 0; k < nblk; ++k) {
      const int j0 = k * NB, nb = min(NB, n - j0);
      mbar_wait(sig, k & 1);
      if (*s_fail >= 0) break;
      __syncwarp();
      if ((threadIdx.x & 31) == 0) mbar_arrive(sig + 1);
      named_bar(kBarB, 32 * (kWorkers + 1));  // panel k complete
      light_store(j0, nb, s0);
      const int jlo = j0 + NB + kd;
      if (jlo < n) {
        light_load(jlo, min(n, jlo + NB), slot_from(s0, j0, jlo));
        ++nload;
      }
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
    if (threadIdx.x == 0) {
      // sig[1] (column 0 done) also counts the light warp's arrival right after it consumed
      // sig[0]: the workers arrive before barrier B, so without it the pivot could complete
      // sig[0] twice before the light warp waited once
      for (int i = 0; i < 4; ++i) mbar_init(sig + i, i == 0 ? 1 : (i == 1 ? kWorkers + 1 : kWorkers));
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
      for (int i = 0; i < 4; ++i) asm volatile("mbarrier.inval.shared::cta.b64 [%0];" ::"r"(smem_u32(sig + i)) : "memory");
    __syncthreads();
    return fail < 0 ? -1 : fail;
  }

  // Whole factorization (+ forward sweep when kSolve, lock-step loop only).  Returns -1 or
  // the failing column.
  __device__ int factor() {
    // (the fused solve runs the lock-step loop below: for kd >= 32 bcg_dpbsv_batched factors with
    // the pipelined kernel and then runs the streamed solve, which measured faster)
    if (!kSolve && g.kd >= 32) return factor_la();
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
        // the previous step's update of this block (tile (0,0)) and of its rhs rows,
        // then POTRF: no CTA barrier between the TRSM that fed them and this POTRF
        if (jp >= 0) {
          update_tiles(sp, jp, nbp, mp, 0, 1, 0, 1);
          if (kSolve) update_rhs(sp, jp, nbp, mp, 0, NB, threadIdx.x & 31, 32);
          __syncwarp();
        }
        trace_stamp(step, 3);
        const int f = potrf_diag<kSolve>(s0, j0, nb);
        if ((threadIdx.x & 31) == 0) s_fail = f;
        trace_stamp(step, 4);
      } else if (wk >= 0 && jp >= 0) {
        // the rest of the previous step's update, on the other three SM sub-partitions
        update_tiles(sp, jp, nbp, mp, 1, 1 << 20, wk, kCtaWarps - 2);
        if (kSolve) update_rhs(sp, jp, nbp, mp, NB, 1 << 20, (threadIdx.x & 31) + 32 * wk, 32 * (kCtaWarps - 2));
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
      store_cols(j0, nb, kSolve ? s0 : -1);
      // prefetch the columns step k+1 brings into the window (into the slots just
      // written back, once the write-back has read them)
      const int jlo = j0 + NB + kd;
      // (the slot hints measured faster in the fused kernel only; the factor-only kernel
      // keeps the self-computed slots)
      if (jlo < n) load_cols(jlo, min(n, jlo + NB), kSolve ? slot_from(s0, j0, jlo) : -1);
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

  // L11^-1 of a column block held in the ring (blk: NB column slots of lds doubles, nb
  // valid columns; columns past nb are identity).  Warp-level: lane j forward-substitutes
  // L11 x = e_j with the reciprocal pivots computed up front (independent: full ILP).
  // kRowMajor: li[i*kLDD + j] = Linv(i, j); else li[j*kLDD + i] = Linv(i, j).
  template <bool kWhole, bool kRowMajor>
  __device__ void invert_l11(const double* blk, int nb, double* li) const {
    if (kWhole) nb = NB;
    const int j = threadIdx.x & 31;
    double dk[NB];
#pragma unroll
    for (int kk = 0; kk < NB; ++kk) dk[kk] = (kWhole || kk < nb) ? rcp_nr(blk[kk * g.lds]) : 1.0;
    double t[NB];
#pragma unroll
    for (int i = 0; i < NB; ++i) t[i] = (i == j) ? 1.0 : 0.0;
#pragma unroll
    for (int kk = 0; kk < NB; ++kk) {
      const double* col = blk + kk * g.lds;
      t[kk] *= dk[kk];
#pragma unroll
      for (int i = kk + 1; i < NB; ++i) {
        if (kWhole) {
          t[i] = fma(-col[i - kk], t[kk], t[i]);
        } else {
          const bool in = i < nb && i - kk <= g.kd;
          const double lv = col[in ? i - kk : 0];
          t[i] = fma(in ? -lv : 0.0, t[kk], t[i]);
        }
      }
    }
    if (j < NB) {
#pragma unroll
      for (int i = 0; i < NB; ++i) li[kRowMajor ? i * kLDD + j : j * kLDD + i] = t[i];
    }
  }
  template <bool kRowMajor>
  __device__ void invert_block(const double* blk, int nb, double* li) const {
    if (nb == NB && g.kd >= NB - 1) invert_l11<true, kRowMajor>(blk, nb, li);
    else invert_l11<false, kRowMajor>(blk, nb, li);
  }

  // Forward sweep L y = b for the standalone solve (rhs holds b, receives y).
  //
  // Column blocks stream in through the same buffer ring as the backward sweep (bulk
  // copies kDepth blocks ahead); bw (nx slots) holds the running right-hand side of the
  // kd+NB rows in flight.  Iteration b (mirror image of backward()):
  //   warp 0:     near update of block b by block b-1 (16x16 GEMV), y_b = L11^-1 s_b
  //   warp 1:     L11^-1 of block b+1
  //   warps 2-7:  far update of the rows beyond block b by block b-1 (one thread per row),
  //               then the rhs entries of the rows entering the ring
  __device__ void forward() {
    const int n = g.n, kd = g.kd;
    const int lane = threadIdx.x & 31, warp = warp_uniform(threadIdx.x >> 5);
    constexpr int kDepth = 4;
    const int nbuf = cta_sweep_buffers(NB, g);
    const int nblk = (n + NB - 1) / NB;
    double* ycur = Dinv;  // y of the last two blocks (2 x NB)
    const bool early_issue = fast && nbuf >= kDepth + 3;
    double* li_buf = P;
    // parity of the next wait on buffer k (bit k) and ring positions, tracked without divisions
    unsigned pbits = 0;
    for (int k = 0; k < nbuf; ++k) pbits |= (bphase[k] & 1u) << k;
    auto wait_buf = [&](int k) {
      mbar_wait(bars + 1 + k, (pbits >> k) & 1u);
      pbits ^= 1u << k;
    };
    auto inc = [](int v, int by, int mod) { v += by; return v >= mod ? v - mod : v; };
    auto issue = [&](int b, int k) {  // k = b % nbuf
      if (b >= nblk) return;
      const int c0 = b * NB;
      const int cols = min(NB, n - c0);
      if (fast) {
        if (threadIdx.x == 0) {
          const unsigned bytes = (unsigned)cols * g.ldab * sizeof(double);
          mbar_expect_tx(bars + 1 + k, bytes);
          bulk_g2s(win + (size_t)(k * NB) * g.lds, ab + (int64_t)c0 * g.ldab, bytes, bars + 1 + k);
        }
      } else {
        for (int c = 0; c < cols; ++c) {
          double* sp = win + (size_t)(k * NB + c) * g.lds;
          const double* gp = ab + (int64_t)(c0 + c) * g.ldab;
          for (int o = threadIdx.x; o < g.ldab; o += kCtaThreads) sp[o] = gp[o];
        }
        if (threadIdx.x == 0) mbar_expect_tx(bars + 1 + k, 0);
      }
    };
    auto invert = [&](int b, int k) {  // warp 1: L11^-1 of block b into li_buf[b & 1]
      invert_block<true>(win + (size_t)k * NB * g.lds, min(NB, n - b * NB), li_buf + (b & 1) * NB * kLDD);
    };
    // bw accumulates the far updates of the rows in flight (zero when a row enters); warp 0
    // adds the right-hand side itself, prefetched one block ahead into a register
    for (int i = threadIdx.x; i < min(n, kd + NB); i += kCtaThreads) bw[i % g.nx] = 0.0;
    double rnext = (warp == 0 && lane < min(NB, n)) ? rhs[lane] : 0.0;
    for (int d = 0; d < kDepth; ++d) issue(d, d % nbuf);
    wait_buf(0);
    __syncthreads();
    if (warp == 1) invert(0, 0);
    int kb = 0, xb = 0;  // buffer of block b, ring slot of row b*NB
    for (int b = 0; b < nblk; ++b) {
      const int kp1 = inc(kb, 1, nbuf), km1 = kb == 0 ? nbuf - 1 : kb - 1;
      const int c0 = b * NB;
      const int nb = min(NB, n - c0);
      if (threadIdx.x < 32) trace_stamp(b, 0);
      if (b + 1 < nblk) wait_buf(kp1);
      __syncthreads();  // L11^-1(b), far(b-1) and the entering rows are in place
      if (threadIdx.x < 32) trace_stamp(b, 1);
      if (warp == 0) {
        const int r = lane;
        const double rcur = rnext;
        if (c0 + NB + r < n && r < NB) rnext = rhs[c0 + NB + r];  // next block's b, in flight
        double v = (r < nb) ? rcur + bw[inc(xb, r, g.nx)] : 0.0;
        if (b > 0 && r < nb) {
          // near: rows of block b in the columns of block b-1
          const double* blk = win + (size_t)km1 * NB * g.lds;
          const double* yp = ycur + ((b - 1) & 1) * NB;
          double a0 = 0.0, a1 = 0.0;
          if (kd >= 2 * NB - 1) {  // every (row of b, column of b-1) pair is in the band
#pragma unroll
            for (int c = 0; c < NB; c += 2) {
              a0 = fma(blk[c * g.lds + NB + r - c], yp[c], a0);
              a1 = fma(blk[(c + 1) * g.lds + NB + r - c - 1], yp[c + 1], a1);
            }
          } else {
#pragma unroll
            for (int c = 0; c < NB; c += 2) {
              const int o0 = NB + r - c, o1 = o0 - 1;
              if (o0 <= kd) a0 = fma(blk[c * g.lds + o0], yp[c], a0);
              if (o1 <= kd) a1 = fma(blk[(c + 1) * g.lds + o1], yp[c + 1], a1);
            }
          }
          v -= a0 + a1;
        }
        double* ss = Dinv + 2 * NB;
        if (r < NB) ss[r] = v;
        __syncwarp();
        const double* li = li_buf + (b & 1) * NB * kLDD + (r < NB ? r : 0) * kLDD;
        double x0 = 0.0, x1 = 0.0;
#pragma unroll
        for (int c = 0; c < NB; c += 4) {
          const double2 l01 = *reinterpret_cast<const double2*>(li + c);
          const double2 l23 = *reinterpret_cast<const double2*>(li + c + 2);
          const double2 s01 = *reinterpret_cast<const double2*>(ss + c);
          const double2 s23 = *reinterpret_cast<const double2*>(ss + c + 2);
          x0 = fma(l01.x, s01.x, x0);
          x1 = fma(l01.y, s01.y, x1);
          x0 = fma(l23.x, s23.x, x0);
          x1 = fma(l23.y, s23.y, x1);
        }
        v = x0 + x1;
        if (r < nb) {
          ycur[(b & 1) * NB + r] = v;
          rhs[c0 + r] = v;
        }
        trace_stamp(b, 2);
        // with >= kDepth + 3 buffers the slot block b + kDepth goes to (block b-3's) is already
        // free: the chain warp issues it now rather than after the barrier
        if (early_issue) issue(b + kDepth, inc(kb, kDepth, nbuf));
      } else if (warp == 1) {
        if (b + 1 < nblk) invert(b + 1, kp1);
        trace_stamp(b, 4);
      } else if (b > 0) {
        // far: rows i in [c0 + nb, (c0 - NB) + NB - 1 + kd] lose L(i, block b-1) . y_{b-1}
        const double* blk = win + (size_t)km1 * NB * g.lds;
        const double* yp = ycur + ((b - 1) & 1) * NB;
        const int cprev = c0 - NB;
        const int ihi = min(n - 1, cprev + NB - 1 + kd);
        for (int i = c0 + nb + (int)threadIdx.x - 64; i <= ihi; i += kCtaThreads - 64) {
          double acc0 = 0.0, acc1 = 0.0;
          const int o0 = i - cprev;
          if (o0 - (NB - 1) <= kd && o0 <= kd) {  // the whole row segment is in the band
#pragma unroll
            for (int c = 0; c < NB; c += 2) {
              acc0 = fma(blk[c * g.lds + o0 - c], yp[c], acc0);
              acc1 = fma(blk[(c + 1) * g.lds + o0 - c - 1], yp[c + 1], acc1);
            }
          } else {
#pragma unroll
            for (int c = 0; c < NB; c += 2) {
              if (o0 - c <= kd) acc0 = fma(blk[c * g.lds + o0 - c], yp[c], acc0);
              if (o0 - c - 1 <= kd) acc1 = fma(blk[(c + 1) * g.lds + o0 - c - 1], yp[c + 1], acc1);
            }
          }
          bw[i % g.nx] -= acc0 + acc1;
        }
        if (warp == 2) trace_stamp(b, 5);
      }
      if (warp >= 2) {
        // rows entering the ring: first touched by far(b) in the next iteration
        const int lo = c0 + kd + NB, hi = min(n, lo + NB);
        for (int i = lo + (int)threadIdx.x - 64; i < hi; i += kCtaThreads - 64) bw[i % g.nx] = 0.0;
      }
      __syncthreads();
      if (threadIdx.x < 32) trace_stamp(b, 3);
      if (!early_issue) issue(b + kDepth, inc(kb, kDepth, nbuf));  // block b-1's buffer is free now
      kb = kp1;
      xb = inc(xb, NB, g.nx);
    }
    __syncthreads();
    if (threadIdx.x < nbuf) {
      int cnt = 0;
      for (int b = threadIdx.x; b < nblk; b += nbuf) ++cnt;
      bphase[threadIdx.x] = (bphase[threadIdx.x] + (unsigned)cnt) & 1u;
    }
    if (threadIdx.x == 0) fence_async_global();  // y (generic stores) -> the backward's bulk reads
    __syncthreads();
  }

  // Backward-sweep inverter (one warp): lane j < 16 solves z^T L_bb = e_j^T (row j of
  // M = L_bb^-1), lane 16 + j solves z^T L_bb = row j of B (row j of G = B M, B = L(rows of
  // the next block, cols of this one)); z_k = r_k / L_kk for k = NB-1..0, then
  // r_i -= z_k L(k, i) for i < k, L entries broadcast from the ring buffer.  Rows go to
  // out[j*kLDD] (M) and out[NB*kLDD + j*kLDD] (G).  kWhole: every entry in the band.
  template <bool kWhole>
  __device__ void invert_bt(const double* blk, int nb, int c0, double* out, double* dsc) const {
    const int lane = threadIdx.x & 31, j = lane & 15;
    const bool isg = lane >= 16;
    if (lane < NB) dsc[lane] = lane < nb ? rcp_nr(blk[lane * g.lds]) : 1.0;
    double r[NB];
#pragma unroll
    for (int kk = 0; kk < NB; ++kk) {
      const int o = NB + j - kk;  // B(j, kk) = L(c0 + NB + j, c0 + kk)
      const bool inb = kWhole || (kk < nb && c0 + NB + j < g.n && o <= g.kd);
      const double bv = blk[kk * g.lds + (inb ? o : 0)];
      r[kk] = isg ? (inb ? bv : 0.0) : (kk == j ? 1.0 : 0.0);
    }
    __syncwarp();
#pragma unroll
    for (int kk = NB - 1; kk >= 0; --kk) {
      const double z = r[kk] * dsc[kk];
      r[kk] = z;
#pragma unroll
      for (int i = 0; i < kk; ++i) {
        if (kWhole) {
          r[i] = fma(-blk[i * g.lds + kk - i], z, r[i]);
        } else {
          const bool inb = kk < nb && kk - i <= g.kd;
          const double lv = blk[i * g.lds + (inb ? kk - i : 0)];
          r[i] = fma(inb ? -lv : 0.0, z, r[i]);
        }
      }
    }
    double* dst = out + (isg ? NB * kLDD : 0) + j * kLDD;
#pragma unroll
    for (int kk = 0; kk < NB; kk += 2) *reinterpret_cast<double2*>(dst + kk) = make_double2(r[kk], r[kk + 1]);
    __syncwarp();
  }

  // Backward sweep L^T x = y (y in rhs after the forward sweep).
  //
  // Block b = columns [b*NB, b*NB+nb).  With M_b = L_bb^-1, B_b = L(rows of block b+1, cols
  // of block b) and G_b = B_b M_b:
  //   x_b = M_b^T (c_b - B_b^T x_{b+1}) = t_b - G_b^T x_{b+1},
  //   c_b = y_b - sum over rows beyond block b+1 of L(i, block b)^T x_i,  t_b = M_b^T c_b,
  // so the per-block chain is one 16x16 product.  Iteration b runs
  //   warp 0 (chain):      x_b = t_b - G_b^T x_{b+1}
  //   warp 1 (inverter):   rows of M_{b-2} (lanes 0-15) and of G_{b-2} (lanes 16-31): one
  //                        back substitution z^T L_bb = [e_j | row j of B], same instructions
  //   warps 2-7 (far):     c_{b-1} (tensor-path partial sums, fixed-order reduction)
  // and one CTA barrier.  L blocks (and the y entries) stream in with bulk copies nbuf-1
  // blocks ahead of their first use (the inverter's), one mbarrier per ring buffer.
  __device__ void backward() {
    const int n = g.n;
    const int lane = threadIdx.x & 31, warp = warp_uniform(threadIdx.x >> 5);
    const int nbuf = cta_sweep_buffers(NB, g);
    const int nblk = (n + NB - 1) / NB;
    const bool bulk_y = fast && !(((uintptr_t)rhs) & 15);
    // parity of the next wait on buffer k's mbarrier, bit k (no divisions in the loop)
    unsigned pbits = 0;
    for (int k = 0; k < nbuf; ++k) pbits |= (bphase[k] & 1u) << k;
    auto wait_buf = [&](int k) {
      mbar_wait(bars + 1 + k, (pbits >> k) & 1u);
      pbits ^= 1u << k;
    };
    auto issue = [&](int b, int k) {  // k = b % nbuf
      if (b < 0) return;
      const int c0 = b * NB;
      const int cols = min(NB, n - c0);
      if (fast) {
        if (threadIdx.x == 0) {
          const unsigned bytes = (unsigned)cols * g.ldab * sizeof(double);
          const unsigned ybytes = (bulk_y && cols % 2 == 0) ? cols * sizeof(double) : 0;
          mbar_expect_tx(bars + 1 + k, bytes + ybytes);
          bulk_g2s(win + (size_t)(k * NB) * g.lds, ab + (int64_t)c0 * g.ldab, bytes, bars + 1 + k);
          if (ybytes) bulk_g2s(yb + k * NB, rhs + c0, ybytes, bars + 1 + k);
          else for (int t = 0; t < cols; ++t) yb[k * NB + t] = rhs[c0 + t];
        }
      } else {
        // element-wise fallback: synchronous copies, visible after the caller's barrier
        for (int c = 0; c < cols; ++c) {
          double* sp = win + (size_t)(k * NB + c) * g.lds;
          const double* gp = ab + (int64_t)(c0 + c) * g.ldab;
          for (int o = threadIdx.x; o < g.ldab; o += kCtaThreads) sp[o] = gp[o];
        }
        for (int t = threadIdx.x; t < cols; t += kCtaThreads) yb[k * NB + t] = rhs[c0 + t];
        if (threadIdx.x == 0) mbar_expect_tx(bars + 1 + k, 0);
      }
    };
    // scratch in P (and the D buffers after it): 3 slots of (M_b, G_b), far partials, c
    constexpr int kMG = 2 * NB * kLDD;
    constexpr int kFarThreads = kCtaThreads - 64, kFarChunks = kFarThreads / NB;
    double* mg = P;
    double* part = P + 3 * kMG;
    double* tbuf = part + kFarThreads + NB;  // c of two blocks (2 x NB), for the chain's M_b^T c_b
    double* dsc = tbuf + 2 * NB;      // the inverter's pivot reciprocals (NB)
    auto mslot = [&](int b) { return mg + (b % 3) * kMG; };
    // inverter: lane j < 16 solves z^T L_bb = e_j^T (row j of M_b), lane 16 + j solves
    // z^T L_bb = row j of B_b (row j of G_b = B_b M_b); z_k = r_k / L_kk for k = 15..0, then
    // r_i -= z_k L(k, i) for i < k (L entries broadcast from the ring buffer)
    auto invert = [&](int b, int k) {
      const int c0 = b * NB, nb = min(NB, n - c0);
      const double* blk = win + (size_t)k * NB * g.lds;
      if (nb == NB && g.kd >= 2 * NB - 1 && c0 + 2 * NB <= n)
        invert_bt<true>(blk, nb, c0, mslot(b), dsc);
      else
        invert_bt<false>(blk, nb, c0, mslot(b), dsc);
    };
    // far warps: c_b = y_b - sum_{rows beyond block b+1} L(i, c0+c) x_i (thread (chunk q,
    // column c) sums rows o_lo + q, + kFarChunks, ...; chunk partials added in a fixed order),
    // then t_b = M_b^T c_b by the first far warp (lane (i, h): half h of row i's products)
    auto far_t = [&](int b, int k, int sx) {  // k = b % nbuf, sx = ring slot of row b*NB + nb + NB
      // (tensor path: sum_rows L(row, c0 + col) x_row is a 16 x R by R x 1 product, k-steps of
      // four rows dealt round-robin to the six warps, x in column 0 of B; the six partial
      // columns are added in a fixed order, so the result is deterministic)
      const int c0 = b * NB;
      const int nb = min(NB, n - c0);
      const double* blk = win + (size_t)k * NB * g.lds;
      const int rlo = c0 + nb + NB;  // first row of block b+2
      const int rhi = min(n - 1, c0 + nb - 1 + g.kd);
      const int t = threadIdx.x - 64;
      const int fw = t >> 5, gr = lane >> 2, gc = lane & 3;
      double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
      const int nks = rhi >= rlo ? (rhi - rlo + 4) >> 2 : 0;
      for (int ks = fw; ks < nks; ks += kFarThreads / 32) {
        const int row = rlo + 4 * ks + gc;
        int sl = sx + 4 * ks + gc;
        if (sl >= g.nx) sl -= g.nx;
        const double xv = (gr == 0 && row <= rhi) ? bw[sl] : 0.0;
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int col = 8 * u + gr;
          const int off = row - c0 - col;
          const bool in = col < nb && row <= rhi && off <= g.kd;
          const double av = blk[col * g.lds + (in ? off : 0)];
          dmma884(acc[u][0], acc[u][1], in ? av : 0.0, xv);
        }
      }
      if (gc == 0) {
        part[fw * NB + gr] = acc[0][0];
        part[fw * NB + 8 + gr] = acc[1][0];
      }
      asm volatile("bar.sync 1, %0;" ::"n"(kFarThreads) : "memory");
      if (t < 32) {
        const int i = t & 15;
        double sum = 0.0;
#pragma unroll
        for (int w = 0; w < kFarThreads / 32; ++w) sum += part[w * NB + i];
        // c_b for the chain (which applies M_b^T itself, in parallel with its G_b^T product)
        if (t < NB) tbuf[(b & 1) * NB + t] = t < nb ? yb[k * NB + t] - sum : 0.0;
      }
    };
    // chain: x_b = M_b^T c_b - G_b^T x_{b+1} (lane (i, h): half h of columns i of M and G, the
    // two products in parallel), to the x ring and to rhs
    auto chain = [&](int b, int xb) {  // xb = ring slot of row b*NB
      const int c0 = b * NB, nb = min(NB, n - c0);
      const int i = lane & 15, h = lane >> 4;
      double a0 = 0.0, a1 = 0.0, m0 = 0.0, m1 = 0.0;
      {
        // t_b = M_b^T c_b (c_b from the far warps), half h of column i of M
        const double* M = mslot(b) + (8 * h) * kLDD + i;  // M(8h + jj, i)
        const double* cv = tbuf + (b & 1) * NB + 8 * h;
#pragma unroll
        for (int jj = 0; jj < 8; jj += 2) {
          m0 = fma(M[jj * kLDD], cv[jj], m0);
          m1 = fma(M[(jj + 1) * kLDD], cv[jj + 1], m1);
        }
      }
      if (b + 1 < nblk) {
        const double* G = mslot(b) + NB * kLDD + (8 * h) * kLDD + i;  // G(8h + jj, i)
        int sx = xb + nb + 8 * h;  // row c0 + nb + 8h
        if (sx >= g.nx) sx -= g.nx;
#pragma unroll
        for (int jj = 0; jj < 8; jj += 2) {
          int s0 = sx + jj, s1 = sx + jj + 1;
          if (s0 >= g.nx) s0 -= g.nx;
          if (s1 >= g.nx) s1 -= g.nx;
          const int r0 = c0 + nb + 8 * h + jj;
          const double x0 = r0 < n ? bw[s0] : 0.0, x1 = r0 + 1 < n ? bw[s1] : 0.0;
          a0 = fma(G[jj * kLDD], x0, a0);
          a1 = fma(G[(jj + 1) * kLDD], x1, a1);
        }
      }
      double s = (m0 + m1) - (a0 + a1);
      s += __shfl_xor_sync(kFull, s, 16);
      const double x = s;
      if (lane < nb) {
        int sr = xb + lane;
        if (sr >= g.nx) sr -= g.nx;
        bw[sr] = x;
        rhs[c0 + lane] = x;
      }
    };
    // ring positions, tracked incrementally: kb = block b's buffer, xb = ring slot of row b*NB
    auto dec = [&](int v, int by, int mod) { v -= by; return v < 0 ? v + mod : v; };
    int kb = (nblk - 1) % nbuf;
    int xb = ((nblk - 1) * NB) % g.nx;
    for (int d = 0; d < nbuf; ++d) issue(nblk - 1 - d, dec(kb, d, nbuf));
    const int tb = nblk + 1;  // trace rows after the factorization's
    // prologue: M/G of the last two blocks, c/t of the last one
    wait_buf(kb);
    __syncthreads();
    if (warp == 1) invert(nblk - 1, kb);
    __syncthreads();
    if (nblk >= 2) wait_buf(dec(kb, 1, nbuf));
    __syncthreads();
    if (warp == 1 && nblk >= 2) invert(nblk - 2, dec(kb, 1, nbuf));
    if (warp >= 2) {
      const int nbl = n - (nblk - 1) * NB;
      int sx = xb + nbl + NB;
      while (sx >= g.nx) sx -= g.nx;
      far_t(nblk - 1, kb, sx);
    }
    __syncthreads();
    issue(nblk - 1 - nbuf, kb);  // the last block is done (inverter, far): its buffer moves on
    for (int b = nblk - 1; b >= 0; --b) {
      const int km1 = dec(kb, 1, nbuf), km2 = dec(kb, 2, nbuf);
      if (threadIdx.x < 32) trace_stamp(tb + b, 0);
      if (b >= 2) wait_buf(km2);  // block b-2 (the inverter's), per thread
      if (threadIdx.x < 32) trace_stamp(tb + b, 1);
      if (warp == 0) {
        chain(b, xb);
        trace_stamp(tb + b, 2);
        // block b is done (far at b+1, inverter at b+2): its buffer takes block b - nbuf, issued
        // here by the chain warp (it has slack) rather than after the barrier
        if (fast && b <= nblk - 2) issue(b - nbuf, kb);
      } else if (warp == 1) {
        if (b >= 2) invert(b - 2, km2);
        trace_stamp(tb + b, 4);
      } else if (b >= 1) {
        int sxf = xb + NB;  // row (b-1)*NB + NB + NB = c0 + NB
        if (sxf >= g.nx) sxf -= g.nx;
        far_t(b - 1, km1, sxf);
        if (warp == 2) trace_stamp(tb + b, 5);
      }
      __syncthreads();
      if (threadIdx.x < 32) trace_stamp(tb + b, 3);
      if (!fast && b <= nblk - 2) issue(b - nbuf, kb);  // element-wise fallback: all threads
      kb = km1;
      xb = dec(xb, NB, g.nx);
    }
    // buffer mbarrier phases advanced by this matrix: one completion per block
    __syncthreads();
    if (threadIdx.x < nbuf) {
      int cnt = 0;
      for (int b = threadIdx.x; b < nblk; b += nbuf) ++cnt;
      bphase[threadIdx.x] = (bphase[threadIdx.x] + (unsigned)cnt) & 1u;
    }
    __syncthreads();
  }
};

}  // namespace bcg
