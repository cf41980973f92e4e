// aderdg_sweep_2d_p3.cuh — the fused 2D sweep at p = 3 (BASELINE cfg 1: 27^2 cells).
//
// 729 cells of 16 nodes cannot fill 148 SMs: the sweep is one cell's latency, so the
// kernel spends threads on shortening the dependent chain of a cell instead of on
// throughput.  One CTA of 128 threads per cell:
//   * Picard loop on two warps: thread = (node x, time level t), every component; lane = i1 |
//     (i0 & 1) << 2 | t << 3, warp = i0 >> 1.  Axis-1 derivative from registers: one
//     DMMA.8x8x4 per component (the node's flux in the A fragment, interleaved diff^T in B, the
//     result in the owning lane), issued before the barrier; axis 0 through the flux slab
//     [t][i0][i1][c] (eight 16-byte loads + 16 FMAs); the four slices of a node meet in an
//     exchange buffer (same warp: __syncwarp) for the time contraction.  Row strides 18 and the
//     time stride 148 put the eight lanes of a quarter-warp on eight distinct 16-byte bank
//     groups in every store and load of the loop.
//   * one barrier per Picard iteration: the flux slabs and the vote words alternate
//     between two buffers; the convergence vote of iteration i rides on the barrier that
//     publishes the flux of iteration i + 1, which is also the final flux of the tail when
//     the vote says stop.  The admissibility / lambda / |Q| reductions of the prologue ride
//     on the first of these barriers.
//   * tail in two barriers: fbar by (axis, x, c) threads straight from the last slab;
//     then warps 0-1 do the volume integral and qbar while warps 2-3 evaluate the Rusanov
//     speeds of all 64 space-time trace nodes at once (half-warp = face, redux max);
//     then 128 threads project qbar / fbar onto the four faces and write the records.
//   * every global read of the prologue (time-control words, Q, D, 4d face records) is
//     issued before the first use.
//   * optional fused time control (FusedFinish): the last CTA to arrive runs finish_body,
//     which removes the finish launch from the step (single GPU, fused driver).
// Arithmetic is that of the generic kernel (aderdg_kernels.cuh: operation order, FMA shapes,
// exact-rounded decisions), which this kernel replaces for (Euler, d = 2, p = 3, periodic, fused
// driver), except for the divergence: axis-0 chain + axis-1 DMMA instead of one chain over
// both axes (a rounding-level difference, as in sweep_kernel_p3).
//
// Reference (src/ = /root/reference/pkg/src/aderdg/): kernels.py:68-229, scheduler.py:370-449.
#pragma once
#include "aderdg_kernels.cuh"
#include "aderdg_sweep_p3.cuh"   // dmma_8x8x4

namespace adg {

// tools/cta_timeline.py (A/B build with -DADG_2P3_TIMING): thread 0 of every CTA stamps
// %clock64 at the phase boundaries and %globaltimer at entry / exit into P.sm_scratch
#ifdef ADG_2P3_TIMING
#define ADG_TSTAMP(i)                                                                   \
  do {                                                                                  \
    if (threadIdx.x == 0 && P.sm_scratch != nullptr)                                    \
      P.sm_scratch[(blockIdx.x) * 32 + (i)] = (double)clock64();                        \
  } while (0)
#define ADG_GSTAMP(i)                                                                   \
  do {                                                                                  \
    if (threadIdx.x == 0 && P.sm_scratch != nullptr) {                                  \
      unsigned long long gt_;                                                           \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt_));                           \
      P.sm_scratch[(blockIdx.x) * 32 + (i)] = (double)gt_;                              \
    }                                                                                   \
  } while (0)
#define ADG_PSTAMP(i)                                                                   \
  do {                                                                                  \
    if (threadIdx.x == 0 && P.sm_scratch != nullptr)                                     \
      P.sm_scratch[(blockIdx.x) * 32 + (i)] = (double)clock64();                        \
  } while (0)
#define ADG_BSTAMP(i)                                  \
  do {                                                 \
    if (ts != nullptr) ts[i] = (double)clock64();      \
  } while (0)
#else
#define ADG_TSTAMP(i) ((void)0)
#define ADG_GSTAMP(i) ((void)0)
#define ADG_BSTAMP(i) ((void)0)
#define ADG_PSTAMP(i) ((void)0)
#endif

struct Shape2P3 {
  static constexpr int DIM = 2, M = 4, NQ = 4, NS = 16, NF = 4;
  static constexpr int THREADS = 128, NWARPS = 4, MINB = 5;
  static constexpr int REC = 2 * NF * M + 2;
  static constexpr int PW = 2;                   // Picard warps
  // flux slab [t][axis][i0][i1][c] (doubles): row stride 18 and time stride 148 put the eight
  // lanes of a quarter-warp (4 time levels x 2 rows) on eight distinct 16-byte bank groups in
  // every store and load of the Picard loop
  static constexpr int RS = NQ * M + 2;          // row (i0) stride
  static constexpr int AS = NQ * RS;             // axis stride
  static constexpr int TS = 2 * AS + 4;          // time-level stride
  static constexpr int SLAB = NQ * TS;
  static constexpr int XS = NQ * M + 2;          // exchange buffer [i1][i0][t][c]: i0 stride
  // shared memory (doubles)
  static constexpr int OFF_Q = 0;                        // [x][c]
  static constexpr int OFF_FACE = OFF_Q + NS * M;        // signed F* [f][y][c]
  static constexpr int OFF_SLAB = OFF_FACE + 2 * DIM * NF * M;   // two flux slabs
  // tail buffers, padded like the slab: final q [t][i0][i1][c] with row stride 18 and level
  // stride 76 (16-byte accesses of the Picard and trace threads conflict-free), fbar / qbar
  // [i0][i1][c] with row stride 20 (8-byte face projections along either axis conflict-free)
  static constexpr int QTS = NQ * RS + 4;        // time-level stride of the final q
  static constexpr int BS = NQ * M + 4;          // row stride of fbar / qbar
  static constexpr int OFF_QT = OFF_SLAB + 2 * SLAB;
  static constexpr int OFF_FB = OFF_QT + NQ * QTS;       // fbar [a][i0][i1][c]
  static constexpr int OFF_QBAR = OFF_FB + DIM * NQ * BS;
  static constexpr int OFF_DV = OFF_QBAR + NQ * BS;      // divergence exchange of the Picard loop
  static constexpr int OFF_RED = OFF_DV + NQ * NQ * XS;  // per-warp words, s_max, votes, outcome
  static constexpr int R_RED = 2 * PW + 2 * DIM + 12;
  static constexpr int TOTAL = OFF_RED + R_RED;
  static constexpr size_t SMEM_BYTES = sizeof(double) * TOTAL;
};

// time control fused into the sweep launch: the last CTA to arrive runs finish_body
struct FusedFinish {
  FinishParams F;
  unsigned* arrive;       // zero between launches
  int on;
};

// max of 64-bit patterns over the lanes of `mask` (see warp_max_u64)
__device__ __forceinline__ unsigned long long group_max_u64(unsigned mask, unsigned long long v) {
  const unsigned hi = (unsigned)(v >> 32), lo = (unsigned)v;
  const unsigned mh = __reduce_max_sync(mask, hi);
  const unsigned ml = __reduce_max_sync(mask, hi == mh ? lo : 0u);
  return ((unsigned long long)mh << 32) | ml;
}

// barrier of the two Picard warps (warps 2-3 wait at the CTA barrier behind the loop)
__device__ __forceinline__ void picard_barrier_2p3() {
#ifdef ADG_DEBUG_CHECKS
  unsigned t;
  asm volatile("mov.u32 %0, %%clock;" : "=r"(t));
  unsigned x = t ^ ((threadIdx.x >> 5) * 0x9e3779b9u) ^ (blockIdx.x * 0x85ebca6bu);
  x ^= x >> 13;
  x *= 0xc2b2ae35u;
  x ^= x >> 16;
  if ((x & 3u) == 0u) __nanosleep(x >> 24);
#endif
  asm volatile("bar.sync 1, 64;" ::: "memory");
}

// one pass over the cells: what a sweep launch reads from SweepParams, as values, so that the
// multi-step kernel below can change them from step to step
struct Pass2P3 {
  int mode, sweep;
  const double* tr_in;
  double* tr_out;
};

__device__ __forceinline__ void sweep_2d_p3_body(const SweepParams& P, const Pass2P3& W, const long long cell,
                                                 double* smem) {
  using S = Shape2P3;
  using PDE = EulerPDE<2>;
  constexpr int DIM = 2, M = 4, NQ = 4, NS = 16, NF = 4, REC = S::REC, NW = S::NWARPS;
  constexpr int TS = S::TS, AS = S::AS, RS = S::RS, XS = S::XS, PW = S::PW, QTS = S::QTS, BS = S::BS;
  constexpr unsigned FULL = 0xffffffffu;

  double* sQ = smem + S::OFF_Q;
  double* sFace = smem + S::OFF_FACE;
  double* sSlab = smem + S::OFF_SLAB;
  double* sQt = smem + S::OFF_QT;
  double* sFb = smem + S::OFF_FB;
  double* sQbar = smem + S::OFF_QBAR;
  double* sDv = smem + S::OFF_DV;
  unsigned long long* sWLam = reinterpret_cast<unsigned long long*>(smem + S::OFF_RED);
  unsigned long long* sWAm = sWLam + PW;
  unsigned long long* sSmax = sWAm + PW;                               // [2 * DIM]
  unsigned* sWOk = reinterpret_cast<unsigned*>(sSmax + 2 * DIM);       // [PW]
  unsigned* sVote = sWOk + PW;                                         // [2][PW], then outcome words
  unsigned long long* sTC = reinterpret_cast<unsigned long long*>(smem + S::OFF_RED + S::R_RED - 6);   // 5 words

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  DevState* st = P.st;
  const int mode = W.mode;
  const bool corr = mode_corrects(mode);
  const long long gcell = cell + P.cell_offset;
  const int plane = (int)cell / P.plane_cells;            // (local cells fit 32 bits: 32-bit division)
  const int rest = (int)cell % P.plane_cells;
  const long long own_slot = (long long)(plane + 1) * P.plane_cells + rest;
  double* Qg = P.Q + cell * (NS * M);
  double* Dg = P.D + cell * (NS * M);

  // neighbour slot across face f (periodic, or the halo slot of an x-slab)
  auto nb_of = [&](int f) -> long long {
    const int dir = (f & 1) ? 1 : -1;
    if ((f >> 1) == 0) {
      int pl = plane + dir;
      if (!P.halo) pl = (pl + P.K) % P.K;
      return (long long)(pl + 1) * P.plane_cells + rest;
    }
    const int ia = rest % P.K;
    const int ja = (ia + dir + P.K) % P.K;
    return (long long)(plane + 1) * P.plane_cells + rest + (ja - ia);
  };

  ADG_GSTAMP(0);
  ADG_TSTAMP(1);
  // ---------------- every global read of the prologue, issued before the first use ----------------
  // (L2 loads: in the multi-step kernel other SMs rewrite these words, the neighbours' records
  // and nothing else between two passes of this CTA, and L1 is not coherent.)  The
  // time-control words: thread 0 alone (three 16-byte loads), handed to the CTA through shared
  // memory at the first barrier -- 729 CTAs x 128 threads reading one L2 line is a hot spot.
  ulonglong2 w_red = make_ulonglong2(0ull, 0ull), w_flag = w_red, w_scale = w_red;
  if (tid == 0) {
    static_assert(offsetof(DevState, rerun_next) % 16 == 0 && offsetof(DevState, status) == offsetof(DevState, rerun_next) + 8 &&
                  offsetof(DevState, step) == offsetof(DevState, rerun_next) + 12, "rerun_next | rerun_this | status | step");
    w_red = __ldcg(reinterpret_cast<const ulonglong2*>(&st->reduce[0]));
    w_flag = __ldcg(reinterpret_cast<const ulonglong2*>(&st->rerun_next));
    w_scale = __ldcg(reinterpret_cast<const ulonglong2*>(&st->scale_old));
  }
  const int e = tid & 63;
  double q_in = 0.0, d_in = 0.0;
  double r_qm = 0.0, r_qp = 0.0, r_fm = 0.0, r_fp = 0.0, r_sm = 0.0, r_sp = 0.0;
  if (tid < 64) {
    q_in = __ldcg(Qg + e);
    if (corr) d_in = __ldcg(Dg + e);
  } else if (corr) {
    const int f = e >> 4, yc = e & 15;
    const double* own = W.tr_in + ((long long)f * P.slots + own_slot) * REC;
    const double* nb = W.tr_in + ((long long)(f ^ 1) * P.slots + nb_of(f)) * REC;
    const double* mr = (f & 1) ? own : nb;   // minus side record
    const double* pr = (f & 1) ? nb : own;   // plus side record
    r_sm = __ldcg(mr + 2 * NF * M); r_sp = __ldcg(pr + 2 * NF * M);
    r_qm = __ldcg(mr + yc); r_qp = __ldcg(pr + yc);
    r_fm = __ldcg(mr + NF * M + yc); r_fp = __ldcg(pr + NF * M + yc);
  }
  ADG_TSTAMP(2);   // after issuing the loads
  if (tid == 0) {
    sTC[0] = w_red.y;                                     // reduce[1]: error key of a failed pass
    sTC[1] = w_flag.x;                                    // rerun_next | rerun_this << 32
    sTC[2] = w_flag.y;                                    // status | step << 32
    sTC[3] = w_scale.x;                                   // scale_old (bits)
    sTC[4] = w_scale.y;                                   // scale_new (bits)
  }
  int st_status = 0, st_rerun = 0, st_step = 0;
  double scale_old = 0.0, scale_new = 0.0;
  bool spike = false;
  // after the first CTA barrier of the pass (no global write happens before it)
#define ADG_2P3_TC_WORDS()                                                          \
  do {                                                                              \
    st_rerun = (int)(unsigned)sTC[1];                                               \
    st_status = (int)(unsigned)sTC[2];                                              \
    st_step = (int)(unsigned)(sTC[2] >> 32);                                        \
    scale_old = __longlong_as_double((long long)sTC[3]);                            \
    scale_new = __longlong_as_double((long long)sTC[4]);                            \
    spike = corr && P.spike_step >= 0 && st_step + 1 == P.spike_step;               \
    if (st_status != 0) return;                                                     \
    if (mode == MODE_RERUN && !st_rerun) return;                                    \
    if (corr && sTC[0] != 0ull) return; /* a predict pass already failed */         \
  } while (0)
#ifdef ADG_DEBUG_CHECKS
  if (corr && tid == 0 && (unsigned)w_flag.y == 0u && w_red.y == 0ull) {
    long long nbs[2 * DIM];
    for (int f = 0; f < 2 * DIM; ++f) nbs[f] = nb_of(f);
    debug_check_records_at<DIM>(P, W.tr_in, expected_stamp_of(mode, W.sweep, (int)(unsigned)w_flag.x), st, cell, gcell,
                                own_slot, nbs, REC, 2 * NF * M);
  }
#endif

  ADG_TSTAMP(3);   // time-control words arrived
  if (corr) {
    // ------------- Riemann (kernels.py:147-179), time-collapsed -------------
    if (tid >= 64) {
      const int f = e >> 4;
      const double alpha = rusanov_alpha(r_sm, r_sp);
      // F* = 0.5*(fm+fp) - 0.5*alpha*(qp-qm)   (kernels.py:175)
      const double fs = __dsub_rn(__dmul_rn(0.5, __dadd_rn(r_fm, r_fp)),
                                  __dmul_rn(__dmul_rn(0.5, alpha), __dsub_rn(r_qp, r_qm)));
      sFace[e] = (f & 1) ? fs : -fs;                      // plus side stores -F* (kernels.py:176-177)
    }
    __syncthreads();
    ADG_2P3_TC_WORDS();
    // ------------- integrate_face + update (kernels.py:183-214): thread = (x, c) -------------
    if (tid < 64) {
      const int xx = e >> 2, c = e & 3;
      const int idx[DIM] = {xx >> 2, xx & 3};
      double Dx = d_in;
#pragma unroll
      for (int a = 0; a < DIM; ++a) {
        const int y = idx[1 - a];
        const double slo = __dmul_rn(scale_old, P.ops.lift_lo[idx[a]]);
        const double shi = __dmul_rn(scale_old, P.ops.lift_hi[idx[a]]);
        Dx = __dsub_rn(Dx, __dmul_rn(slo, sFace[((2 * a) * NF + y) * M + c]));
        Dx = __dsub_rn(Dx, __dmul_rn(shi, sFace[((2 * a + 1) * NF + y) * M + c]));
      }
      q_in = __dadd_rn(q_in, Dx);
      if (!spike) Qg[e] = q_in;
    }
  }
  if (tid < 64) sQ[e] = q_in;
  __syncthreads();
  if (!corr) ADG_2P3_TC_WORDS();
#undef ADG_2P3_TC_WORDS
  if (spike) {
    // Driver._apply_spike (scheduler.py:166-178)
    if (tid < NS) {
      double Qx[M];
#pragma unroll
      for (int c = 0; c < M; ++c) Qx[c] = sQ[tid * M + c];
      const double rho = Qx[0];
      const double pr = pressure_exact<DIM>(Qx);
#pragma unroll
      for (int b = 0; b < DIM; ++b) Qx[1 + b] = __dmul_rn(Qx[1 + b], P.spike_factor);
      double jj = __dmul_rn(Qx[1], Qx[1]);
#pragma unroll
      for (int b = 1; b < DIM; ++b) jj = __dadd_rn(jj, __dmul_rn(Qx[1 + b], Qx[1 + b]));
      Qx[M - 1] = __dadd_rn(__ddiv_rn(pr, 0.4), __ddiv_rn(__dmul_rn(0.5, jj), rho));
#pragma unroll
      for (int c = 0; c < M; ++c) sQ[tid * M + c] = Qx[c];
    }
    __syncthreads();
    if (tid < 64) Qg[e] = sQ[e];
  }

  ADG_TSTAMP(4);   // corrector done, Q published
  // ---------------- predictor roles ----------------
  // warps 0-1 run the Picard loop: thread = (node x, time level t), every component; lane = i1 |
  // (i0 & 1) << 2 | t << 3, warp = i0 >> 1.  Warps 2-3 wait at the barrier behind the loop.
  // (Alternating the working pair between the CTAs of an SM, by a per-SM ticket, changed
  // nothing: the loop is bound by the SM's shared-memory wavefronts.)
  // lane = i1 | (i0 & 1) << 2 | t << 3: the axis-1 line of a node sits in lanes & 3, where the
  // DMMA A fragment wants its k index
  const int i1 = lane & 3, i0 = 2 * (warp & 1) + ((lane >> 2) & 1), t = lane >> 3;
  const int x = i0 * NQ + i1;
  unsigned* sOut = sVote + 2 * PW;                        // [0] outcome, [1] iterations, [2] final slab
  if (warp < PW) {
    const int pw = warp;
    double qf[M];                                         // q at (x, t), every component
    {
      const double2 a = *reinterpret_cast<const double2*>(sQ + x * M);
      const double2 b = *reinterpret_cast<const double2*>(sQ + x * M + 2);
      qf[0] = a.x; qf[1] = a.y; qf[2] = b.x; qf[3] = b.y;
    }
    const double Qn[M] = {qf[0], qf[1], qf[2], qf[3]};
    ADG_PSTAMP(5);
    if (mode != MODE_SEED) {
      // ---------------- predictor (kernels.py:68-105) ----------------
      const double scale = (mode == MODE_RERUN) ? scale_old : scale_new;   // dt / h
      constexpr int cap = 2 * NQ;
      double drow0[NQ], ig[NQ];
#pragma unroll
      for (int j = 0; j < NQ; ++j) {
        drow0[j] = P.ops.diff[i0][j];
        ig[j] = P.ops.integ[t][j];
      }
      const int rd0 = t * TS + i1 * M;                    // axis 0: node (j, i1), + RS j
      const int wr = t * TS + i0 * RS + i1 * M;
      const int xo = i0 * (NQ * XS) + i1 * XS;            // this node's slot of the exchange buffer
      // B fragment of the axis-1 derivative: B[k = lane & 3][n = lane >> 2] = diff[n / 2][k], n even
      const double bfrag = ((lane >> 2) & 1) ? 0.0 : P.ops.diff[lane >> 3][lane & 3];
      double tol = 0.0;
      unsigned outcome = 0u;                              // 2: predictor failed (non-finite difference)
      int iters = 0;
      bool conv = false, bad = false;
      int it = 0;
      double F[DIM][M];
      for (;; ++it) {
        ADG_PSTAMP(16 + it);
        PDE::flux(qf, F, P);
        double* slab = sSlab + (it & 1) * S::SLAB;
        // axis 1 from registers: one DMMA per component (the node's flux in A, interleaved
        // diff^T in B, the result in the lane that owns the node); only axis 0 goes through
        // the slab (axis 1 of the final iterate is stored behind the loop, for fbar)
        double d1[M];
#pragma unroll
        for (int c = 0; c < M; ++c) {
          double z;
          dmma_8x8x4(d1[c], z, F[1][c], bfrag, 0.0, 0.0);
        }
        *reinterpret_cast<double2*>(slab + wr) = make_double2(F[0][0], F[0][1]);
        *reinterpret_cast<double2*>(slab + wr + 2) = make_double2(F[0][2], F[0][3]);
        // vote word: bit 0 = every thread converged in the previous iteration, bit 1 = some
        // difference non-finite
        const bool wc = __all_sync(FULL, conv);
        const bool wb = __any_sync(FULL, bad);
        if (lane == 0) sVote[(it & 1) * PW + pw] = (wc ? 1u : 0u) | (wb ? 2u : 0u);
        if (it == 2) ADG_PSTAMP(10);
        picard_barrier_2p3();
        if (it == 2) ADG_PSTAMP(11);
        const unsigned v0 = sVote[(it & 1) * PW], v1 = sVote[(it & 1) * PW + 1];
        if (it > 0) {
          if ((v0 | v1) & 2u) { outcome = 2u; break; }
          if ((v0 & v1 & 1u) || it == cap) break;
        }
        // divergence of the slice at this node: the axis-0 chain from the slab + the axis-1 DMMA
        double dv[M];
#pragma unroll
        for (int c = 0; c < M; ++c) dv[c] = 0.0;
#pragma unroll
        for (int j = 0; j < NQ; ++j) {
          const double2 lo = *reinterpret_cast<const double2*>(slab + rd0 + j * RS);
          const double2 hi = *reinterpret_cast<const double2*>(slab + rd0 + j * RS + 2);
          dv[0] = fma(drow0[j], lo.x, dv[0]); dv[1] = fma(drow0[j], lo.y, dv[1]);
          dv[2] = fma(drow0[j], hi.x, dv[2]); dv[3] = fma(drow0[j], hi.y, dv[3]);
        }
#pragma unroll
        for (int c = 0; c < M; ++c) dv[c] += d1[c];
        if (it == 2) ADG_PSTAMP(12);
        // time contraction: the four slices of a node are in four lanes of one warp; they
        // meet in the node's slot of the exchange buffer (written before, read after a
        // __syncwarp; the next write comes behind the next Picard barrier)
        *reinterpret_cast<double2*>(sDv + xo + t * M) = make_double2(dv[0], dv[1]);
        *reinterpret_cast<double2*>(sDv + xo + t * M + 2) = make_double2(dv[2], dv[3]);
        __syncwarp();
        double acc[M];
#pragma unroll
        for (int c = 0; c < M; ++c) acc[c] = 0.0;
#pragma unroll
        for (int k = 0; k < NQ; ++k) {
          const double2 lo = *reinterpret_cast<const double2*>(sDv + xo + k * M);
          const double2 hi = *reinterpret_cast<const double2*>(sDv + xo + k * M + 2);
          acc[0] = fma(ig[k], lo.x, acc[0]); acc[1] = fma(ig[k], lo.y, acc[1]);
          acc[2] = fma(ig[k], hi.x, acc[2]); acc[3] = fma(ig[k], hi.y, acc[3]);
        }
        BitMax bm;
#pragma unroll
        for (int c = 0; c < M; ++c) {
          const double qn = Qn[c] - scale * acc[c];
          bm.add(fabs(qn - qf[c]));
          qf[c] = qn;
        }
        if (it == 0) {
          // warp 2's max |Q| is first needed here (its admissibility / lambda words follow at
          // the barrier behind the loop: the loop itself lets nothing out of the CTA)
          asm volatile("bar.sync 2, 96;" ::: "memory");
          tol = 1e-10 * (1.0 + __longlong_as_double((long long)sWAm[0]));
        }
        conv = bm.conv(tol);
        bad = bm.bad();
        if (it == 2) ADG_PSTAMP(31);
      }
      iters = it;
      // the slab of the last barrier holds the flux of the final iterate at every (t, axis, x, c)
      if (outcome == 0u) {
        double* slab = sSlab + (it & 1) * S::SLAB + AS;
        *reinterpret_cast<double2*>(slab + wr) = make_double2(F[1][0], F[1][1]);
        *reinterpret_cast<double2*>(slab + wr + 2) = make_double2(F[1][2], F[1][3]);
        *reinterpret_cast<double2*>(sQt + t * QTS + i0 * RS + i1 * M) = make_double2(qf[0], qf[1]);
        *reinterpret_cast<double2*>(sQt + t * QTS + i0 * RS + i1 * M + 2) = make_double2(qf[2], qf[3]);
      }
      if (tid == 0) {
        sOut[0] = outcome;
        sOut[1] = (unsigned)iters;
        sOut[2] = (unsigned)(it & 1);
      }
    }
  } else if (warp == PW) {
    // warp 2, idle during the Picard loop, lane = node: max |Q| for the Picard tolerance (the
    // Picard warps pick it up at the end of their first iteration, barrier 2), then
    // calc_time_step (kernels.py:216-229) / predict's finiteness check (kernels.py:80-81),
    // three exact divisions and a root per node, read behind the loop.
    double qn[M] = {0.0, 0.0, 0.0, 0.0};
    if (lane < NS) {
      const double2 a = *reinterpret_cast<const double2*>(sQ + lane * M);
      const double2 b = *reinterpret_cast<const double2*>(sQ + lane * M + 2);
      qn[0] = a.x; qn[1] = a.y; qn[2] = b.x; qn[3] = b.y;
    }
    double am = 0.0;
#pragma unroll
    for (int c = 0; c < M; ++c) am = fmax(am, fabs(qn[c]));
    const unsigned long long wa = warp_max_u64((unsigned long long)__double_as_longlong(am));
    if (lane == 0) sWAm[0] = wa;
    if (mode != MODE_SEED) {
      __threadfence_block();
      asm volatile("bar.arrive 2, 96;" ::: "memory");
    }
    bool ok = true;
    double lam = 0.0;
    if (lane < NS) {
      if (!mode_predict_only(mode)) {
        ok = PDE::node_lambda(qn, lam, P);
      } else {
#pragma unroll
        for (int c = 0; c < M; ++c) ok = ok && finite(qn[c]);
      }
    }
    const bool wok = __all_sync(FULL, ok);
    const unsigned long long wl = warp_max_u64((unsigned long long)__double_as_longlong(ok ? lam : 0.0));
    if (lane == 0) {
      sWOk[0] = wok ? 1u : 0u;
      sWLam[0] = wl;
    }
  }
  __syncthreads();
  if (mode == MODE_SEED) {
    if (tid == 0) {
      if (!sWOk[0]) report_error(st, 2 * gcell + 0);
      else atomicMax(&st->reduce[0], (long long)sWLam[0]);
    }
    return;
  }
  ADG_TSTAMP(6);   // Picard loop done
  // calc_time_step comes before predict (scheduler.py:370-449): its verdict first
  if (!sWOk[0]) {
    if (tid == 0) report_error(st, 2 * gcell + (mode_predict_only(mode) ? 1 : 0));
    return;
  }
  if (sOut[0] != 0u) {
    if (tid == 0) report_error(st, 2 * gcell + 1);
    return;
  }
  if (!mode_predict_only(mode) && tid == 0) atomicMax(&st->reduce[0], (long long)sWLam[0]);
  const double scale = (mode == MODE_RERUN) ? scale_old : scale_new;
  const double* cur = sSlab + sOut[2] * S::SLAB;
  const int iters = (int)sOut[1];

  // ---------------- tail: fbar, volume integral, traces ----------------
  {
    // fbar[a][x][c] = sum_k w_k F_k (integrate_volume, kernels.py:130-143): thread = (a, x, c)
    const int a = tid >> 6;
    const int so = (e >> 4) * RS + (e & 15);              // (x, c) in the slab's padded node rows
    double fb = 0.0;
    bool badf = false;                                    // predict's check of the final flux (kernels.py:99-101)
#pragma unroll
    for (int k = 0; k < NQ; ++k) {
      const double Fk = cur[k * TS + a * AS + so];
      badf |= !finite(Fk);
      fb = fma(P.ops.w[k], Fk, fb);
    }
    sFb[a * (NQ * BS) + (e >> 4) * BS + (e & 15)] = fb;
    if (__syncthreads_or(badf)) {
      if (tid == 0) report_error(st, 2 * gcell + 1);
      return;
    }
  }
  if (tid == 0) {
    atomicAdd((unsigned long long*)&st->picard_iters, (unsigned long long)iters);
    atomicAdd((unsigned long long*)&st->predicts, 1ull);
    atomicAdd((unsigned long long*)&st->hist[iters < HIST_BINS ? iters : HIST_BINS - 1], 1ull);
  }
  ADG_TSTAMP(7);   // fbar published
  if (tid < 64) {
    // volume integral, thread = (x, c); then qbar = sum_t w_t q
    const int xx = e >> 2, c = e & 3;
    const int j0 = xx >> 2, j1 = xx & 3;
    double s = 0.0;
#pragma unroll
    for (int j = 0; j < NQ; ++j) s = fma(P.ops.kvol[j0][j], sFb[j * BS + j1 * M + c], s);
#pragma unroll
    for (int j = 0; j < NQ; ++j) s = fma(P.ops.kvol[j1][j], sFb[NQ * BS + j0 * BS + j * M + c], s);
    Dg[e] = s * scale;
    double v = 0.0;
#pragma unroll
    for (int k = 0; k < NQ; ++k) v = fma(P.ops.w[k], sQt[k * QTS + j0 * RS + (e & 15)], v);
    sQbar[j0 * BS + (e & 15)] = v;
  } else {
    // s_max over the space-time trace of q, per face (Rusanov alpha input, kernels.py:107-128):
    // thread = (face f, face node y, time level): half-warp = face
    const int f = e >> 4, y = (e >> 2) & 3, tt = e & 3, a = f >> 1;
    const double* vec = (f & 1) ? P.ops.right : P.ops.left;
    // trace line of face node y: nodes (i, y) across axis 0, (y, i) across axis 1
    const int xb = (a == 0) ? y * M : y * RS, sta = (a == 0) ? RS : M;
    // axis 0: the eight lanes of a quarter-warp (4 levels x 2 face nodes) sit on even 16-byte
    // groups only; odd face nodes fetch their upper component pair first
    const int sw = (a == 0 && (y & 1)) ? 2 : 0;
    double qs[M];
#pragma unroll
    for (int c = 0; c < M; ++c) qs[c] = 0.0;
#pragma unroll
    for (int i = 0; i < NQ; ++i) {
      const double vi = vec[i];
      const double* src = sQt + tt * QTS + xb + i * sta;
      const double2 u = *reinterpret_cast<const double2*>(src + sw);
      const double2 v = *reinterpret_cast<const double2*>(src + (sw ^ 2));
      const double2 lo = sw ? v : u, hi = sw ? u : v;
      qs[0] = fma(vi, lo.x, qs[0]); qs[1] = fma(vi, lo.y, qs[1]);
      qs[2] = fma(vi, hi.x, qs[2]); qs[3] = fma(vi, hi.y, qs[3]);
    }
    // PDE::trace_speed(qs, a) with the axis' momentum selected by value (no indexed array)
    const double pr = pressure_exact<DIM>(qs);
    const double qa[2] = {qs[0], a ? qs[2] : qs[1]};
    const double sp = speed_exact<DIM>(qa, 0, pr);
    const unsigned half = (lane & 16) ? 0xffff0000u : 0x0000ffffu;
    const unsigned long long m = group_max_u64(half, (unsigned long long)__double_as_longlong(sp));
    if ((lane & 15) == 0) sSmax[f] = m;
  }
  __syncthreads();
  ADG_TSTAMP(8);   // D stored, qbar / s_max published
  {
    // face records: threads 0-63 project qbar, threads 64-127 project fbar; item = (f, y, c)
    const int f = e >> 4, yc = e & 15, y = yc >> 2, c = yc & 3, a = f >> 1;
    const double* vec = (f & 1) ? P.ops.right : P.ops.left;
    const int xb = (a == 0) ? y * M : y * BS, sta = (a == 0) ? BS : M;
    const double* src = (tid < 64) ? sQbar : sFb + a * (NQ * BS);
    double v = 0.0;
#pragma unroll
    for (int i = 0; i < NQ; ++i) v = fma(vec[i], src[xb + i * sta + c], v);
    double* rec = W.tr_out + ((long long)f * P.slots + own_slot) * REC;
    rec[(tid < 64 ? 0 : NF * M) + yc] = v;
  }
  if (tid < 2 * DIM) {
    double* rec = W.tr_out + ((long long)tid * P.slots + own_slot) * REC;
    rec[2 * NF * M] = __longlong_as_double((long long)sSmax[tid]);
    rec[2 * NF * M + 1] = record_stamp_of(mode, W.sweep);
  }
  ADG_TSTAMP(9);     // records issued
#ifdef ADG_2P3_TIMING
  if (tid == 0 && P.sm_scratch != nullptr) P.sm_scratch[blockIdx.x * 32 + 13] = (double)iters;
#else
  (void)iters;
#endif
}

__global__ void __launch_bounds__(Shape2P3::THREADS, Shape2P3::MINB)
sweep_kernel_2d_p3(const SweepParams P, const FusedFinish X) {
  extern __shared__ __align__(16) double smem[];
  ADG_DEBUG_POISON();
  const Pass2P3 W{P.mode, P.sweep, P.tr_in, P.tr_out};
  sweep_2d_p3_body(P, W, sweep_cell(P), smem);
  if (X.on) {
    // the last CTA to arrive has every CTA's reductions behind its fence: it is the time control
    __syncthreads();
    if (threadIdx.x == 0) {
      ADG_TSTAMP(10);
      __threadfence();
      ADG_TSTAMP(11);
      const unsigned n = atomicAdd(X.arrive, 1u);
#ifdef ADG_2P3_TIMING
      if (P.sm_scratch != nullptr) P.sm_scratch[blockIdx.x * 32 + 14] = (double)n;
#endif
      ADG_TSTAMP(12);
      if (n == gridDim.x - 1) {
        __threadfence();
        *X.arrive = 0u;
        const unsigned fl = finish_body(X.F);
        if (X.F.has_cond) cudaGraphSetConditional(X.F.cond, (fl & FINISH_RERUN) ? 1u : 0u);
      }
    }
  }
  ADG_GSTAMP(15);
}

// ---------------------------------------------------------------------------
// Multi-step launch: `steps` realisation steps of the fused driver (scheduler.py:190-226:
// rerun pass when the time control asked for one, sweep, time control) in ONE cooperative
// kernel.  At 729 cells a step's launches cost as much as its arithmetic; here the steps are
// separated by a grid barrier (arrival counter + generation word) whose last arriver runs the
// time control before it releases the others.  CTA b owns the cells b, b + grid, ... in every
// pass; what other CTAs write between two passes (neighbour records, DevState) is read
// through L2.  Results are bitwise those of the per-step launches.
struct RunParams2P3 {
  FinishParams F;
  unsigned* sync;           // [0] arrival counter (zero between barriers), [1] generation
  double* tr[2];            // the two record parities
  int steps;
};

// The release word is generation | flags: the last arriver's `last()` returns the flags
// (GB_RERUN: the time control asked for a rerun pass, GB_STOP: the run has a status / a pass
// failed), every CTA gets them back without another trip to DevState.
constexpr unsigned GB_RERUN = FINISH_RERUN, GB_STOP = FINISH_STOP, GB_GEN = GB_RERUN - 1u;

template <class LastFn>
__device__ __forceinline__ unsigned grid_barrier_2p3(unsigned* sync, unsigned& gen, unsigned* sflags, LastFn last,
                                                     double* ts = nullptr) {
  (void)ts;
  __syncthreads();
  if (threadIdx.x == 0) {
    ADG_BSTAMP(26);
    __threadfence();
    ADG_BSTAMP(27);
    const unsigned n = atomicAdd(&sync[0], 1u);
    ADG_BSTAMP(28);
    if (n == gridDim.x - 1) {
      __threadfence();
      sync[0] = 0u;
      const unsigned fl = last();
      ADG_BSTAMP(29);
      __threadfence();
      atomicExch(&sync[1], ((gen + 1u) & GB_GEN) | fl);      // release
      *sflags = fl;
      ADG_BSTAMP(30);
    } else {
      // acquire loads: what the CTA reads after the barrier is ordered behind the release
      unsigned g;
      do {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(&sync[1]) : "memory");
      } while ((g & GB_GEN) == gen);
      *sflags = g & ~GB_GEN;
      ADG_BSTAMP(29);
      ADG_BSTAMP(30);
    }
#ifdef ADG_2P3_TIMING
    if (ts != nullptr) {
      ts[14] = (double)n;
      unsigned long long gt_;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt_));
      ts[15] = (double)gt_;
    }
#endif
  }
  gen = (gen + 1u) & GB_GEN;
  __syncthreads();
  return *sflags;
}

__global__ void __launch_bounds__(Shape2P3::THREADS, Shape2P3::MINB)
run_kernel_2d_p3(const SweepParams P, const RunParams2P3 R) {
  extern __shared__ __align__(16) double smem[];
  __shared__ unsigned s_flags;
  ADG_DEBUG_POISON();
  const long long cells = (long long)P.planes_local * P.plane_cells;
  // every CTA reads the generation before any barrier of this launch can complete
  unsigned gen = *reinterpret_cast<volatile unsigned*>(&R.sync[1]) & GB_GEN;
  if (threadIdx.x == 0) {                                     // the state the launch starts from
    const ulonglong2 w = __ldcg(reinterpret_cast<const ulonglong2*>(&P.st->rerun_next));
    s_flags = ((unsigned)w.x ? GB_RERUN : 0u) | ((unsigned)w.y ? GB_STOP : 0u);
  }
  __syncthreads();
  unsigned flags = s_flags;
#ifdef ADG_DEBUG_CHECKS
  const long long first = (long long)(gridDim.x - 1 - blockIdx.x);   // reversed cell order (sweep_cell)
#else
  const long long first = (long long)blockIdx.x;
#endif
#ifdef ADG_2P3_TIMING
  double* ts = P.sm_scratch ? P.sm_scratch + blockIdx.x * 32 : nullptr;
#else
  double* ts = nullptr;
#endif
  for (int s = 0; s < R.steps; ++s) {
    if (flags & GB_STOP) break;                                // uniform: the release word of the last barrier
    const int sweep = P.sweep + s;
    const double* tr_in = R.tr[sweep & 1];
    bool skip = false;
    if (flags & GB_RERUN) {                                    // _maybe_rerun (scheduler.py:446-449)
      const Pass2P3 W{MODE_RERUN, sweep, tr_in, R.tr[sweep & 1]};
      for (long long cell = first; cell < cells; cell += gridDim.x) {
        sweep_2d_p3_body(P, W, cell, smem);
        __syncthreads();
      }
      // a failed predict of the rerun pass (error key in reduce[1]) cancels the sweep
      skip = (grid_barrier_2p3(R.sync, gen, &s_flags, [&]() -> unsigned {
                return __ldcg(&P.st->reduce[1]) != 0 ? GB_STOP : 0u;
              }) & GB_STOP) != 0u;
    }
    if (!skip) {
      const Pass2P3 W{MODE_NORMAL, sweep, tr_in, R.tr[(sweep & 1) ^ 1]};
      for (long long cell = first; cell < cells; cell += gridDim.x) {
        sweep_2d_p3_body(P, W, cell, smem);
        __syncthreads();
      }
    }
    flags = grid_barrier_2p3(R.sync, gen, &s_flags, [&]() -> unsigned { return finish_body(R.F); }, ts);
  }
}

}  // namespace adg
