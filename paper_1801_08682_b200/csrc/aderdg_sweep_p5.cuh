// aderdg_sweep_p5.cuh — the fused 3D sweep at p = 5 with the Picard derivatives
// on the FP64 tensor cores.
//
// One CTA per cell, 224 threads (7 warps; thread = spatial node in the p = 5 warp
// blocks of block_map_p5), two CTAs per SM (<= 144 registers, 104 KB of shared
// memory).  The per-node time line q[t][c] and the Picard accumulator acc[t][c]
// stay in registers, so the time contraction (integ) is register-local DFMA work.
// The spatial derivatives of a time slice are three small GEMMs per slice,
//
//     Out_a[i][col] = sum_j diff[i][j] F_a[j][col],   col = c*36 + (other two indices)
//
// (180 columns + 4 zero pad columns = 23 n-tiles of 8), issued as DMMA m8n8k4 with
// diff as the A operand (two constant fragments per lane: k = 0..3 and 4..5, rows
// and columns 6..7 zero) and the flux as the B operand straight from shared memory;
// each tile writes its 6 useful output rows back in place over its own columns
// (a tile's outputs depend only on its own columns), and the node owner sums the
// three axes.  Per slice: flux -> 15 owner stores -> barrier -> 69 tiles over the 7
// warps -> barrier -> 15 owner loads + 30 FMAs of the time contraction; the operand
// arrays are double-buffered by slice parity, so two barriers per slice.
//
// The rest (TMA bulk staging of Q, D and the 4d face records, Riemann, corrector,
// calc_time_step, final flux, volume integral, face traces, s_max) follows
// sweep_kernel_v2 with the node layout in C order.
//
// Row stride STR = 196 == 4 (mod 16): a B-fragment load (4 rows x 8 columns) hits 32
// distinct bank pairs per half-warp pair (two wavefronts, the minimum); the owner
// stores / loads of the warp blocks cost 2.4 wavefronts per instruction (model,
// tools/p5_banks.py).
//
// Reference (src/ = /root/reference/pkg/src/aderdg/): kernels.py:68-229 (predict,
// extrapolate, integrate_volume, solve_riemann, integrate_face, update,
// calc_time_step), scheduler.py:370-449 (fused sweep).
#pragma once
#include "aderdg_sweep_ho.cuh"   // TMEM helpers (and the v2 TMA / DMMA helpers)

namespace adg {

// D = A(8x4) * B(4x8) + C (fp64) without the volatile qualifier: a pure register
// operation the compiler may schedule across the independent tiles
__device__ __forceinline__ void dmma_nv(double& d0, double& d1, double a, double b, double c0, double c1) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};\n"
      : "=d"(d0), "=d"(d1)
      : "d"(a), "d"(b), "d"(c0), "d"(c1));
}

template <int COLS>
__device__ __forceinline__ void tmem_alloc_cols(uint32_t* dst) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n"
               "tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::"r"(smem_u32(dst)), "n"(COLS)
               : "memory");
}
template <int COLS>
__device__ __forceinline__ void tmem_dealloc_cols(uint32_t t) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(t), "n"(COLS) : "memory");
}

struct ShapeP5 {
  static constexpr int DIM = 3, M = 5, NQ = 6;
  static constexpr int NS = 216, NF = 36;
  static constexpr int THREADS = 224, NW = 7;
  static constexpr int REC = 2 * NF * M + 2;
  // DMMA operand arrays [slice parity][axis][j][STR]
  static constexpr int NCOL = 180, NTILE = 23, STR = 196;
  static constexpr int ABUF = NQ * STR;
  static constexpr int FBUF = DIM * ABUF;
  static constexpr int TILES = DIM * NTILE;
  static constexpr int R_PRED = 2 * FBUF;
  // after the Picard loop: q of every time level [t][c][NS] | qbar [c][NS] | fbar [a][c][NS]
  static constexpr int R_QT = NQ * M * NS, R_QB = M * NS, R_FB = DIM * M * NS;
  static constexpr int R_POST = R_QT + R_QB + R_FB;
  // corrector: staged records (own 2d | neighbour 2d) + signed F* per face
  static constexpr int R_REC = 4 * DIM * REC, R_FACE = 2 * DIM * NF * M;
  static constexpr int R_CORR = R_REC + R_FACE;
  static constexpr int R_U = (R_PRED > R_POST ? (R_PRED > R_CORR ? R_PRED : R_CORR)
                                               : (R_POST > R_CORR ? R_POST : R_CORR));
  static constexpr int R_RED = 3 * NW + 2 * DIM + 4;
  static constexpr int OFF_BAR = 0;
  static constexpr int OFF_RED = 2;
  static constexpr int OFF_Q = OFF_RED + ((R_RED + 1) & ~1);
  static constexpr int OFF_D = OFF_Q + NS * M;
  static constexpr int OFF_U = OFF_D + NS * M;
  static constexpr int TOTAL = OFF_U + R_U;
  static constexpr size_t SMEM_BYTES = sizeof(double) * TOTAL;
  static_assert(SMEM_BYTES <= 112 * 1024, "two CTAs per SM");
  static_assert(STR >= NTILE * 8 && STR % 16 == 4, "B-fragment bank layout");
};

__global__ void __maxnreg__(144) sweep_kernel_p5(const SweepParams P) {
  using S = ShapeP5;
  constexpr int DIM = 3, M = 5, NQ = 6, NS = S::NS, NF = S::NF, REC = S::REC, NW = S::NW;
  constexpr int THREADS = S::THREADS, STR = S::STR, ABUF = S::ABUF, FBUF = S::FBUF;

  extern __shared__ __align__(16) double smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + S::OFF_BAR);
  double* sRed = smem + S::OFF_RED;
  unsigned long long* sSmax = reinterpret_cast<unsigned long long*>(sRed + 2 * NW);
  unsigned* sFlags = reinterpret_cast<unsigned*>(sRed + 2 * NW + 2 * DIM);
  double* sQ = smem + S::OFF_Q;
  double* sD = smem + S::OFF_D;
  double* sU = smem + S::OFF_U;
  double* sRec = sU;                       // corrector
  double* sFace = sU + S::R_REC;
  double* sQt = sU;                        // after the Picard loop
  double* sQb = sU + S::R_QT;
  double* sFb = sQb + S::R_QB;
  ADG_DEBUG_POISON();

  DevState* st = P.st;
  if (st->status != 0) return;
  const int mode = P.mode;
  if (mode == MODE_RERUN && !st->rerun_next) return;
  if (mode_corrects(mode) && st->reduce[1] != 0) return;   // a predict pass already failed

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int i0, i1, i2;
  bool act;
  block_map_p5(tid, i0, i1, i2, act);
  const int x = (i0 * NQ + i1) * NQ + i2;
  const long long cell = sweep_cell(P);
  const long long gcell = cell + P.cell_offset;
  const int plane = (int)(cell / P.plane_cells);
  const int rest = (int)(cell % P.plane_cells);
  const long long own_slot = (long long)(plane + 1) * P.plane_cells + rest;
  const int step_idx = mode_corrects(mode) ? st->step + 1 : 0;
  double* Qg = P.Q + cell * (NS * M);
  double* Dg = P.D + cell * (NS * M);

  // ---------------- TMA bulk staging of Q (+ D and the 4d face records) ----------------
  if (tid == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (tid == 0) {
    uint32_t bytes = NS * M * 8;
    if (mode_corrects(mode)) bytes += NS * M * 8 + 4 * DIM * REC * 8;
    mbar_arrive_expect_tx(bar, bytes);
    bulk_g2s(sQ, Qg, NS * M * 8, bar);
    if (mode_corrects(mode)) {
      bulk_g2s(sD, Dg, NS * M * 8, bar);
      long long nbs[2 * DIM];
      for (int f = 0; f < 2 * DIM; ++f) {
        const int a = f >> 1;
        const int dir = (f & 1) ? 1 : -1;
        long long nb;
        if (a == 0) {
          int pl = plane + dir;
          if (!P.halo) pl = (pl + P.K) % P.K;
          nb = (long long)(pl + 1) * P.plane_cells + rest;
        } else {
          const int st_a = (a == 1) ? P.K : 1;
          const int ia = (rest / st_a) % P.K;
          const int ja = (ia + dir + P.K) % P.K;
          nb = (long long)(plane + 1) * P.plane_cells + rest + (ja - ia) * st_a;
        }
        bulk_g2s(sRec + f * REC, P.tr_in + ((long long)f * P.slots + own_slot) * REC, REC * 8, bar);
        bulk_g2s(sRec + (2 * DIM + f) * REC, P.tr_in + ((long long)(f ^ 1) * P.slots + nb) * REC, REC * 8,
                 bar);
        nbs[f] = nb;
      }
      debug_check_records<DIM>(P, st, cell, gcell, own_slot, nbs, REC, 2 * NF * M);
    }
  }
  // DMMA A fragments (diff, rows / k >= 6 zero): lane = (row << 2) | k
  const int fr = lane >> 2, fk = lane & 3;
  const double a_lo = (fr < NQ) ? P.ops.diff[fr][fk] : 0.0;
  const double a_hi = (fr < NQ && fk < 2) ? P.ops.diff[fr][fk + 4] : 0.0;
  // owner offsets into one slice buffer: axis a, row i_a, column (other two indices)
  const int own0 = 0 * ABUF + i0 * STR + i1 * NQ + i2;
  const int own1 = 1 * ABUF + i1 * STR + i0 * NQ + i2;
  const int own2 = 2 * ABUF + i2 * STR + i0 * NQ + i1;

  mbar_wait(bar, 0);

  double Qx[M];
#pragma unroll
  for (int c = 0; c < M; ++c) Qx[c] = sQ[x * M + c];

  if (mode_corrects(mode)) {
    // ------------- Riemann (kernels.py:147-179), time-collapsed -------------
    for (int e = tid; e < 2 * DIM * NF * M; e += THREADS) {
      const int f = e / (NF * M);
      const int yc = e % (NF * M);
      const double* own = sRec + f * REC;
      const double* nb = sRec + (2 * DIM + f) * REC;
      const double* mr = (f & 1) ? own : nb;
      const double* pr = (f & 1) ? nb : own;
      const double alpha = rusanov_alpha(mr[2 * NF * M], pr[2 * NF * M]);
      const double fs = __dsub_rn(__dmul_rn(0.5, __dadd_rn(mr[NF * M + yc], pr[NF * M + yc])),
                                  __dmul_rn(__dmul_rn(0.5, alpha), __dsub_rn(pr[yc], mr[yc])));
      sFace[e] = (f & 1) ? fs : -fs;
    }
    __syncthreads();
    // ------------- integrate_face + update (kernels.py:183-214) -------------
    if (act) {
      double Dx[M];
#pragma unroll
      for (int c = 0; c < M; ++c) Dx[c] = sD[x * M + c];
      const double scale_old = (mode == MODE_SF_CORRECT) ? st->scale_new : st->scale_old;
      const int idx[3] = {i0, i1, i2};
#pragma unroll
      for (int a = 0; a < DIM; ++a) {
        const int y = (a == 0) ? i1 * NQ + i2 : (a == 1) ? i0 * NQ + i2 : i0 * NQ + i1;
        const double slo = __dmul_rn(scale_old, P.ops.lift_lo[idx[a]]);
        const double shi = __dmul_rn(scale_old, P.ops.lift_hi[idx[a]]);
#pragma unroll
        for (int c = 0; c < M; ++c) {
          Dx[c] = __dsub_rn(Dx[c], __dmul_rn(slo, sFace[((2 * a) * NF + y) * M + c]));
          Dx[c] = __dsub_rn(Dx[c], __dmul_rn(shi, sFace[((2 * a + 1) * NF + y) * M + c]));
        }
      }
#pragma unroll
      for (int c = 0; c < M; ++c) Qx[c] = __dadd_rn(Qx[c], Dx[c]);
      if (P.spike_step >= 0 && step_idx == P.spike_step) {
        const double rho = Qx[0];
        const double pr = pressure_exact<DIM>(Qx);
#pragma unroll
        for (int b = 0; b < DIM; ++b) Qx[1 + b] = __dmul_rn(Qx[1 + b], P.spike_factor);
        double jj = __dmul_rn(Qx[1], Qx[1]);
#pragma unroll
        for (int b = 1; b < DIM; ++b) jj = __dadd_rn(jj, __dmul_rn(Qx[1 + b], Qx[1 + b]));
        Qx[M - 1] = __dadd_rn(__ddiv_rn(pr, 0.4), __ddiv_rn(__dmul_rn(0.5, jj), rho));
      }
#pragma unroll
      for (int c = 0; c < M; ++c) sQ[x * M + c] = Qx[c];
      fence_proxy_async();
    }
    __syncthreads();
    if (tid == 0) bulk_s2g(Qg, sQ, NS * M * 8);   // committed with the D store below
  }

  if (!mode_predict_only(mode)) {
    // ------------- calc_time_step (kernels.py:216-229) -------------
    bool ok = true;
    double lam = 0.0;
    if (act) {
#pragma unroll
      for (int c = 0; c < M; ++c) ok = ok && finite(Qx[c]);
      bool adm = false;
      lam = max_speed_fast<DIM>(Qx, 0, DIM, adm);
      ok = ok && adm;
      if (!ok) lam = 0.0;
    }
    if (!__syncthreads_and(ok)) {
      if (tid == 0) {
        report_error(st, 2 * gcell + 0);
        if (mode_corrects(mode)) bulk_commit_wait();
      }
      return;
    }
    lam = block_max<NW>(lam, sRed);
    if (tid == 0) atomicMax(&st->reduce[0], __double_as_longlong(lam));
    if (mode == MODE_SEED) return;
    if (mode == MODE_SF_CORRECT) {                       // straightforward: no predictor in this pass
      if (tid == 0) bulk_commit_wait_if_any();
      return;
    }
  } else {
    bool ok = true;
    if (act) {
#pragma unroll
      for (int c = 0; c < M; ++c) ok = ok && finite(Qx[c]);
    }
    if (!__syncthreads_and(ok)) {
      if (tid == 0) report_error(st, 2 * gcell + 1);
      return;
    }
  }

  // ---------------- predictor (kernels.py:68-105) ----------------
  const double scale = (mode == MODE_RERUN) ? st->scale_old : st->scale_new;   // dt / h (SF: dt_new)
  // the 4 pad columns (180..183) of every operand row are read by the last n-tile: zero
  for (int e = tid; e < 2 * DIM * NQ * 4; e += THREADS) sU[(e >> 2) * STR + S::NCOL + (e & 3)] = 0.0;
  // Per-thread time line in tensor memory: 256 columns per CTA (two CTAs per SM fill
  // the 512), warp w on lanes 32*(w%4) and columns (w/4)*128.. : q[t][c] at column
  // 2(5t+c), the slice divergences dv[k][c] at 64 + 2(5k+c)
  __shared__ uint32_t s_tmem;
  if (warp == 0) tmem_alloc_cols<256>(&s_tmem);
  tmem_fence_before();
  double absmax;
  {
    double am = 0.0;
#pragma unroll
    for (int c = 0; c < M; ++c) am = fmax(am, fabs(Qx[c]));
    absmax = block_max<NW>(act ? am : 0.0, sRed);       // (its barriers publish the pad zeros
  }                                                     //  and the TMEM address)
  tmem_fence_after();
  const uint32_t tq = s_tmem + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * 128);
  const uint32_t td = tq + 64;
  const double tol = 1e-10 * (1.0 + absmax);
  const int cap = 2 * NQ;

#pragma unroll
  for (int t = 0; t < NQ; ++t)
#pragma unroll
    for (int c = 0; c < M; ++c) tmem_st_d(tq + 2 * (M * t + c), Qx[c]);
  tmem_wait_st();

  int iters = 0;
  bool failed = false;
#pragma unroll 1
  for (int it = 0; it < cap; ++it) {
#pragma unroll
    for (int k = 0; k < NQ; ++k) {
      double* B = sU + (k & 1) * FBUF;
      {
        double qk[M], F[DIM][M];
        tmem_ld_doubles<M>(tq + 2 * M * k, 2, qk);
        flux<DIM>(qk, F);
        if (act) {
#pragma unroll
          for (int c = 0; c < M; ++c) {
            B[own0 + c * 36] = F[0][c];
            B[own1 + c * 36] = F[1][c];
            B[own2 + c * 36] = F[2][c];
          }
        }
      }
      __syncthreads();
      // Out_a = diff . F_a on the tensor cores, in place, tile by tile
#pragma unroll 2
      for (int tile = warp; tile < S::TILES; tile += NW) {
        const int a = tile >= 2 * S::NTILE ? 2 : (tile >= S::NTILE ? 1 : 0);
        double* base = B + a * ABUF + (tile - a * S::NTILE) * 8;
        const double b0 = base[fk * STR + fr];
        const double b1 = (fk < 2) ? base[(fk + 4) * STR + fr] : 0.0;
        double d0, d1;
        dmma_nv(d0, d1, a_lo, b0, 0.0, 0.0);
        dmma_nv(d0, d1, a_hi, b1, d0, d1);
        if (lane < 4 * NQ) *reinterpret_cast<double2*>(base + fr * STR + 2 * fk) = make_double2(d0, d1);
      }
      __syncthreads();
      // the node's divergence of slice k (idle lanes read a real node's sums and discard them)
#pragma unroll
      for (int c = 0; c < M; ++c)
        tmem_st_d(td + 2 * (M * k + c), (B[own0 + c * 36] + B[own1 + c * 36]) + B[own2 + c * 36]);
    }
    tmem_wait_st();
    // time contraction of the divergence history + Picard update (kernels.py:86-97);
    // convergence from the bit patterns of |q_new - q|
    double dvh[NQ * M];
    tmem_ld_doubles<NQ * M>(td, 2, dvh);
    BitMax bm;
#pragma unroll
    for (int t = 0; t < NQ; ++t) {
      double qo[M];
      tmem_ld_doubles<M>(tq + 2 * M * t, 2, qo);
#pragma unroll
      for (int c = 0; c < M; ++c) {
        double acc = P.ops.integ[t][0] * dvh[c];
#pragma unroll
        for (int k = 1; k < NQ; ++k) acc = fma(P.ops.integ[t][k], dvh[M * k + c], acc);
        const double qn = sQ[x * M + c] - scale * acc;
        bm.add(fabs(qn - qo[c]));
        tmem_st_d(tq + 2 * (M * t + c), qn);
      }
    }
    tmem_wait_st();
    iters = it + 1;
    const int fl = block_flags<NW>(!act || bm.conv(tol), act && bm.bad(), sFlags, it & 1);
    if (fl & 2) { failed = true; break; }
    if (fl & 1) break;
  }

  // final flux: time average (fbar) + finiteness; q of every level back to registers
  double q[NQ][M];
#pragma unroll
  for (int t = 0; t < NQ; ++t) tmem_ld_doubles<M>(tq + 2 * M * t, 2, q[t]);
  tmem_fence_before();
  double fb[DIM][M];
#pragma unroll
  for (int a = 0; a < DIM; ++a)
#pragma unroll
    for (int c = 0; c < M; ++c) fb[a][c] = 0.0;
  if (!failed) {
    bool bad = false;
#pragma unroll
    for (int t = 0; t < NQ; ++t) {
      double F[DIM][M];
      flux<DIM>(q[t], F);
#pragma unroll
      for (int a = 0; a < DIM; ++a)
#pragma unroll
        for (int c = 0; c < M; ++c) {
          bad |= !finite(F[a][c]);
          fb[a][c] = fma(P.ops.w[t], F[a][c], fb[a][c]);
        }
    }
    failed = __syncthreads_or(act && bad);
  } else {
    __syncthreads();
  }
  // every TMEM access of the CTA precedes the barrier above: release the columns
  tmem_fence_after();
  if (warp == 0) tmem_dealloc_cols<256>(s_tmem);
  if (failed) {
    if (tid == 0) {
      report_error(st, 2 * gcell + 1);
      if (mode_corrects(mode)) bulk_commit_wait();
    }
    return;
  }
  if (tid == 0) {
    atomicAdd((unsigned long long*)&st->picard_iters, (unsigned long long)iters);
    atomicAdd((unsigned long long*)&st->predicts, 1ull);
    atomicAdd((unsigned long long*)&st->hist[iters < HIST_BINS ? iters : HIST_BINS - 1], 1ull);
  }

  // every time level of q, qbar and fbar in C-order node layout (the operand buffers
  // are free: the last slice's owner loads precede the convergence barrier)
  if (act) {
#pragma unroll
    for (int c = 0; c < M; ++c) {
      double v = 0.0;
#pragma unroll
      for (int t = 0; t < NQ; ++t) {
        sQt[(t * M + c) * NS + x] = q[t][c];
        v = fma(P.ops.w[t], q[t][c], v);
      }
      sQb[c * NS + x] = v;
#pragma unroll
      for (int a = 0; a < DIM; ++a) sFb[(a * M + c) * NS + x] = fb[a][c];
    }
  }
  if (tid < 2 * DIM) sSmax[tid] = 0ull;
  __syncthreads();

  // ---------------- integrate_volume (kernels.py:130-143) ----------------
  if (act) {
    const int idx[3] = {i0, i1, i2};
    constexpr int gstr[3] = {NQ * NQ, NQ, 1};
#pragma unroll
    for (int c = 0; c < M; ++c) {
      double s = 0.0;
#pragma unroll
      for (int a = 0; a < DIM; ++a) {
        const double* b = sFb + (a * M + c) * NS + x - idx[a] * gstr[a];
#pragma unroll
        for (int j = 0; j < NQ; ++j) s = fma(P.ops.kvol[idx[a]][j], b[j * gstr[a]], s);
      }
      sD[x * M + c] = s * scale;
    }
    fence_proxy_async();
  }

  // ---------------- s_max over the space-time face traces ----------------
  // tasks per face axis a: (t, face node y, side), side fastest (the two lanes of a
  // pair read the same trace nodes); per-thread maxima reduced over the warp and
  // merged with one shared atomic per warp and side
  double smx[2 * DIM];
#pragma unroll
  for (int f = 0; f < 2 * DIM; ++f) smx[f] = 0.0;
#pragma unroll
  for (int a = 0; a < DIM; ++a) {
    const int sa = (a == 0) ? NQ * NQ : (a == 1) ? NQ : 1;
    for (int e = tid; e < 2 * NQ * NF; e += THREADS) {
      const int side = e & 1;
      const int y = (e >> 1) % NF;
      const int t = (e >> 1) / NF;
      const double* vec = side ? P.ops.right : P.ops.left;
      const int ya = y / NQ, yb = y % NQ;
      const int base = (a == 0) ? ya * NQ + yb : (a == 1) ? ya * NQ * NQ + yb : (ya * NQ + yb) * NQ;
      double qs[M];
#pragma unroll
      for (int c = 0; c < M; ++c) qs[c] = 0.0;
#pragma unroll
      for (int i = 0; i < NQ; ++i) {
        const double v = vec[i];
#pragma unroll
        for (int c = 0; c < M; ++c) qs[c] = fma(v, sQt[(t * M + c) * NS + base + i * sa], qs[c]);
      }
      bool adm;
      const double sp = max_speed_fast<DIM>(qs, a, a + 1, adm);
      // NaN must win the max like the reference's np.max: compare bit patterns
      if (side) smx[2 * a + 1] = (__double_as_longlong(sp) > __double_as_longlong(smx[2 * a + 1])) ? sp : smx[2 * a + 1];
      else smx[2 * a] = (__double_as_longlong(sp) > __double_as_longlong(smx[2 * a])) ? sp : smx[2 * a];
    }
  }
#pragma unroll
  for (int f = 0; f < 2 * DIM; ++f) {
    const unsigned long long v = warp_max_u64((unsigned long long)__double_as_longlong(smx[f]));
    if (lane == 0) atomicMax(&sSmax[f], v);
  }
  __syncthreads();
  if (tid == 0) {
    bulk_s2g(Dg, sD, NS * M * 8);
    bulk_commit_wait();   // also covers the Q store issued in the corrector
  }
  // ---------------- face records: qbar and fbar traces (kernels.py:107-128) ----------------
#pragma unroll
  for (int a = 0; a < DIM; ++a) {
    const int sa = (a == 0) ? NQ * NQ : (a == 1) ? NQ : 1;
    for (int e = tid; e < 2 * M * NF; e += THREADS) {
      const int side = e & 1;
      const int y = (e >> 1) % NF;
      const int c = (e >> 1) / NF;
      const double* vec = side ? P.ops.right : P.ops.left;
      const int ya = y / NQ, yb = y % NQ;
      const int base = (a == 0) ? ya * NQ + yb : (a == 1) ? ya * NQ * NQ + yb : (ya * NQ + yb) * NQ;
      double vq = 0.0, vf = 0.0;
#pragma unroll
      for (int i = 0; i < NQ; ++i) {
        vq = fma(vec[i], sQb[c * NS + base + i * sa], vq);
        vf = fma(vec[i], sFb[(a * M + c) * NS + base + i * sa], vf);
      }
      double* rec = P.tr_out + ((long long)(2 * a + side) * P.slots + own_slot) * REC;
      rec[y * M + c] = vq;
      rec[NF * M + y * M + c] = vf;
    }
  }
  if (tid < 2 * DIM) {
    double* rec = P.tr_out + ((long long)tid * P.slots + own_slot) * REC;
    rec[2 * NF * M] = __longlong_as_double((long long)sSmax[tid]);
    rec[2 * NF * M + 1] = record_stamp(P);
  }
}

}  // namespace adg
