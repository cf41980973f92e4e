// aderdg_sweep_st.cuh — fused sweep kernel with one thread per SPACE-TIME node (3D, p = 3).
//
// 256 threads per cell (4^3 spatial nodes x 4 time levels).  Lane bits:
//   lane = t + 4*i0lo + 8*i1lo + 16*i2lo,   warp = 4*i0hi + 2*i1hi + i2hi
// so each warp owns a 2x2x2 spatial block over all time levels.  Compared to
// the thread-per-spatial-node kernel (sweep_kernel_v2) this removes the
// per-thread time line (no register rotation, ~1/4 of the registers, 2x the
// resident warps), and puts the time contraction of the Picard update on the
// FP64 tensor cores: with t in lane bits 0-1, `acc = integ . dv` over the time
// levels of a node is one DMMA.8x8x4 per component with dv in the A fragment
// and an interleaved integ^T in B (the result lands in the lane that owns the
// space-time node).  The time averages (f̄, q̄) use the same trick with a
// weight column.  Spatial derivatives gather the flux of all time levels from
// shared memory in an XOR-swizzled layout:
//   addr(t, c, node) = (5t + c)*68 + 8*block + 4*i0lo + 2*(i0lo^i2lo) + (i1lo^i2lo)
// for which every axis gather of a warp (16 distinct words) hits 16 distinct
// 8-byte banks, and the stores hit every bank exactly twice.
//
// Reference (src/ = /root/reference/pkg/src/aderdg/): kernels.py:68-229,
// scheduler.py:370-449 (same tasks and order as sweep_kernel).
#pragma once
#include "aderdg_kernels.cuh"
#include "aderdg_sweep_v2.cuh"

namespace adg {

struct ShapeST {
  static constexpr int NQ = 4, DIM = 3, M = 5;
  static constexpr int NS = 64, NF = 16, THREADS = 256, NW = 8;
  static constexpr int REC = 2 * NF * M + 2;
  static constexpr int SX = 68;                         // per (t, c) stride of the swizzled layout
  static constexpr int SLAB = 4 * M * SX;               // one axis of flux, all time levels (1360)
  // shared memory (doubles)
  static constexpr int R_RED = 2 * NW + 2 * DIM + 4;
  static constexpr int R_Q = NS * M;
  static constexpr int R_REC = 4 * DIM * REC;           // 1944
  static constexpr int R_PIC = DIM * SLAB;              // 4080: flux of the 3 axes (Picard)
  static constexpr int R_U = R_REC > R_PIC ? R_REC : R_PIC;
  static constexpr int R_FACE = 2 * DIM * NF * M;
  static constexpr int OFF_BAR = 0;
  static constexpr int OFF_RED = 2;
  static constexpr int OFF_Q = OFF_RED + ((R_RED + 1) & ~1);
  static constexpr int OFF_D = OFF_Q + R_Q;
  static constexpr int OFF_U = OFF_D + R_Q;
  static constexpr int OFF_FACE = OFF_U + R_U;
  static constexpr int TOTAL = OFF_FACE + R_FACE;
  static constexpr size_t SMEM_BYTES = sizeof(double) * TOTAL;
};

__device__ __forceinline__ int st_sw(int i0, int i1, int i2) {
  const int blk = 4 * (i0 >> 1) + 2 * (i1 >> 1) + (i2 >> 1);
  const int a = i0 & 1, b = i1 & 1, c = i2 & 1;
  return 8 * blk + 4 * a + 2 * (a ^ c) + (b ^ c);
}

__global__ void __launch_bounds__(256, 3) sweep_kernel_st(const SweepParams P) {
  using S = ShapeST;
  constexpr int NQ = 4, DIM = 3, M = 5, NS = S::NS, NF = S::NF, REC = S::REC;
  constexpr int THREADS = S::THREADS, NW = S::NW, SX = S::SX, SLAB = S::SLAB;

  extern __shared__ __align__(16) double smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + S::OFF_BAR);
  double* sRed = smem + S::OFF_RED;
  unsigned long long* sSmax = reinterpret_cast<unsigned long long*>(sRed + 2 * NW);
  double* sQ = smem + S::OFF_Q;
  double* sD = smem + S::OFF_D;
  double* sU = smem + S::OFF_U;
  double* sRec = sU;                   // corrector phase
  double* sF = sU;                     // predictor: [axis][t][c][SX]
  double* sFace = smem + S::OFF_FACE;

  DevState* st = P.st;
  if (st->status != 0) return;
  const int mode = P.mode;
  if (mode == MODE_RERUN && !st->rerun_next) return;
  if (mode_corrects(mode) && st->reduce[1] != 0) return;   // a predict pass already failed

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int t = lane & 3;
  const int i0 = 2 * ((warp >> 2) & 1) + ((lane >> 2) & 1);
  const int i1 = 2 * ((warp >> 1) & 1) + ((lane >> 3) & 1);
  const int i2 = 2 * (warp & 1) + ((lane >> 4) & 1);
  const int x = (i0 * NQ + i1) * NQ + i2;
  const bool lead = (t == 0);          // one lane per spatial node for the per-node work
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
      for (int f = 0; f < 2 * DIM; ++f) {
        const int a = f >> 1, dir = (f & 1) ? 1 : -1;
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
      }
    }
  }
  mbar_wait(bar, 0);

  double Qx[M];
#pragma unroll
  for (int c = 0; c < M; ++c) Qx[c] = sQ[x * M + c];

  if (mode_corrects(mode)) {
    // ------------- Riemann (kernels.py:147-179), time-collapsed -------------
    for (int e = tid; e < 2 * DIM * NF * M; e += THREADS) {
      const int f = e / (NF * M), yc = e % (NF * M);
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
    // ------------- integrate_face + update (kernels.py:183-214), one lane per node -------------
    if (lead) {
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
    if (!lead) {
#pragma unroll
      for (int c = 0; c < M; ++c) Qx[c] = sQ[x * M + c];
    }
  }

  if (!mode_predict_only(mode)) {
    // ------------- calc_time_step (kernels.py:216-229) -------------
    bool ok = true;
    double lam = 0.0;
    if (lead) {
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
#pragma unroll
    for (int c = 0; c < M; ++c) ok = ok && finite(Qx[c]);
    if (!__syncthreads_and(ok)) {
      if (tid == 0) report_error(st, 2 * gcell + 1);
      return;
    }
  }

  // ---------------- predictor (kernels.py:68-105) ----------------
  const double dt = (mode == MODE_RERUN) ? st->dt_old : st->dt_new;
  const double scale = (mode == MODE_RERUN) ? st->scale_old : st->scale_new;   // dt / h (SF: dt_new)
  double absmax;
  {
    double am = 0.0;
#pragma unroll
    for (int c = 0; c < M; ++c) am = fmax(am, fabs(Qx[c]));
    absmax = block_max<NW>(am, sRed);
  }
  const double tol = 1e-10 * (1.0 + absmax);
  const int cap = 2 * NQ;

  // derivative rows and gather bases (swizzled addresses of the 4 nodes on each axis line)
  double drow[DIM][NQ];
  int gad[DIM][NQ];
  {
    const int idx[3] = {i0, i1, i2};
#pragma unroll
    for (int a = 0; a < DIM; ++a)
#pragma unroll
      for (int j = 0; j < NQ; ++j) {
        drow[a][j] = P.ops.diff[idx[a]][j];
        gad[a][j] = (a == 0) ? st_sw(j, i1, i2) : (a == 1) ? st_sw(i0, j, i2) : st_sw(i0, i1, j);
      }
  }
  const int own = st_sw(i0, i1, i2);
  // DMMA B fragments: time contraction (interleaved integ^T) and time average (weights)
  double bint, bw;
  {
    const int g = lane >> 2, t4 = lane & 3;      // B[k = t4][n = g]
    bint = (g & 1) ? 0.0 : P.ops.integ[g >> 1][t4];
    bw = (g == 0) ? P.ops.w[t4] : 0.0;
  }

  double q[M];
#pragma unroll
  for (int c = 0; c < M; ++c) q[c] = Qx[c];
  int iters = 0;
  bool failed = false;
#pragma unroll 1
  for (int it = 0; it < cap; ++it) {
    double F[DIM][M];
    flux<DIM>(q, F);
#pragma unroll
    for (int a = 0; a < DIM; ++a)
#pragma unroll
      for (int c = 0; c < M; ++c) sF[a * SLAB + (t * M + c) * SX + own] = F[a][c];
    __syncthreads();
    double dmax = 0.0, dsum = 0.0;
#pragma unroll
    for (int c = 0; c < M; ++c) {
      double part[DIM];
#pragma unroll
      for (int a = 0; a < DIM; ++a) {
        const double* b = sF + a * SLAB + (t * M + c) * SX;
        double v = drow[a][0] * b[gad[a][0]];
#pragma unroll
        for (int j = 1; j < NQ; ++j) v = fma(drow[a][j], b[gad[a][j]], v);
        part[a] = v;
      }
      const double dv = (part[0] + part[1]) + part[2];
      // acc[t] = sum_k integ[t][k] dv[k] over the 4 time lanes of this node
      double acc, junk;
      dmma_8x8x4(acc, junk, dv, bint, 0.0, 0.0);
      const double qn = Qx[c] - scale * acc;
      const double dd = fabs(qn - q[c]);
      dmax = fmax(dmax, dd);
      dsum += dd;
      q[c] = qn;
    }
    iters = it + 1;
    if (__syncthreads_or(!finite(dsum))) { failed = true; break; }
    const double delta = block_max<NW>(dmax, sRed);
    if (delta <= tol) break;
  }

  // final flux, its finiteness, and the time averages f̄ and q̄ (DMMA with a weight column:
  // the lead lane of every node receives the sums over its 4 time lanes)
  double fb[DIM][M], qb[M];
  if (!failed) {
    double F[DIM][M];
    flux<DIM>(q, F);
    bool bad = false;
#pragma unroll
    for (int a = 0; a < DIM; ++a)
#pragma unroll
      for (int c = 0; c < M; ++c) {
        bad |= !finite(F[a][c]);
        double junk;
        dmma_8x8x4(fb[a][c], junk, F[a][c], bw, 0.0, 0.0);
      }
#pragma unroll
    for (int c = 0; c < M; ++c) {
      double junk;
      dmma_8x8x4(qb[c], junk, q[c], bw, 0.0, 0.0);
    }
    failed = __syncthreads_or(bad);
  }
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

  // stage for the per-node tail: fbar (t = 0 slot of each axis slab), qbar (slab 0, t = 1),
  // and q at every time level (slab 1/2 reused after the volume integral)
  __syncthreads();   // all Picard gathers done before the slabs are overwritten
  if (lead) {
#pragma unroll
    for (int a = 0; a < DIM; ++a)
#pragma unroll
      for (int c = 0; c < M; ++c) sF[a * SLAB + c * SX + own] = fb[a][c];
  }
  if (tid < 2 * DIM) sSmax[tid] = 0ull;
  __syncthreads();

  // ---------------- integrate_volume (kernels.py:130-143): lane t takes components t, t+4 ----------------
  {
    const double sdt = scale;
    const int idx[3] = {i0, i1, i2};
    for (int c = t; c < M; c += 4) {
      double s = 0.0;
#pragma unroll
      for (int a = 0; a < DIM; ++a) {
        const double* b = sF + a * SLAB + c * SX;
#pragma unroll
        for (int j = 0; j < NQ; ++j) s = fma(P.ops.kvol[idx[a]][j], b[gad[a][j]], s);
      }
      sD[x * M + c] = s * sdt;
    }
    fence_proxy_async();
  }
  // f̄ face traces (records, second half) from the staged fbar
#pragma unroll
  for (int a = 0; a < DIM; ++a) {
    for (int e = tid; e < 2 * M * NF; e += THREADS) {
      const int y = e % NF, sc = e / NF, c = sc % M, side = sc / M;
      const double* vec = side ? P.ops.right : P.ops.left;
      const int ya = y / NQ, yb = y % NQ;
      double v = 0.0;
#pragma unroll
      for (int i = 0; i < NQ; ++i) {
        const int ad = (a == 0) ? st_sw(i, ya, yb) : (a == 1) ? st_sw(ya, i, yb) : st_sw(ya, yb, i);
        v = fma(vec[i], sF[a * SLAB + c * SX + ad], v);
      }
      P.tr_out[((long long)(2 * a + side) * P.slots + own_slot) * REC + NF * M + y * M + c] = v;
    }
  }
  __syncthreads();
  if (tid == 0) {
    bulk_s2g(Dg, sD, NS * M * 8);   // D (and the Q store issued in the corrector)
  }
  // q at every time level and q̄ into slab 0 / slab 1 (t-slot 0)
#pragma unroll
  for (int c = 0; c < M; ++c) sF[(t * M + c) * SX + own] = q[c];
  if (lead) {
#pragma unroll
    for (int c = 0; c < M; ++c) sF[SLAB + c * SX + own] = qb[c];
  }
  __syncthreads();
  // s_max over the space-time traces: task = (face axis a, side, t, face node y)
#pragma unroll
  for (int a = 0; a < DIM; ++a) {
    for (int e = tid; e < 2 * NQ * NF; e += THREADS) {
      const int y = e % NF, st_ = e / NF, tt = st_ % NQ, side = st_ / NQ;
      const double* vec = side ? P.ops.right : P.ops.left;
      const int ya = y / NQ, yb = y % NQ;
      double qs[M];
#pragma unroll
      for (int c = 0; c < M; ++c) qs[c] = 0.0;
#pragma unroll
      for (int i = 0; i < NQ; ++i) {
        const int ad = (a == 0) ? st_sw(i, ya, yb) : (a == 1) ? st_sw(ya, i, yb) : st_sw(ya, yb, i);
        const double v = vec[i];
#pragma unroll
        for (int c = 0; c < M; ++c) qs[c] = fma(v, sF[(tt * M + c) * SX + ad], qs[c]);
      }
      bool adm;
      const double sp = max_speed_fast<DIM>(qs, a, a + 1, adm);
      atomicMax(&sSmax[2 * a + side], (unsigned long long)__double_as_longlong(sp));
    }
  }
  // q̄ face traces (records, first half)
#pragma unroll
  for (int a = 0; a < DIM; ++a) {
    for (int e = tid; e < 2 * M * NF; e += THREADS) {
      const int y = e % NF, sc = e / NF, c = sc % M, side = sc / M;
      const double* vec = side ? P.ops.right : P.ops.left;
      const int ya = y / NQ, yb = y % NQ;
      double v = 0.0;
#pragma unroll
      for (int i = 0; i < NQ; ++i) {
        const int ad = (a == 0) ? st_sw(i, ya, yb) : (a == 1) ? st_sw(ya, i, yb) : st_sw(ya, yb, i);
        v = fma(vec[i], sF[SLAB + c * SX + ad], v);
      }
      P.tr_out[((long long)(2 * a + side) * P.slots + own_slot) * REC + y * M + c] = v;
    }
  }
  __syncthreads();
  if (tid < 2 * DIM) {
    double* rec = P.tr_out + ((long long)tid * P.slots + own_slot) * REC;
    rec[2 * NF * M] = __longlong_as_double((long long)sSmax[tid]);
    rec[2 * NF * M + 1] = 0.0;
  }
  if (tid == 0) bulk_commit_wait();
}

}  // namespace adg
