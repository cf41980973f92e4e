// aderdg_sweep_hoc.cuh — high-order fused sweep on a 2-CTA thread-block cluster
// (3D, even n = p + 1; the p = 9 path).
//
// At p = 9 one cell's Picard time line (old iterate + divergence history,
// 2 x 10^4 x 5 doubles = 800 KB) lives in local memory, and with one cell per SM
// the 148 working sets (118 MB) do not stay in L2: ~250 GB of DRAM traffic per
// sweep (profiles/r01/s3).  Here a cell runs on a cluster of two CTAs on two SMs:
// CTA r owns the node planes i0 in [r n/2, (r+1) n/2) (500 nodes, one per
// thread), so each SM keeps half a time line (400 KB, ~60 MB across the GPU) and
// a thread carries one node instead of two (no register spills).
//   * flux slabs [axis][c][SC] are full-cell in each CTA; a thread writes its
//     node's three fluxes locally and its axis-0 flux into the partner's slab
//     through distributed shared memory, so the axis-0 derivative lines (the only
//     ones that cross the cut) read everything locally;
//   * each CTA computes the axis-0 lines' outputs on its own planes and the axis-1
//     and axis-2 lines of its planes (one line per thread, diff from the constant
//     bank): 1000 line tasks per CTA and slice;
//   * two cluster barriers per slice (slabs complete; partner done reading);
//     every exit decision (admissibility, convergence, failure) is taken
//     cluster-wide so both CTAs always leave together;
//   * the tail stages f̄, q̄ and q_t per axis the same way (axis-0 data mirrored),
//     x-face records are written by the CTA of that side, y/z-face records by the
//     owner of the face node's plane, s_max maxima are combined in rank 0.
//
// Reference (src/ = /root/reference/pkg/src/aderdg/): kernels.py:68-229,
// scheduler.py:370-449 (same tasks as sweep_kernel / sweep_kernel_ho).
#pragma once
#include <cooperative_groups.h>
#include "aderdg_sweep_ho.cuh"

namespace adg {

namespace cgx = cooperative_groups;

// outputs i0 in [R*H, R*H + H) of one axis-0 line (stride SA), rows of diff from
// the constant bank with compile-time indices
template <int NQ, int SA, int R>
__device__ __forceinline__ void deriv_half_line(double* ln, const SweepParams& P) {
  constexpr int H = NQ / 2;
  double in[NQ];
#pragma unroll
  for (int j = 0; j < NQ; ++j) in[j] = ln[j * SA];
  double out[H];
#pragma unroll
  for (int ii = 0; ii < H; ++ii) {
    double s = P.ops.diff[R * H + ii][0] * in[0];
#pragma unroll
    for (int j = 1; j < NQ; ++j) s = fma(P.ops.diff[R * H + ii][j], in[j], s);
    out[ii] = s;
  }
#pragma unroll
  for (int ii = 0; ii < H; ++ii) ln[(R * H + ii) * SA] = out[ii];
}

template <int NQ>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(512, 1) sweep_kernel_hoc(const SweepParams P) {
  using S = ShapeHO<NQ, true>;
  static_assert(NQ % 2 == 0 && (NQ / 2) * NQ * NQ <= 512, "one node per thread on half a cell");
  constexpr int DIM = 3, M = 5, NS = S::NS, NF = S::NF, REC = S::REC;
  constexpr int THREADS = S::THREADS, NW = S::NW;
  constexpr int SC = S::SC, P0 = S::P0, P1 = S::P1;
  constexpr int H = NQ / 2, NSH = H * NF;

  extern __shared__ __align__(16) double smem[];
  double* sRed = smem + S::OFF_RED;
  unsigned long long* sSmax = reinterpret_cast<unsigned long long*>(sRed + 2 * NW);
  double* sFA = smem + S::OFF_FA;     // [axis][M][SC] flux slabs (full cell)
  double* sN = smem + S::OFF_NODE;    // [M][NS] node staging (aliases the slabs in the tail)
  double* sFace = smem + S::OFF_FACE;
  // cluster exchange words: [0..1] flags, [2..3] maxima, [4..9] partner s_max
  __shared__ unsigned long long sX[16];

  cgx::cluster_group cl = cgx::this_cluster();
  const int rank = (int)cl.block_rank();
  const int peer = rank ^ 1;
  unsigned long long* pX = cl.map_shared_rank(sX, peer);
  double* pFA = cl.map_shared_rank(sFA, peer);
  double* pN = cl.map_shared_rank(sN, peer);
  const int tid = threadIdx.x;
  cl.sync();   // both CTAs resident before any distributed-shared-memory access

  // cluster-wide OR / max of one 64-bit word per CTA (slot s of sX); every call is
  // a cluster barrier, so both CTAs take the same branch afterwards
  auto cluster_or = [&](bool v, int s) -> bool {
    const bool b = __syncthreads_or(v);
    if (tid == 0) pX[s] = b ? 1ull : 0ull;
    cl.sync();
    const bool r = b || (sX[s] != 0ull);
    cl.sync();                       // the slot may be rewritten by the next call
    return r;
  };
  auto cluster_max = [&](double v, int s) -> double {
    const double b = block_max<NW>(v, sRed);
    if (tid == 0) pX[s] = (unsigned long long)__double_as_longlong(b);
    cl.sync();
    const unsigned long long o = sX[s], m = (unsigned long long)__double_as_longlong(b);
    cl.sync();
    return __longlong_as_double((long long)(o > m ? o : m));
  };

  DevState* st = P.st;
  const int mode = P.mode;
  bool skip = (st->status != 0) || (mode == MODE_RERUN && !st->rerun_next) ||
              (mode_corrects(mode) && st->reduce[1] != 0);
  if (cluster_or(skip, 0)) return;

  const int b = (int)(blockIdx.x >> 1);
  const long long cell = (long long)b + (b < P.blk_split ? P.cell_a : P.cell_jump);
  const long long gcell = cell + P.cell_offset;
  const int plane = (int)(cell / P.plane_cells);
  const int rest = (int)(cell % P.plane_cells);
  const long long own_slot = (long long)(plane + 1) * P.plane_cells + rest;
  const int step_idx = mode_corrects(mode) ? st->step + 1 : 0;
  double* Qg = P.Q + cell * (NS * M);
  double* Dg = P.D + cell * (NS * M);

  // this thread's node (one per thread on the CTA's planes)
  const bool an = tid < NSH;
  const int xn = rank * NSH + (an ? tid : 0);
  int i3[3];
  i3[0] = xn / NF; i3[1] = (xn / NQ) % NQ; i3[2] = xn % NQ;
  const int pn = i3[0] * P0 + i3[1] * P1 + i3[2];

  double Qx[M];
#pragma unroll
  for (int c = 0; c < M; ++c) Qx[c] = Qg[xn * M + c];

  if (mode_corrects(mode)) {
    // ------------- Riemann on the 2d faces (kernels.py:147-179), both CTAs -------------
    long long nb_slot[2 * DIM];
#pragma unroll
    for (int f = 0; f < 2 * DIM; ++f) {
      const int a = f >> 1, dir = (f & 1) ? 1 : -1;
      if (a == 0) {
        int pl = plane + dir;
        if (!P.halo) pl = (pl + P.K) % P.K;
        nb_slot[f] = (long long)(pl + 1) * P.plane_cells + rest;
      } else {
        const int st_a = (a == 1) ? P.K : 1;
        const int ia = (rest / st_a) % P.K;
        const int ja = (ia + dir + P.K) % P.K;
        nb_slot[f] = (long long)(plane + 1) * P.plane_cells + rest + (ja - ia) * st_a;
      }
    }
    for (int e = tid; e < 2 * DIM * NF * M; e += THREADS) {
      const int f = e / (NF * M), yc = e % (NF * M);
      const double* own = P.tr_in + ((long long)f * P.slots + own_slot) * REC;
      const double* nb = P.tr_in + ((long long)(f ^ 1) * P.slots + nb_slot[f]) * REC;
      const double* mr = (f & 1) ? own : nb;
      const double* pr = (f & 1) ? nb : own;
      const double alpha = rusanov_alpha(mr[2 * NF * M], pr[2 * NF * M]);
      const double fs = __dsub_rn(__dmul_rn(0.5, __dadd_rn(mr[NF * M + yc], pr[NF * M + yc])),
                                  __dmul_rn(__dmul_rn(0.5, alpha), __dsub_rn(pr[yc], mr[yc])));
      sFace[e] = (f & 1) ? fs : -fs;
    }
    __syncthreads();
    // ------------- integrate_face + update (kernels.py:183-214), own nodes -------------
    const double scale_old = (mode == MODE_SF_CORRECT) ? st->scale_new : st->scale_old;
    if (an) {
      double Dx[M];
#pragma unroll
      for (int c = 0; c < M; ++c) Dx[c] = Dg[xn * M + c];
#pragma unroll
      for (int a = 0; a < DIM; ++a) {
        const int y = (a == 0) ? i3[1] * NQ + i3[2] : (a == 1) ? i3[0] * NQ + i3[2] : i3[0] * NQ + i3[1];
        const double slo = __dmul_rn(scale_old, P.ops.lift_lo[i3[a]]);
        const double shi = __dmul_rn(scale_old, P.ops.lift_hi[i3[a]]);
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
        for (int bb = 0; bb < DIM; ++bb) Qx[1 + bb] = __dmul_rn(Qx[1 + bb], P.spike_factor);
        double jj = __dmul_rn(Qx[1], Qx[1]);
#pragma unroll
        for (int bb = 1; bb < DIM; ++bb) jj = __dadd_rn(jj, __dmul_rn(Qx[1 + bb], Qx[1 + bb]));
        Qx[M - 1] = __dadd_rn(__ddiv_rn(pr, 0.4), __ddiv_rn(__dmul_rn(0.5, jj), rho));
      }
#pragma unroll
      for (int c = 0; c < M; ++c) Qg[xn * M + c] = Qx[c];
    }
  }

  if (!mode_predict_only(mode)) {
    // ------------- calc_time_step (kernels.py:216-229) -------------
    bool ok = true;
    double lam = 0.0;
    if (an) {
      bool fin = true;
#pragma unroll
      for (int c = 0; c < M; ++c) fin = fin && finite(Qx[c]);
      bool adm = false;
      const double l = max_speed_fast<DIM>(Qx, 0, DIM, adm);
      ok = fin && adm;
      if (ok) lam = l;
    }
    if (cluster_or(!ok, 0)) {
      if (tid == 0 && rank == 0) report_error(st, 2 * gcell + 0);
      return;
    }
    lam = block_max<NW>(lam, sRed);
    if (tid == 0) atomicMax(&st->reduce[0], __double_as_longlong(lam));
    if (mode == MODE_SEED) return;
    if (mode == MODE_SF_CORRECT) return;
  } else {
    bool ok = true;
    if (an) {
#pragma unroll
      for (int c = 0; c < M; ++c) ok = ok && finite(Qx[c]);
    }
    if (cluster_or(!ok, 0)) {
      if (tid == 0 && rank == 0) report_error(st, 2 * gcell + 1);
      return;
    }
  }

  // ---------------- predictor (kernels.py:68-105) ----------------
  const double scale = (mode == MODE_RERUN) ? st->scale_old : st->scale_new;   // dt / h (SF: dt_new)
  double am = 0.0;
  if (an) {
#pragma unroll
    for (int c = 0; c < M; ++c) am = fmax(am, fabs(Qx[c]));
  }
  const double tol = 1e-10 * (1.0 + cluster_max(am, 2));
  const int cap = 2 * NQ;

  double qo[NQ][M];
  double dh[NQ][M];
  int iters = 0;
  bool failed = false;
#pragma unroll 1
  for (int it = 0; it < cap; ++it) {
#pragma unroll 1
    for (int k = 0; k < NQ; ++k) {
      double F[DIM][M];
      {
        double qq[M];
#pragma unroll
        for (int c = 0; c < M; ++c) qq[c] = (it == 0) ? Qx[c] : qo[k][c];
        flux<DIM>(qq, F);
      }
      if (an) {
#pragma unroll
        for (int a = 0; a < DIM; ++a)
#pragma unroll
          for (int c = 0; c < M; ++c) sFA[a * S::R_FA + c * SC + pn] = F[a][c];
#pragma unroll
        for (int c = 0; c < M; ++c) pFA[c * SC + pn] = F[0][c];          // mirror for the axis-0 lines
      }
      cl.sync();
      // line tasks: [0, NF*M) axis-0 lines (own output planes), then the axis-1 and
      // axis-2 lines of the own planes (H*NQ*M each)
      for (int l = tid; l < NF * M + 2 * H * NQ * M; l += THREADS) {
        if (l < NF * M) {
          const int c = l / NF, y = l % NF;
          double* ln = sFA + c * SC + (y / NQ) * P1 + (y % NQ);
          if (rank == 0) deriv_half_line<NQ, P0, 0>(ln, P);
          else deriv_half_line<NQ, P0, 1>(ln, P);
        } else if (l < NF * M + H * NQ * M) {
          const int u = l - NF * M, c = u / (H * NQ), r = u % (H * NQ);
          const int i0 = rank * H + r / NQ, i2 = r % NQ;
          deriv_line<NQ, P1>(sFA + S::R_FA + c * SC + i0 * P0 + i2, P);
        } else {
          const int u = l - NF * M - H * NQ * M, c = u / (H * NQ), r = u % (H * NQ);
          const int i0 = rank * H + r / NQ, i1 = r % NQ;
          deriv_line<NQ, 1>(sFA + 2 * S::R_FA + c * SC + i0 * P0 + i1 * P1, P);
        }
      }
      cl.sync();   // own outputs complete here, the partner done reading its mirror of ours
#pragma unroll
      for (int c = 0; c < M; ++c)
        dh[k][c] = (sFA[c * SC + pn] + sFA[S::R_FA + c * SC + pn]) + sFA[2 * S::R_FA + c * SC + pn];
    }
    // time contraction + Picard update (the node's history read once per component)
    BitMax bm;
#pragma unroll 1
    for (int c = 0; c < M; ++c) {
      double dk[NQ];
#pragma unroll
      for (int k = 0; k < NQ; ++k) dk[k] = dh[k][c];
#pragma unroll
      for (int t = 0; t < NQ; ++t) {
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < NQ; ++k) acc = fma(P.ops.integ[t][k], dk[k], acc);
        const double qn = Qx[c] - scale * acc;
        const double qold = (it == 0) ? Qx[c] : qo[t][c];
        if (an) bm.add(fabs(qn - qold));
        qo[t][c] = qn;
      }
    }
    iters = it + 1;
    if (cluster_or(bm.bad(), 0)) { failed = true; break; }
    const double delta = cluster_max(__longlong_as_double((long long)bm.m), 2);
    if (delta <= tol) break;
  }

  // final flux: time average fbar, qbar + finiteness
  double fb[DIM][M], qb[M];
#pragma unroll
  for (int a = 0; a < DIM; ++a)
#pragma unroll
    for (int c = 0; c < M; ++c) fb[a][c] = 0.0;
#pragma unroll
  for (int c = 0; c < M; ++c) qb[c] = 0.0;
  if (!failed) {
    bool bad = false;
#pragma unroll 1
    for (int t = 0; t < NQ; ++t) {
      double F[DIM][M];
      flux<DIM>(qo[t], F);
      const double w = P.ops.w[t];
#pragma unroll
      for (int a = 0; a < DIM; ++a)
#pragma unroll
        for (int c = 0; c < M; ++c) {
          bad |= an && !finite(F[a][c]);
          fb[a][c] = fma(w, F[a][c], fb[a][c]);
        }
#pragma unroll
      for (int c = 0; c < M; ++c) qb[c] = fma(w, qo[t][c], qb[c]);
    }
    failed = cluster_or(bad, 0);
  }
  if (failed) {
    if (tid == 0 && rank == 0) report_error(st, 2 * gcell + 1);
    return;
  }
  if (tid == 0 && rank == 0) {
    atomicAdd((unsigned long long*)&st->picard_iters, (unsigned long long)iters);
    atomicAdd((unsigned long long*)&st->predicts, 1ull);
    atomicAdd((unsigned long long*)&st->hist[iters < HIST_BINS ? iters : HIST_BINS - 1], 1ull);
  }

  // stage one value per own node in sN, mirrored into the partner's sN when the
  // axis-0 lines need it; a cluster barrier before (readers of the previous
  // contents done) and after (staging complete)
  auto stage = [&](const double (&v)[M], bool mirror) {
    cl.sync();
    if (an) {
#pragma unroll
      for (int c = 0; c < M; ++c) {
        sN[c * NS + xn] = v[c];
        if (mirror) pN[c * NS + xn] = v[c];
      }
    }
    cl.sync();
  };
  // does this CTA write the face record entry (face f, face node y)?
  auto owns_face = [&](int a, int side, int y) -> bool {
    return (a == 0) ? (side == rank) : ((y / NQ) / H == rank);
  };

  // ---------------- integrate_volume + f̄ traces, one axis at a time ----------------
  double Dv[M];
#pragma unroll
  for (int c = 0; c < M; ++c) Dv[c] = 0.0;
#pragma unroll 1
  for (int a = 0; a < DIM; ++a) {
    double fa[M];
#pragma unroll
    for (int c = 0; c < M; ++c) fa[c] = (a == 0) ? fb[0][c] : (a == 1) ? fb[1][c] : fb[2][c];
    stage(fa, a == 0);
    const int sa = (a == 0) ? NQ * NQ : (a == 1) ? NQ : 1;
    if (an) {
      const int base = xn - i3[a] * sa;
#pragma unroll
      for (int c = 0; c < M; ++c) {
        double s = Dv[c];
#pragma unroll
        for (int j = 0; j < NQ; ++j) s = fma(P.ops.kvol[i3[a]][j], sN[c * NS + base + j * sa], s);
        Dv[c] = s;
      }
    }
    for (int e = tid; e < 2 * NF * M; e += THREADS) {
      const int y = e % NF, sc = e / NF, c = sc % M, side = sc / M;
      if (!owns_face(a, side, y)) continue;
      const double* vec = side ? P.ops.right : P.ops.left;
      const int ya = y / NQ, yb = y % NQ;
      const int xb = (a == 0) ? ya * NQ + yb : (a == 1) ? ya * NQ * NQ + yb : (ya * NQ + yb) * NQ;
      double v = 0.0;
#pragma unroll
      for (int i = 0; i < NQ; ++i) v = fma(vec[i], sN[c * NS + xb + i * sa], v);
      P.tr_out[((long long)(2 * a + side) * P.slots + own_slot) * REC + NF * M + y * M + c] = v;
    }
  }
  if (an) {
#pragma unroll
    for (int c = 0; c < M; ++c) Dg[xn * M + c] = Dv[c] * scale;
  }

  // ---------------- q̄ face traces ----------------
  stage(qb, true);
  if (tid < 2 * DIM) sSmax[tid] = 0ull;
  for (int e = tid; e < 2 * DIM * NF * M; e += THREADS) {
    const int y = e % NF, fc = e / NF, c = fc % M, f = fc / M, a = f >> 1;
    if (!owns_face(a, f & 1, y)) continue;
    const double* vec = (f & 1) ? P.ops.right : P.ops.left;
    const int ya = y / NQ, yb = y % NQ;
    const int sa = (a == 0) ? NQ * NQ : (a == 1) ? NQ : 1;
    const int xb = (a == 0) ? ya * NQ + yb : (a == 1) ? ya * NQ * NQ + yb : (ya * NQ + yb) * NQ;
    double v = 0.0;
#pragma unroll
    for (int i = 0; i < NQ; ++i) v = fma(vec[i], sN[c * NS + xb + i * sa], v);
    P.tr_out[((long long)f * P.slots + own_slot) * REC + y * M + c] = v;
  }
  // ---------------- s_max over the space-time traces, one time level at a time ----------------
#pragma unroll 1
  for (int t = 0; t < NQ; ++t) {
    stage(qo[t], true);
    for (int e = tid; e < 2 * DIM * NF; e += THREADS) {
      const int y = e % NF, f = e / NF, a = f >> 1;
      if (!owns_face(a, f & 1, y)) continue;
      const double* vec = (f & 1) ? P.ops.right : P.ops.left;
      const int ya = y / NQ, yb = y % NQ;
      const int sa = (a == 0) ? NQ * NQ : (a == 1) ? NQ : 1;
      const int xb = (a == 0) ? ya * NQ + yb : (a == 1) ? ya * NQ * NQ + yb : (ya * NQ + yb) * NQ;
      double qs[M];
#pragma unroll
      for (int c = 0; c < M; ++c) {
        double v = 0.0;
#pragma unroll
        for (int i = 0; i < NQ; ++i) v = fma(vec[i], sN[c * NS + xb + i * sa], v);
        qs[c] = v;
      }
      bool adm;
      const double sp = max_speed_fast<DIM>(qs, a, a + 1, adm);
      atomicMax(&sSmax[f], (unsigned long long)__double_as_longlong(sp));
    }
  }
  // combine the side maxima in rank 0 (bit-pattern max keeps NaNs like np.max)
  __syncthreads();
  if (rank == 1 && tid < 2 * DIM) pX[4 + tid] = sSmax[tid];
  cl.sync();
  if (rank == 0 && tid < 2 * DIM) {
    const unsigned long long o = sX[4 + tid], m = sSmax[tid];
    double* rec = P.tr_out + ((long long)tid * P.slots + own_slot) * REC;
    rec[2 * NF * M] = __longlong_as_double((long long)(o > m ? o : m));
    rec[2 * NF * M + 1] = 0.0;
  }
  cl.sync();   // no CTA leaves while its partner may still touch its shared memory
}

}  // namespace adg
