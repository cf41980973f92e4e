// aderdg_sweep_p3.cuh — the fused 3D sweep at p = 3 (n = 4), and the TMA / mbarrier /
// DMMA helpers the other sweep kernels share.
//
// One CTA of 64 threads per cell (thread = spatial node, i2 in lane bits 0-1, i1 in bits
// 2-3), six CTAs per SM (168 registers); the node's whole time line q[t][c] and the time
// contraction accumulators stay in registers.
//   * TMA bulk copies (cp.async.bulk + mbarrier) stage Q, D and the 4d face records of the
//     cell into shared memory in one shot; Q and D go back with bulk stores.
//   * derivatives of a time slice: axis 2 is one DMMA.8x8x4 per component with the flux in
//     the A fragment and an interleaved diff^T in B, so the result lands in the lane that
//     owns the node; axis 1 the same through a lane transpose (__shfl_sync swaps the i1 and
//     i2 lane bits: one shuffle in, one out); only axis 0 goes through shared memory
//     (padded plane stride 20: the gathers of a warp are broadcasts, no bank conflicts).
//   * software-pipelined slices: the flux slices alternate between two buffers, one
//     barrier per slice; the interval after the barrier that publishes slice s also
//     produces slice s + 1 (flux, axis-0 store, axis-1 / axis-2 DMMAs) and contracts
//     slice s - 1 in time.
//   * the first Picard iteration (q_t = Q at every level: four identical slices)
//     computes one slice.
//   * Latin-cube swizzled trace layout for the face-trace gathers of the tail.
//
// Reference (src/ = /root/reference/pkg/src/aderdg/): kernels.py:68-229 (predict,
// extrapolate, integrate_volume, solve_riemann, integrate_face, update, calc_time_step),
// scheduler.py:370-449 (fused sweep).
#pragma once
#include "aderdg_kernels.cuh"

namespace adg {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void bulk_s2g(void* dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src)),
               "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void bulk_commit_wait() {
  asm volatile("cp.async.bulk.commit_group;\ncp.async.bulk.wait_group.read 0;" ::: "memory");
}

__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// D = A(8x4) * B(4x8) + C, fp64, one element of A and B per lane.
__device__ __forceinline__ void dmma_8x8x4(double& d0, double& d1, double a, double b, double c0, double c1) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};\n"
               : "=d"(d0), "=d"(d1)
               : "d"(a), "d"(b), "d"(c0), "d"(c1));
}

// Node address in the trace-phase q layout: Latin-cube swizzle 16 i2 + 4 ((i0 + i2) & 3) +
// ((i1 + i2) & 3): for every axis, the 16 nodes of a face plane hit 16 distinct 8-byte
// banks, so the face-trace gathers of a half-warp are conflict free along all three axes.
__device__ __forceinline__ int trace_addr(int i0, int i1, int i2) {
  return 16 * i2 + 4 * ((i0 + i2) & 3) + ((i1 + i2) & 3);
}

struct ShapeP3 {
  static constexpr int DIM = 3, M = 5, NQ = 4;
  static constexpr int NS = 64, NF = 16;
  static constexpr int THREADS = 64, NWARPS = 2, MINB = 6;
  static constexpr int P1 = NQ, P0 = NQ * NQ + 4;      // padded axis-0 plane stride: (P0 mod 16) in [4, 12]
  static constexpr int PS = NQ * P0;                   // padded slice size
  static constexpr int REC = 2 * NF * M + 2;
  // shared memory (doubles), all region sizes even (16-byte alignment)
  static constexpr int R_RED = 3 * NWARPS + 2 * DIM + 4;   // block_max | s_max | convergence flags
  static constexpr int R_Q = NS * M;
  static constexpr int R_REC = 4 * DIM * REC;
  static constexpr int R_F = M * PS;                   // one axis-0 flux slice (two buffers)
  static constexpr int R_FB = DIM * M * PS;            // fbar (after the Picard loop)
  static constexpr int R_DIV = (NQ + 1) * M * NS;      // q of every time level + qbar (tail)
  static constexpr int R_PRED = R_FB + R_DIV;
  static constexpr int R_U = R_REC > R_PRED ? R_REC : R_PRED;
  static constexpr int R_FACE = 2 * DIM * NF * M;
  static constexpr int OFF_BAR = 0;                    // 2 doubles for the mbarrier
  static constexpr int OFF_RED = 2;
  static constexpr int OFF_Q = OFF_RED + ((R_RED + 1) & ~1);
  static constexpr int OFF_D = OFF_Q + R_Q;
  static constexpr int OFF_U = OFF_D + R_Q;
  static constexpr int OFF_FACE = OFF_U + R_U;
  static constexpr int TOTAL = OFF_FACE + R_FACE;
  static constexpr size_t SMEM_BYTES = sizeof(double) * TOTAL;
  static_assert(2 * R_F <= R_PRED, "the two flux-slice buffers alias the tail region");
};

__global__ void __launch_bounds__(ShapeP3::THREADS, ShapeP3::MINB) sweep_kernel_p3(const SweepParams P) {
  using S = ShapeP3;
  constexpr int DIM = 3, M = 5, NQ = S::NQ, NS = S::NS, NF = S::NF, REC = S::REC;
  constexpr int THREADS = S::THREADS, NW = S::NWARPS, P0 = S::P0, P1 = S::P1, PS = S::PS;

  extern __shared__ __align__(16) double smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + S::OFF_BAR);
  double* sRed = smem + S::OFF_RED;
  unsigned long long* sSmax = reinterpret_cast<unsigned long long*>(sRed + 2 * NW);
  unsigned* sFlags = reinterpret_cast<unsigned*>(sRed + 2 * NW + 2 * 3);
  double* sQ = smem + S::OFF_Q;
  double* sD = smem + S::OFF_D;
  double* sU = smem + S::OFF_U;
  double* sRec = sU;                                   // corrector phase
  double* sF = sU;                                     // predictor: axis-0 flux slices [parity][M][PS]
  double* sDiv = sU + S::R_FB;                         // tail: q of every level [NQ][M][NS] + qbar
  double* sFace = smem + S::OFF_FACE;
  ADG_DEBUG_POISON();

  DevState* st = P.st;
  if (st->status != 0) return;
  const int mode = P.mode;
  if (mode == MODE_RERUN && !st->rerun_next) return;
  if (mode_corrects(mode) && st->reduce[1] != 0) return;   // a predict pass already failed

  const int tid = threadIdx.x;
  const int x = tid;                                   // thread = spatial node (64 nodes, two warps)
  const long long cell = sweep_cell(P);
  const long long gcell = cell + P.cell_offset;
  const int i0 = x / (NQ * NQ), i1 = (x / NQ) % NQ, i2 = x % NQ;
  const int px = i0 * P0 + i1 * P1 + i2;              // padded slice index

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
  // predictor setup that needs no cell data, while the bulk copies land
  // derivative row of the shared-memory axis (axis 0); DMMA B fragment of axes 1, 2
  double drow[NQ];
#pragma unroll
  for (int j = 0; j < NQ; ++j) drow[j] = P.ops.diff[i0][j];
  double bfrag;
  {
    const int lane = tid & 31;
    const int g = lane >> 2, t4 = lane & 3;      // B[k=t4][n=g]: n even -> diff[n/2][k]
    bfrag = (g & 1) ? 0.0 : P.ops.diff[g >> 1][t4];
  }
  // lane sigma(L) swaps lane bits 0-1 (i2) with bits 2-3 (i1).  The DMMA
  // A operand taken from lane sigma(L) has the i1 line in k; the product lands
  // in lane sigma(owner), so one shuffle in and one out replace the axis-1
  // shared-memory gather.
  const int sig = (tid & 16) | ((tid & 3) << 2) | ((tid >> 2) & 3);
  // padded gather bases for the shared-memory axes
  int gbase[DIM], gstr[DIM];
  gbase[0] = px - i0 * P0; gstr[0] = P0;
  gbase[1] = px - i1 * P1; gstr[1] = P1;
  gbase[2] = px - i2;      gstr[2] = 1;

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
    {
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
    {
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

  double q[NQ][M];
#pragma unroll
  for (int s = 0; s < NQ; ++s)
#pragma unroll
    for (int c = 0; c < M; ++c) q[s][c] = Qx[c];

  int iters = 0;
  bool failed = false;
  // Software-pipelined slice loop: the interval after the barrier
  // that publishes slice s also computes the flux of slice s+1 — its axis-0 flux
  // goes to the other buffer, whose readers (slice s-1) all passed this barrier —
  // and issues its axis-1 DMMA, so two independent dependency chains share every
  // barrier interval.  The slice's axis-2 DMMA (C = 0) is issued there too and
  // the axis-1 result transposed back, leaving only the axis-0 gather after the barrier.
  auto produce = [&](int sl, double (&f2)[M], double (&d1)[M]) {
    double F[DIM][M];
    flux<DIM>(q[sl], F);
    double* sFn = sF + (sl & 1) * (M * PS);
#pragma unroll
    for (int c = 0; c < M; ++c) sFn[c * PS + px] = F[0][c];
#pragma unroll
    for (int c = 0; c < M; ++c) {
      const double a1 = __shfl_sync(0xffffffffu, F[1][c], sig);
      double z1;
      dmma_8x8x4(d1[c], z1, a1, bfrag, 0.0, 0.0);
      dmma_8x8x4(f2[c], z1, F[2][c], bfrag, 0.0, 0.0);
    }
  };
  auto finish_produce = [&](double (&d1)[M]) {
#pragma unroll
    for (int c = 0; c < M; ++c) d1[c] = __shfl_sync(0xffffffffu, d1[c], sig);
  };
  bool first_done = false;
  // First iteration: q_t = Q at every time level, so its NQ slices are identical —
  // one slice is computed and its divergence contracted against every integ column
  // (the same operations in the same order as NQ equal slices).
  {
    double F2c[M], d1c[M];
    produce(0, F2c, d1c);
    finish_produce(d1c);
    __syncthreads();
    BitMax bm;
#pragma unroll
    for (int c = 0; c < M; ++c) {
      const double* b = sF + c * PS + gbase[0];
      double v = 0.0;
#pragma unroll
      for (int j = 0; j < NQ; ++j) v = fma(drow[j], b[j * gstr[0]], v);
      const double dv = (v + d1c[c]) + F2c[c];
#pragma unroll
      for (int t = 0; t < NQ; ++t) {
        double a = P.ops.integ[t][0] * dv;
#pragma unroll
        for (int k = 1; k < NQ; ++k) a = fma(P.ops.integ[t][k], dv, a);
        const double qn = Qx[c] - scale * a;
        bm.add(fabs(qn - q[t][c]));
        q[t][c] = qn;
      }
    }
    iters = 1;
    const int fl = block_flags<NW>(bm.conv(tol), bm.bad(), sFlags, 0);
    if (fl & 2) failed = true;
    first_done = fl != 0;
  }
#pragma unroll 1
  for (int it = 1; it < cap && !first_done; ++it) {
    double accr[NQ][M];
    double dvp[M];
    double F2c[M], d1c[M];           // current slice: axis-2 and axis-1 derivatives (DMMA results)
    produce(0, F2c, d1c);
    finish_produce(d1c);
#pragma unroll
    for (int s = 0; s < NQ; ++s) {
      __syncthreads();
      const double* sFs = sF + (s & 1) * (M * PS);
      double dv[M];
#pragma unroll
      for (int c = 0; c < M; ++c) {
        const double* b = sFs + c * PS + gbase[0];
        double v = 0.0;
#pragma unroll
        for (int j = 0; j < NQ; ++j) v = fma(drow[j], b[j * gstr[0]], v);
        dv[c] = (v + d1c[c]) + F2c[c];
      }
      double F2n[M], d1n[M];
      if (s + 1 < NQ) produce(s + 1 < NQ ? s + 1 : 0, F2n, d1n);
      if (s > 0) {
        // time contraction of slice s-1, deferred past its DMMA latency
#pragma unroll
        for (int t = 0; t < NQ; ++t)
#pragma unroll
          for (int c = 0; c < M; ++c)
            accr[t][c] = (s == 1) ? P.ops.integ[t][0] * dvp[c] : fma(P.ops.integ[t][s - 1], dvp[c], accr[t][c]);
      }
#pragma unroll
      for (int c = 0; c < M; ++c) dvp[c] = dv[c];
      if (s + 1 < NQ) {
        finish_produce(d1n);
#pragma unroll
        for (int c = 0; c < M; ++c) { F2c[c] = F2n[c]; d1c[c] = d1n[c]; }
      }
    }
#pragma unroll
    for (int t = 0; t < NQ; ++t)
#pragma unroll
      for (int c = 0; c < M; ++c) accr[t][c] = fma(P.ops.integ[t][NQ - 1], dvp[c], accr[t][c]);
    BitMax bm;
#pragma unroll
    for (int t = 0; t < NQ; ++t)
#pragma unroll
      for (int c = 0; c < M; ++c) {
        const double qn = Qx[c] - scale * accr[t][c];
        bm.add(fabs(qn - q[t][c]));
        q[t][c] = qn;
      }
    iters = it + 1;
    const int fl = block_flags<NW>(bm.conv(tol), bm.bad(), sFlags, it & 1);
    if (fl & 2) { failed = true; break; }
    if (fl & 1) break;
  }

  // final flux: time average fbar + finiteness
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

  // all time levels of q: [t][c][NS] in the trace layout
  double* sQt = sDiv;
  double* sQb = sDiv + NQ * M * NS;                    // qbar [c][NS] (trace layout)
  double* sFb = sF;                                    // [DIM][M][PS] total fbar
  const int qax = trace_addr(i0, i1, i2);
#pragma unroll
  for (int t = 0; t < NQ; ++t)
#pragma unroll
    for (int c = 0; c < M; ++c) sQt[(t * M + c) * NS + qax] = q[t][c];
#pragma unroll
  for (int a = 0; a < DIM; ++a)
#pragma unroll
    for (int c = 0; c < M; ++c) sFb[(a * M + c) * PS + px] = fb[a][c];
  if (tid < 2 * DIM) sSmax[tid] = 0ull;
  __syncthreads();

  // ---------------- integrate_volume (kernels.py:130-143) ----------------
  {
    const double sdt = scale;
    const int idx[3] = {i0, i1, i2};
#pragma unroll
    for (int c = 0; c < M; ++c) {
      double s = 0.0;
#pragma unroll
      for (int a = 0; a < DIM; ++a) {
        const double* b = sFb + (a * M + c) * PS + gbase[a];
#pragma unroll
        for (int j = 0; j < NQ; ++j) s = fma(P.ops.kvol[idx[a]][j], b[j * gstr[a]], s);
      }
      sD[x * M + c] = s * sdt;
    }
    fence_proxy_async();
  }

  // qbar = sum_t w_t q_t per node (trace layout)
  {
#pragma unroll
    for (int c = 0; c < M; ++c) {
      double v = 0.0;
#pragma unroll
      for (int t = 0; t < NQ; ++t) v = fma(P.ops.w[t], sQt[(t * M + c) * NS + qax], v);
      sQb[c * NS + qax] = v;
    }
  }

  // ---------------- s_max over the space-time face traces ----------------
  // tasks per face axis a (compile-time): (t, face node y, side), side fastest at
  // NQ != 4: the two lanes of a pair read the same trace nodes, so every lane quad
  // touches two distinct doubles per load (one wavefront, tools/smem_wavefronts.cu);
  // per-thread maxima are reduced over the warp and merged with one shared atomic per
  // warp and side
  double smx[2 * DIM];
#pragma unroll
  for (int f = 0; f < 2 * DIM; ++f) smx[f] = 0.0;
#pragma unroll
  for (int a = 0; a < DIM; ++a) {
    for (int e = tid; e < 2 * NQ * NF; e += THREADS) {
      // (y fastest: the Latin-cube trace layout is conflict-free per face plane)
      const int side = e / (NQ * NF);
      const int y = e % NF;
      const int t = (e / NF) % NQ;
      const double* vec = side ? P.ops.right : P.ops.left;
      const int ya = y / NQ, yb = y % NQ;
      double qs[M];
#pragma unroll
      for (int c = 0; c < M; ++c) qs[c] = 0.0;
#pragma unroll
      for (int i = 0; i < NQ; ++i) {
        const int ad = (a == 0) ? trace_addr(i, ya, yb)
                     : (a == 1) ? trace_addr(ya, i, yb) : trace_addr(ya, yb, i);
        const double v = vec[i];
#pragma unroll
        for (int c = 0; c < M; ++c) qs[c] = fma(v, sQt[(t * M + c) * NS + ad], qs[c]);
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
    if ((tid & 31) == 0) atomicMax(&sSmax[f], v);
  }
  __syncthreads();
  if (tid == 0) {
    bulk_s2g(Dg, sD, NS * M * 8);
    bulk_commit_wait();   // also covers the Q store issued in the corrector
  }
  // ---------------- face records: qbar and fbar traces ----------------
#pragma unroll
  for (int a = 0; a < DIM; ++a) {
    const int pst = (a == 0) ? P0 : (a == 1) ? P1 : 1;
    for (int e = tid; e < 2 * M * NF; e += THREADS) {
      const int side = e / (M * NF);
      const int y = e % NF;
      const int c = (e / NF) % M;
      const double* vec = side ? P.ops.right : P.ops.left;
      const int ya = y / NQ, yb = y % NQ;
      const int pxb = (a == 0) ? ya * P1 + yb : (a == 1) ? ya * P0 + yb : ya * P0 + yb * P1;
      double vq = 0.0, vf = 0.0;
#pragma unroll
      for (int i = 0; i < NQ; ++i) {
        const int ad = (a == 0) ? trace_addr(i, ya, yb)
                     : (a == 1) ? trace_addr(ya, i, yb) : trace_addr(ya, yb, i);
        vq = fma(vec[i], sQb[c * NS + ad], vq);
        vf = fma(vec[i], sFb[(a * M + c) * PS + pxb + i * pst], vf);
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
