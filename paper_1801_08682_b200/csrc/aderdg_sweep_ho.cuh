// aderdg_sweep_ho.cuh — fused sweep kernel of the 3D orders without a dedicated kernel
// (p = 6 and p = 8), and the tensor-memory helpers the dedicated kernels share.
//
//   * 512 threads per cell, each owning NPT = ceil(n^3/512) nodes;
//   * per-node time line (old iterate, divergence history) in thread-private local memory
//     (L1/L2 backed, coalesced); at n <= 8 the first node's old iterate lives in tensor
//     memory instead (tcgen05.alloc of all 512 columns, released before the CTA exits);
//   * the spatial derivatives of a time slice as three GEMMs on the FP64 tensor cores,
//     Out_a[i'][r] = sum_j diff[i'][j] F_a[j][r], r = (the two other node indices,
//     component): A = diff (constant fragments in registers), B = the flux of all three
//     axes staged at once in a padded natural layout, every tile written back in place (a
//     tile's outputs depend only on its own columns): two barriers per slice;
//   * the first Picard iteration (q_t = Q at every level) computes one slice;
//   * the time contraction reads each node's divergence history once per component and
//     forms every time level from registers;
//   * everything else (Riemann, corrector, calc_time_step, final flux, volume integral,
//     face traces, s_max) staged per axis / per time level through one shared node buffer.
// The BASELINE orders p = 3, 5, 7, 9 have their own kernels (aderdg_sweep_p{3,5,7,9}.cuh).
//
// Reference (src/ = /root/reference/pkg/src/aderdg/): kernels.py:68-229,
// scheduler.py:370-449 (same tasks as sweep_kernel).
#pragma once
#include "aderdg_kernels.cuh"
#include "aderdg_sweep_p3.cuh"   // TMA / mbarrier / DMMA helpers

namespace adg {

template <int NQ>
struct ShapeHO {
  static constexpr int DIM = 3, M = 5;
  static constexpr int NS = NQ * NQ * NQ;
  static constexpr int NF = NQ * NQ;
  static constexpr int THREADS = 512;
  static constexpr int NW = THREADS / 32;
  static constexpr int NPT = (NS + THREADS - 1) / THREADS;   // nodes per thread
  static constexpr int KC = (NQ + 3) / 4;                    // k-chunks of m8n8k4
  static constexpr int MT = (NQ + 7) / 8;                    // m-tiles (output positions)
  static constexpr int RR = NF * M;                          // GEMM columns per axis
  static constexpr int NT = (RR + 7) / 8;                    // n-tiles
  static constexpr int RP = NT * 8;
  // padded natural node layout [c][SC]: strides searched against a wavefront model of
  // this kernel's accesses (n = 8: node stores and DMMA B loads conflict-free)
  static constexpr int P1 = (NQ == 10) ? 10 : (NQ == 6) ? 6 : (NQ == 8) ? 12 : 11;
  static constexpr int P0 = (NQ == 6) ? 36 : (NQ == 7) ? 77 : (NQ == 8) ? 100 : (NQ == 9) ? 107 : 111;
  static constexpr int SC = (NQ == 6) ? 217 : (NQ == 7) ? 541 : (NQ == 8) ? 800 : (NQ == 9) ? 965 : 1124;
  static constexpr int REC = 2 * NF * M + 2;
  // TM: the first node's old iterate in tensor memory (measured: a gain at n <= 8 only)
  static constexpr bool TM = (NQ <= 8);
  // shared memory (doubles)
  static constexpr int R_RED = 2 * NW + 2 * DIM + 4;
  static constexpr int R_FA = M * SC;                        // flux of one axis (padded natural layout)
  static constexpr int R_NODE = M * NS;                      // per-node staging (q_t / qbar / fbar_a)
  static constexpr int R_FACE = 2 * DIM * NF * M;
  static constexpr int R_OFF = (3 * RP + 1) / 2;             // int column-offset table (3 axes)
  static constexpr int OFF_RED = 0;
  static constexpr int OFF_TAB = (R_RED + 1) & ~1;
  static constexpr int OFF_FA = OFF_TAB + ((R_OFF + 1) & ~1);
  static constexpr int OFF_NODE = OFF_FA;                    // tail / corrector buffers alias the slabs
  static constexpr int OFF_FACE = OFF_NODE + R_NODE;
  static constexpr int TOTAL = OFF_FA + (3 * R_FA > R_NODE + R_FACE ? 3 * R_FA : R_NODE + R_FACE);
  static constexpr size_t SMEM_BYTES = sizeof(double) * TOTAL;
};



// ---------------------------------------------------------------------------
// Tensor memory (TMEM, 256 KB per SM) as per-thread storage for the Picard
// time line.  tcgen05.ld/st with the 32x32b shape move one 32-bit column per
// thread; warp w owns lanes 32*(w%4).. and, with 16 warps sharing the four lane
// quadrants, columns (w/4)*128 .. +127 of a 512-column allocation: 64 doubles
// per thread.  One CTA per SM (512 threads x 128 registers), so the CTA takes
// the whole TMEM and releases it before it exits.
__device__ __forceinline__ void tmem_alloc_512(uint32_t* dst) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n"
               "tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::"r"(smem_u32(dst))
               : "memory");
}
__device__ __forceinline__ void tmem_dealloc_512(uint32_t t) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(t) : "memory");
}
__device__ __forceinline__ void tmem_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
// one double = two columns; the wait carries the registers as operands so no use
// of a loaded value can be scheduled before the load completes
__device__ __forceinline__ void tmem_ld_d(uint32_t a, uint32_t& lo, uint32_t& hi) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];" : "=r"(lo), "=r"(hi) : "r"(a));
}
__device__ __forceinline__ double tmem_wait_d(uint32_t& lo, uint32_t& hi) {
  asm volatile("tcgen05.wait::ld.sync.aligned;" : "+r"(lo), "+r"(hi)::"memory");
  return __hiloint2double((int)hi, (int)lo);
}
__device__ __forceinline__ void tmem_st_d(uint32_t a, double v) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(a), "r"((uint32_t)__double2loint(v)),
               "r"((uint32_t)__double2hiint(v))
               : "memory");
}
// K doubles at columns base + stride*i (loads issued back to back, one wait)
template <int K>
__device__ __forceinline__ void tmem_ld_doubles(uint32_t base, uint32_t stride, double (&v)[K]) {
  uint32_t lo[K], hi[K];
#pragma unroll
  for (int i = 0; i < K; ++i) tmem_ld_d(base + stride * i, lo[i], hi[i]);
#pragma unroll
  for (int i = 0; i < K; ++i) v[i] = tmem_wait_d(lo[i], hi[i]);
}

template <int NQ>
__global__ void __launch_bounds__(512, 1) sweep_kernel_ho(const SweepParams P) {
  using S = ShapeHO<NQ>;
  constexpr int DIM = 3, M = 5, NS = S::NS, NF = S::NF, NPT = S::NPT, REC = S::REC;
  constexpr int THREADS = S::THREADS, NW = S::NW, KC = S::KC, MT = S::MT, NT = S::NT;
  constexpr int RR = S::RR, SC = S::SC, P0 = S::P0, P1 = S::P1;
  constexpr bool TM = S::TM;

  extern __shared__ __align__(16) double smem[];
  double* sRed = smem + S::OFF_RED;
  unsigned long long* sSmax = reinterpret_cast<unsigned long long*>(sRed + 2 * NW);
  double* sFA = smem + S::OFF_FA;     // [3][M][SC] flux / derivative of the three axes
  double* sN = smem + S::OFF_NODE;    // [M][NS] node staging
  double* sFace = smem + S::OFF_FACE;
  int* sTab = reinterpret_cast<int*>(smem + S::OFF_TAB);   // [axis][RP]: c*SC + ib*sb + ic*sc2
  ADG_DEBUG_POISON();

  DevState* st = P.st;
  if (st->status != 0) return;
  const int mode = P.mode;
  if (mode == MODE_RERUN && !st->rerun_next) return;
  if (mode_corrects(mode) && st->reduce[1] != 0) return;   // a predict pass already failed

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long cell = sweep_cell(P);
  const long long gcell = cell + P.cell_offset;
  const int plane = (int)(cell / P.plane_cells);
  const int rest = (int)(cell % P.plane_cells);
  const long long own_slot = (long long)(plane + 1) * P.plane_cells + rest;
  const int step_idx = mode_corrects(mode) ? st->step + 1 : 0;
  double* Qg = P.Q + cell * (NS * M);
  double* Dg = P.D + cell * (NS * M);

  // nodes of this thread
  int xn[NPT];
  bool an[NPT];
#pragma unroll
  for (int n = 0; n < NPT; ++n) {
    xn[n] = tid + n * THREADS;
    an[n] = xn[n] < NS;
    if (!an[n]) xn[n] = 0;
  }
  auto idx3 = [](int x, int& i0, int& i1, int& i2) {
    i0 = x / (NQ * NQ); i1 = (x / NQ) % NQ; i2 = x % NQ;
  };

  auto pad = [](int i0, int i1, int i2) { return i0 * P0 + i1 * P1 + i2; };
  int pn[NPT];
#pragma unroll
  for (int n = 0; n < NPT; ++n) {
    int a0, a1, a2;
    idx3(xn[n], a0, a1, a2);
    pn[n] = pad(a0, a1, a2);
  }

  double Qx[NPT][M];
#pragma unroll
  for (int n = 0; n < NPT; ++n)
#pragma unroll
    for (int c = 0; c < M; ++c) Qx[n][c] = Qg[xn[n] * M + c];

  if (mode_corrects(mode)) {
    // ------------- Riemann on the 2d faces (kernels.py:147-179), time-collapsed -------------
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
    if (tid == 0) debug_check_records<DIM>(P, st, cell, gcell, own_slot, nb_slot, REC, 2 * NF * M);
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
    // ------------- integrate_face + update (kernels.py:183-214) -------------
    const double scale_old = (mode == MODE_SF_CORRECT) ? st->scale_new : st->scale_old;
#pragma unroll
    for (int n = 0; n < NPT; ++n) {
      if (!an[n]) continue;
      int i[3];
      idx3(xn[n], i[0], i[1], i[2]);
      double Dx[M];
#pragma unroll
      for (int c = 0; c < M; ++c) Dx[c] = Dg[xn[n] * M + c];
#pragma unroll
      for (int a = 0; a < DIM; ++a) {
        const int y = (a == 0) ? i[1] * NQ + i[2] : (a == 1) ? i[0] * NQ + i[2] : i[0] * NQ + i[1];
        const double slo = __dmul_rn(scale_old, P.ops.lift_lo[i[a]]);
        const double shi = __dmul_rn(scale_old, P.ops.lift_hi[i[a]]);
#pragma unroll
        for (int c = 0; c < M; ++c) {
          Dx[c] = __dsub_rn(Dx[c], __dmul_rn(slo, sFace[((2 * a) * NF + y) * M + c]));
          Dx[c] = __dsub_rn(Dx[c], __dmul_rn(shi, sFace[((2 * a + 1) * NF + y) * M + c]));
        }
      }
#pragma unroll
      for (int c = 0; c < M; ++c) Qx[n][c] = __dadd_rn(Qx[n][c], Dx[c]);
      if (P.spike_step >= 0 && step_idx == P.spike_step) {
        const double rho = Qx[n][0];
        const double pr = pressure_exact<DIM>(Qx[n]);
#pragma unroll
        for (int b = 0; b < DIM; ++b) Qx[n][1 + b] = __dmul_rn(Qx[n][1 + b], P.spike_factor);
        double jj = __dmul_rn(Qx[n][1], Qx[n][1]);
#pragma unroll
        for (int b = 1; b < DIM; ++b) jj = __dadd_rn(jj, __dmul_rn(Qx[n][1 + b], Qx[n][1 + b]));
        Qx[n][M - 1] = __dadd_rn(__ddiv_rn(pr, 0.4), __ddiv_rn(__dmul_rn(0.5, jj), rho));
      }
#pragma unroll
      for (int c = 0; c < M; ++c) Qg[xn[n] * M + c] = Qx[n][c];
    }
  }

  if (!mode_predict_only(mode)) {
    // ------------- calc_time_step (kernels.py:216-229) -------------
    bool ok = true;
    double lam = 0.0;
#pragma unroll
    for (int n = 0; n < NPT; ++n) {
      if (!an[n]) continue;
      bool fin = true;
#pragma unroll
      for (int c = 0; c < M; ++c) fin = fin && finite(Qx[n][c]);
      bool adm = false;
      const double l = max_speed_fast<DIM>(Qx[n], 0, DIM, adm);
      ok = ok && fin && adm;
      if (fin && adm) lam = fmax(lam, l);
    }
    if (!__syncthreads_and(ok)) {
      if (tid == 0) report_error(st, 2 * gcell + 0);
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
    for (int n = 0; n < NPT; ++n)
      if (an[n])
#pragma unroll
        for (int c = 0; c < M; ++c) ok = ok && finite(Qx[n][c]);
    if (!__syncthreads_and(ok)) {
      if (tid == 0) report_error(st, 2 * gcell + 1);
      return;
    }
  }

  // ---------------- predictor (kernels.py:68-105) ----------------
  const double dt = (mode == MODE_RERUN) ? st->dt_old : st->dt_new;
  const double scale = (mode == MODE_RERUN) ? st->scale_old : st->scale_new;   // dt / h (SF: dt_new)
  double am = 0.0;
#pragma unroll
  for (int n = 0; n < NPT; ++n)
    if (an[n])
#pragma unroll
      for (int c = 0; c < M; ++c) am = fmax(am, fabs(Qx[n][c]));
  const double tol = 1e-10 * (1.0 + block_max<NW>(am, sRed));
  const int cap = 2 * NQ;

  // constant A fragments: A[i'][j] = diff[i'][j]; lane holds A[mt*8 + g][kc*4 + t4]
  double afr[MT][KC];
  {
    const int g = lane >> 2, t4 = lane & 3;
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
      for (int kc = 0; kc < KC; ++kc) {
        const int ii = mt * 8 + g, jj = kc * 4 + t4;
        afr[mt][kc] = (ii < NQ && jj < NQ) ? P.ops.diff[ii][jj] : 0.0;
      }
  }
  // GEMM column offsets: column r = c*NF + (ib*NQ + ic) of axis a -> padded address
  // of (c, i_a = 0, ib, ic); padded columns clamp to the last real column
  for (int e = tid; e < 3 * S::RP; e += THREADS) {
    const int a = e / S::RP, r = min(e % S::RP, RR - 1);
    const int sb = (a == 0) ? P1 : P0;
    const int sc2 = (a == 2) ? P1 : 1;
    const int c = r / NF, y = r % NF;
    sTab[e] = c * SC + (y / NQ) * sb + (y % NQ) * sc2;
  }
  // per-node time line in thread-private (local) memory
  // (TM: node 0's old iterate is in TMEM; qo holds the others, index n - 1)
  constexpr int QN = TM ? (NPT > 1 ? NPT - 1 : 1) : NPT;
  constexpr int Q0 = TM ? 1 : 0;
  double qo[QN][NQ][M];
  double dh[NPT][NQ][M];                 // divergence history
  int iters = 0;
  bool failed = false;
  // TM: the time line of the thread's first node lives in TMEM, column
  // (c*NQ + t)*2 of the thread's 128-column slice
  __shared__ uint32_t s_tmem;
  uint32_t tq = 0;
  if constexpr (TM) {
    if (warp == 0) tmem_alloc_512(&s_tmem);
    tmem_fence_before();
  }
  __syncthreads();
  if constexpr (TM) {
    tmem_fence_after();
    tq = s_tmem + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * 128);
  }
  auto qo_slice = [&](int n, int k, double (&qq)[M]) {
    if (TM && n == 0) {
      tmem_ld_doubles<M>(tq + 2 * k, 2 * NQ, qq);
    } else {
#pragma unroll
      for (int c = 0; c < M; ++c) qq[c] = qo[n - Q0][k][c];
    }
  };
#pragma unroll 1
  for (int it = 0; it < cap; ++it) {
    // first iteration: q_t = Q at every time level, so its NQ slices are identical —
    // one is computed and its divergence stored for every k
    const int nsl = (it == 0) ? 1 : NQ;
#pragma unroll 1
    for (int k = 0; k < nsl; ++k) {
      double F[NPT][DIM][M];
#pragma unroll
      for (int n = 0; n < NPT; ++n) {
        double qq[M];
        if (it == 0) {
#pragma unroll
          for (int c = 0; c < M; ++c) qq[c] = Qx[n][c];
        } else {
          qo_slice(n, k, qq);
        }
        flux<DIM>(qq, F[n]);
      }
      // stage the flux of all three axes (padded natural layout, one slab per axis)
#pragma unroll
      for (int n = 0; n < NPT; ++n) {
        if (!an[n]) continue;
#pragma unroll
        for (int a = 0; a < DIM; ++a)
#pragma unroll
          for (int c = 0; c < M; ++c) sFA[a * S::R_FA + c * SC + pn[n]] = F[n][a][c];
      }
      __syncthreads();
      for (int item = warp; item < DIM * NT; item += NW) {
        const int a = item / NT, nt = item - a * NT;
        const int sa = (a == 0) ? P0 : (a == 1) ? P1 : 1;
        double* slab = sFA + a * S::R_FA;
        const int* tab = sTab + a * S::RP;
        double cacc[MT][2];
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) { cacc[mt][0] = 0.0; cacc[mt][1] = 0.0; }
        const double* bbase = slab + tab[nt * 8 + (lane >> 2)];
        double bv[KC];
#pragma unroll
        for (int kc = 0; kc < KC; ++kc) bv[kc] = bbase[min(kc * 4 + (lane & 3), NQ - 1) * sa];
        __syncwarp();
#pragma unroll
        for (int kc = 0; kc < KC; ++kc)
#pragma unroll
          for (int mt = 0; mt < MT; ++mt)
            dmma_8x8x4(cacc[mt][0], cacc[mt][1], afr[mt][kc], bv[kc], cacc[mt][0], cacc[mt][1]);
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)
#pragma unroll
          for (int e2 = 0; e2 < 2; ++e2) {
            const int ip = mt * 8 + (lane >> 2);
            const int r = nt * 8 + 2 * (lane & 3) + e2;
            if (ip < NQ && r < RR) slab[tab[r] + ip * sa] = cacc[mt][e2];
          }
      }
      __syncthreads();
#pragma unroll
      for (int n = 0; n < NPT; ++n)
#pragma unroll
        for (int c = 0; c < M; ++c) {
          const double v = (sFA[c * SC + pn[n]] + sFA[S::R_FA + c * SC + pn[n]]) +
                           sFA[2 * S::R_FA + c * SC + pn[n]];
          if (it == 0) {
#pragma unroll
            for (int kk = 0; kk < NQ; ++kk) dh[n][kk][c] = v;
          } else {
            dh[n][k][c] = v;
          }
        }
    }
    // time contraction + Picard update per node
    BitMax bm;
#pragma unroll
    for (int n = 0; n < NPT; ++n) {
#pragma unroll 1
      for (int c = 0; c < M; ++c) {
        // the divergence history of (n, c) is read once; every time level from registers
        double dk[NQ];
#pragma unroll
        for (int k = 0; k < NQ; ++k) dk[k] = dh[n][k][c];
        double ql[NQ];                                   // TM: the old time line of (0, c)
        if (TM && n == 0) {
          if (it > 0) tmem_ld_doubles<NQ>(tq + 2 * NQ * c, 2, ql);
          else {
#pragma unroll
            for (int t = 0; t < NQ; ++t) ql[t] = Qx[n][c];
          }
        }
#pragma unroll
        for (int t = 0; t < NQ; ++t) {
          double acc = 0.0;
#pragma unroll
          for (int k = 0; k < NQ; ++k) acc = fma(P.ops.integ[t][k], dk[k], acc);
          const double qn = Qx[n][c] - scale * acc;
          const double qold = (TM && n == 0) ? ql[t] : (it == 0) ? Qx[n][c] : qo[n - Q0][t][c];
          const double dd = fabs(qn - qold);
          if (an[n]) bm.add(dd);
          if (TM && n == 0) tmem_st_d(tq + 2 * (NQ * c + t), qn);
          else qo[n - Q0][t][c] = qn;
        }
      }
    }
    if constexpr (TM) tmem_wait_st();
    iters = it + 1;
    if (__syncthreads_or(bm.bad())) { failed = true; break; }
    const double delta = block_max<NW>(__longlong_as_double((long long)bm.m), sRed);
    if (delta <= tol) break;
  }

  // final flux: time average fbar (per node, registers) + finiteness
  double fb[NPT][DIM][M];
  double qb[NPT][M];
#pragma unroll
  for (int n = 0; n < NPT; ++n) {
#pragma unroll
    for (int a = 0; a < DIM; ++a)
#pragma unroll
      for (int c = 0; c < M; ++c) fb[n][a][c] = 0.0;
#pragma unroll
    for (int c = 0; c < M; ++c) qb[n][c] = 0.0;
  }
  if (!failed) {
    bool bad = false;
#pragma unroll
    for (int n = 0; n < NPT; ++n) {
#pragma unroll 1
      for (int t = 0; t < NQ; ++t) {
        double F[DIM][M];
        double qt[M];
        qo_slice(n, t, qt);
        flux<DIM>(qt, F);
        const double w = P.ops.w[t];
#pragma unroll
        for (int a = 0; a < DIM; ++a)
#pragma unroll
          for (int c = 0; c < M; ++c) {
            bad |= an[n] && !finite(F[a][c]);
            fb[n][a][c] = fma(w, F[a][c], fb[n][a][c]);
          }
#pragma unroll
        for (int c = 0; c < M; ++c) qb[n][c] = fma(w, qt[c], qb[n][c]);
      }
    }
    failed = __syncthreads_or(bad);
  }
  auto tmem_release = [&]() {
    if constexpr (TM) {
      tmem_fence_before();
      __syncthreads();
      tmem_fence_after();
      if (warp == 0) tmem_dealloc_512(s_tmem);
    }
  };
  if (failed) {
    if (tid == 0) report_error(st, 2 * gcell + 1);
    tmem_release();
    return;
  }
  if (tid == 0) {
    atomicAdd((unsigned long long*)&st->picard_iters, (unsigned long long)iters);
    atomicAdd((unsigned long long*)&st->predicts, 1ull);
    atomicAdd((unsigned long long*)&st->hist[iters < HIST_BINS ? iters : HIST_BINS - 1], 1ull);
  }

  // ---------------- integrate_volume + f̄ traces, one axis at a time ----------------
  double Dv[NPT][M];
#pragma unroll
  for (int n = 0; n < NPT; ++n)
#pragma unroll
    for (int c = 0; c < M; ++c) Dv[n][c] = 0.0;
#pragma unroll 1
  for (int a = 0; a < DIM; ++a) {
    __syncthreads();
#pragma unroll
    for (int n = 0; n < NPT; ++n)
      if (an[n])
#pragma unroll
        for (int c = 0; c < M; ++c)
          sN[c * NS + xn[n]] = (a == 0) ? fb[n][0][c] : (a == 1) ? fb[n][1][c] : fb[n][2][c];
    __syncthreads();
    const int sa = (a == 0) ? NQ * NQ : (a == 1) ? NQ : 1;
#pragma unroll
    for (int n = 0; n < NPT; ++n) {
      if (!an[n]) continue;
      int i[3];
      idx3(xn[n], i[0], i[1], i[2]);
      const int base = xn[n] - i[a] * sa;
#pragma unroll
      for (int c = 0; c < M; ++c) {
        double s = Dv[n][c];
#pragma unroll
        for (int j = 0; j < NQ; ++j) s = fma(P.ops.kvol[i[a]][j], sN[c * NS + base + j * sa], s);
        Dv[n][c] = s;
      }
    }
    // f̄ face traces of axis a (both sides)
    for (int e = tid; e < 2 * NF * M; e += THREADS) {
      // side fastest at n <= 8: the two lanes of a pair read the same line (one
      // wavefront per quad); n = 10 keeps y fastest (measured: the reordered tail
      // changes the register allocation of the whole kernel, 8.55 -> 5.84 TF/s)
      constexpr bool SF = (NQ <= 8);
      const int side = SF ? (e & 1) : e / (NF * M);
      const int y = SF ? (e >> 1) % NF : e % NF;
      const int c = SF ? (e >> 1) / NF : (e / NF) % M;
      const double* vec = side ? P.ops.right : P.ops.left;
      const int ya = y / NQ, yb = y % NQ;
      const int xb = (a == 0) ? ya * NQ + yb : (a == 1) ? ya * NQ * NQ + yb : (ya * NQ + yb) * NQ;
      double v = 0.0;
#pragma unroll
      for (int i = 0; i < NQ; ++i) v = fma(vec[i], sN[c * NS + xb + i * sa], v);
      P.tr_out[((long long)(2 * a + side) * P.slots + own_slot) * REC + NF * M + y * M + c] = v;
    }
  }
  {
    const double sdt = scale;
#pragma unroll
    for (int n = 0; n < NPT; ++n)
      if (an[n])
#pragma unroll
        for (int c = 0; c < M; ++c) Dg[xn[n] * M + c] = Dv[n][c] * sdt;
  }

  // ---------------- q̄ face traces ----------------
  __syncthreads();
#pragma unroll
  for (int n = 0; n < NPT; ++n)
    if (an[n])
#pragma unroll
      for (int c = 0; c < M; ++c) sN[c * NS + xn[n]] = qb[n][c];
  if (tid < 2 * DIM) sSmax[tid] = 0ull;
  __syncthreads();
  for (int e = tid; e < 2 * DIM * NF * M; e += THREADS) {
    constexpr bool SF = (NQ <= 8);
    const int y = SF ? (e >> 1) % NF : e % NF;
    const int ca = SF ? (e >> 1) / NF : 0;
    const int c = SF ? ca % M : (e / NF) % M;
    const int f = SF ? 2 * (ca / M) + (e & 1) : e / (NF * M);
    const int a = f >> 1;
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
    __syncthreads();
#pragma unroll
    for (int n = 0; n < NPT; ++n) {
      double qt[M];
      qo_slice(n, t, qt);
      if (an[n])
#pragma unroll
        for (int c = 0; c < M; ++c) sN[c * NS + xn[n]] = qt[c];
    }
    __syncthreads();
    for (int e = tid; e < 2 * DIM * NF; e += THREADS) {
      constexpr bool SF = (NQ <= 8);
      const int y = SF ? (e >> 1) % NF : e % NF;
      const int f = SF ? 2 * ((e >> 1) / NF) + (e & 1) : e / NF;
      const int a = f >> 1;
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
  tmem_release();   // (its barrier also orders the s_max atomics)
  __syncthreads();
  if (tid < 2 * DIM) {
    double* rec = P.tr_out + ((long long)tid * P.slots + own_slot) * REC;
    rec[2 * NF * M] = __longlong_as_double((long long)sSmax[tid]);
    rec[2 * NF * M + 1] = record_stamp(P);
  }
}

}  // namespace adg
