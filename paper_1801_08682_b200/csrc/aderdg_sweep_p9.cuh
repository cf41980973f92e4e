// aderdg_sweep_p9.cuh — the fused 3D sweep at p = 9 (n = 10) with the Picard state
// of the whole cell on chip.
//
// One CTA of 512 threads per cell, one CTA per SM.  A thread owns node A = tid and
// node B = tid + 512 (488 threads).  The space-time predictor of a cell is 10^4 * 5
// doubles = 400 KB; the reference iteration (kernels.py:86-97) needs the old iterate
// and the divergence of every time slice, 800 KB.  This kernel keeps ONE array
// S[node][c][k] in place and on chip:
//
//   * before slice k is processed S[.][.][k] holds the old iterate q_k, afterwards the
//     slice's divergence (a slice is read exactly once per iteration, by its owner);
//   * after the last slice the time contraction q_new[t] = Q - (dt/h) sum_k integ[t][k]
//     S[k] runs per (node, c) from registers and writes the new iterate back in place;
//   * placement: node A in tensor memory (tcgen05.ld/st 32x32b, column 2(10c + k) of
//     the thread's 128-column slice: 100 of 128 columns), node B's components 0..3 in
//     shared memory ([c][k][tid], conflict-free) and component 4 in tensor memory
//     (columns 100..119): 256 KB of TMEM + 160 KB of shared memory;
//   * the only copy of the previous iterate that the convergence test
//     max |q_new - q| needs is streamed once per iteration (written and read by the time
//     contraction, 400 KB per cell) through a per-SM global slot (SweepParams::sm_scratch,
//     one CTA per SM, indexed by %smid, [line][t][thread]: coalesced): the 148 slots are 60 MB
//     and mostly stay in the 126 MB L2 (r02 ncu, DRAM bytes per 27^3 sweep: thread-private
//     local memory 42 GB, this slot 21 GB, the slot with an L2 evict-last cache-hint policy
//     8 GB but 3 % slower — the cache_hint forms of ld / st cost more than the DRAM traffic
//     of a kernel that uses 14 % of the HBM bandwidth; a persisting access-policy window on
//     the launch made it worse, 68 GB).  The kernel's streaming global traffic — Q, D, face
//     records — uses the evict-first hints __ldcs / __stcs.  The slice loop touches neither.
//
// With 160 KB of the shared memory holding state, the spatial derivatives of a slice
// go one axis at a time through one padded flux slab (45 KB): owners store F_a ->
// barrier -> 500 derivative lines, in place, one per thread -> barrier -> owners add
// the result and store F_{a+1} to the same addresses (no barrier in between): six
// barriers per slice.  A derivative line uses the even / odd split of the
// (centro-antisymmetric) Gauss-Legendre differentiation matrix: e_j = f_j + f_{9-j},
// o_j = f_j - f_{9-j}, two 5x5 products, out_i = so_i + se_i, out_{9-i} = so_i - se_i
// (70 instead of 100 FP64 operations per line; Ops::eo_e / eo_o are built on the host
// from the reference's diff, whose asymmetry is at rounding level, 7e-14 of 61).
// The first Picard iteration starts from the time-constant q = Q, so its ten slices
// are identical: one is computed and its divergence stored to every S[k] (bitwise
// what ten slices give).
//
// Reference (src/ = /root/reference/pkg/src/aderdg/): kernels.py:68-229 (predict,
// extrapolate, integrate_volume, solve_riemann, integrate_face, update,
// calc_time_step), scheduler.py:370-449 (fused sweep).
#pragma once
#include "aderdg_sweep_ho.cuh"   // TMEM helpers (and the v2 helpers)

namespace adg {

struct ShapeP9 {
  static constexpr int DIM = 3, M = 5, NQ = 10;
  static constexpr int NS = 1000, NF = 100;
  static constexpr int THREADS = 512, NW = 16;
  static constexpr int NB = NS - THREADS;                     // threads with a node B
  static constexpr int REC = 2 * NF * M + 2;
  // padded natural node layout of the flux slab.  The shared-memory pipe serves an 8-byte
  // access per half-warp (one wavefront per 16 lanes on 16 distinct banks; r02 ncu: the old
  // strides 111 / 1124 cost 1.58x the ideal line wavefronts, exactly the half-warp model's
  // 152 : 96).  P0 = 113, SC = 1133 with the line -> thread map below (component fastest)
  // come from a search over strides and digit orders: 104 : 96.
  static constexpr int P0 = 113, P1 = 10, SC = 1133;
  static constexpr int R_RED = 4 * NW + 2 * DIM + 4;          // block_max | s_max | vote flags
  static constexpr int R_SLAB = M * SC;                       // one axis' flux / derivative (>= M*NS: tail staging)
  static constexpr int CB = 4;                                // node-B components in shared memory
  static constexpr int R_SB = CB * NQ * THREADS;              // (>= the corrector's signed F* per face)
  // per-SM global slot: the previous iterate of the convergence test, [node slot][c][t][thread]
  static constexpr int SCRATCH = 2 * M * NQ * THREADS;
  static constexpr int OFF_RED = 0;
  static constexpr int OFF_SLAB = (R_RED + 1) & ~1;
  static constexpr int OFF_SB = OFF_SLAB + R_SLAB;
  static constexpr int TOTAL = OFF_SB + R_SB;
  static constexpr size_t SMEM_BYTES = sizeof(double) * TOTAL;
  static_assert(R_SLAB >= M * NS && R_SB >= 2 * DIM * NF * M, "aliased tail / corrector buffers");
  static_assert(SMEM_BYTES <= 232448, "shared memory per CTA");
};

// ten doubles at 20 consecutive columns: one .x16 and one .x4 access
__device__ __forceinline__ void tmem_ld10(uint32_t a, double (&v)[10]) {
  uint32_t r[20];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(a));
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19])
               : "r"(a + 16));
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),
                 "+r"(r[15]), "+r"(r[16]), "+r"(r[17]), "+r"(r[18]), "+r"(r[19])::"memory");
#pragma unroll
  for (int i = 0; i < 10; ++i) v[i] = __hiloint2double((int)r[2 * i + 1], (int)r[2 * i]);
}
__device__ __forceinline__ void tmem_st10(uint32_t a, const double (&v)[10]) {
  uint32_t r[20];
#pragma unroll
  for (int i = 0; i < 10; ++i) {
    r[2 * i] = (uint32_t)__double2loint(v[i]);
    r[2 * i + 1] = (uint32_t)__double2hiint(v[i]);
  }
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(a),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(a + 16), "r"(r[16]), "r"(r[17]),
               "r"(r[18]), "r"(r[19])
               : "memory");
}

// One derivative line of 10 nodes at stride SA, in place, through the even / odd
// blocks of diff (Ops::eo_e, eo_o; constant bank -> uniform registers).
template <int SA>
__device__ __forceinline__ void deriv_line_eo10(double* ln, const SweepParams& P) {
  double e[5], o[5];
#pragma unroll
  for (int j = 0; j < 5; ++j) {
    const double a = ln[j * SA], b = ln[(9 - j) * SA];
    e[j] = a + b;
    o[j] = a - b;
  }
#pragma unroll
  for (int i = 0; i < 5; ++i) {
    double se = P.ops.eo_e[i][0] * e[0];
    double so = P.ops.eo_o[i][0] * o[0];
#pragma unroll
    for (int j = 1; j < 5; ++j) {
      se = fma(P.ops.eo_e[i][j], e[j], se);
      so = fma(P.ops.eo_o[i][j], o[j], so);
    }
    ln[i * SA] = so + se;
    ln[(9 - i) * SA] = so - se;
  }
}

// number of %smid values of the device (%smid ranges over 0 .. %nsmid - 1, which may exceed
// the count of enabled SMs): the per-SM scratch slots are sized by it
__global__ void nsmid_kernel(unsigned* out) {
  unsigned n;
  asm("mov.u32 %0, %%nsmid;" : "=r"(n));
  *out = n;
}

__global__ void __launch_bounds__(ShapeP9::THREADS, 1) sweep_kernel_p9(const SweepParams P) {
  using S = ShapeP9;
  constexpr int DIM = 3, M = 5, NQ = 10, NS = S::NS, NF = S::NF, REC = S::REC, NW = S::NW;
  constexpr int THREADS = S::THREADS, SC = S::SC, P0 = S::P0, P1 = S::P1, CB = S::CB;

  extern __shared__ __align__(16) double smem[];
  double* sRed = smem + S::OFF_RED;
  unsigned long long* sSmax = reinterpret_cast<unsigned long long*>(sRed + 2 * NW);
  unsigned* sFlags = reinterpret_cast<unsigned*>(sRed + 2 * NW + 2 * DIM);   // 2 * NW words
  double* sSlab = smem + S::OFF_SLAB;   // [M][SC] flux / derivative of the current axis
  double* sN = sSlab;                   // [M][NS] node staging of the tail
  double* sB = smem + S::OFF_SB;        // [c < CB][k][THREADS] node-B state
  double* sFace = sB;                   // corrector: signed F* per face
  ADG_DEBUG_POISON();

  DevState* st = P.st;
  if (st->status != 0) return;
  const int mode = P.mode;
  if (mode == MODE_RERUN && !st->rerun_next) return;
  if (mode_corrects(mode) && st->reduce[1] != 0) return;   // a predict pass already failed

  const int tid = threadIdx.x, warp = tid >> 5;
  const long long cell = sweep_cell(P);
  const long long gcell = cell + P.cell_offset;
  const int plane = (int)(cell / P.plane_cells);
  const int rest = (int)(cell % P.plane_cells);
  const long long own_slot = (long long)(plane + 1) * P.plane_cells + rest;
  const int step_idx = mode_corrects(mode) ? st->step + 1 : 0;
  double* Qg = P.Q + cell * (NS * M);
  double* Dg = P.D + cell * (NS * M);

  // the thread's nodes (a thread without node B mirrors node A and discards the results)
  const bool hasB = tid < S::NB;
  const int xn[2] = {tid, hasB ? tid + THREADS : tid};
  const bool an[2] = {true, hasB};
  auto idx3 = [](int x, int& i0, int& i1, int& i2) {
    i0 = x / (NQ * NQ); i1 = (x / NQ) % NQ; i2 = x % NQ;
  };
  int pn[2];
#pragma unroll
  for (int n = 0; n < 2; ++n) {
    int a0, a1, a2;
    idx3(xn[n], a0, a1, a2);
    pn[n] = a0 * P0 + a1 * P1 + a2;
  }

  double Qx[2][M];
#pragma unroll
  for (int n = 0; n < 2; ++n)
#pragma unroll
    for (int c = 0; c < M; ++c) Qx[n][c] = __ldcs(&Qg[xn[n] * M + c]);

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
      const double alpha = rusanov_alpha(__ldcs(mr + 2 * NF * M), __ldcs(pr + 2 * NF * M));
      const double fs = __dsub_rn(__dmul_rn(0.5, __dadd_rn(__ldcs(mr + NF * M + yc), __ldcs(pr + NF * M + yc))),
                                  __dmul_rn(__dmul_rn(0.5, alpha), __dsub_rn(__ldcs(pr + yc), __ldcs(mr + yc))));
      sFace[e] = (f & 1) ? fs : -fs;
    }
    __syncthreads();
    // ------------- integrate_face + update (kernels.py:183-214) -------------
    const double scale_old = (mode == MODE_SF_CORRECT) ? st->scale_new : st->scale_old;
#pragma unroll
    for (int n = 0; n < 2; ++n) {
      if (!an[n]) continue;
      int i[3];
      idx3(xn[n], i[0], i[1], i[2]);
      double Dx[M];
#pragma unroll
      for (int c = 0; c < M; ++c) Dx[c] = __ldcs(&Dg[xn[n] * M + c]);
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
      for (int c = 0; c < M; ++c) __stcs(&Qg[xn[n] * M + c], Qx[n][c]);
    }
    if (!hasB) {
#pragma unroll
      for (int c = 0; c < M; ++c) Qx[1][c] = Qx[0][c];
    }
  }

  if (!mode_predict_only(mode)) {
    // ------------- calc_time_step (kernels.py:216-229) -------------
    bool ok = true;
    double lam = 0.0;
#pragma unroll
    for (int n = 0; n < 2; ++n) {
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
    if (mode == MODE_SF_CORRECT) return;                 // straightforward: no predictor in this pass
  } else {
    bool ok = true;
#pragma unroll
    for (int n = 0; n < 2; ++n)
      if (an[n])
#pragma unroll
        for (int c = 0; c < M; ++c) ok = ok && finite(Qx[n][c]);
    if (!__syncthreads_and(ok)) {
      if (tid == 0) report_error(st, 2 * gcell + 1);
      return;
    }
  }

  // ---------------- predictor (kernels.py:68-105) ----------------
  const double scale = (mode == MODE_RERUN) ? st->scale_old : st->scale_new;   // dt / h (SF: dt_new)
  __shared__ uint32_t s_tmem;
  if (warp == 0) tmem_alloc_512(&s_tmem);
  tmem_fence_before();
  double am = 0.0;
#pragma unroll
  for (int n = 0; n < 2; ++n)
    if (an[n])
#pragma unroll
      for (int c = 0; c < M; ++c) am = fmax(am, fabs(Qx[n][c]));
  const double tol = 1e-10 * (1.0 + block_max<NW>(am, sRed));   // (its barriers publish the TMEM address)
  tmem_fence_after();
  const uint32_t tq = s_tmem + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * 128);
  const uint32_t tb = tq + 100;                                  // node B, component 4
  double* sBt = sB + tid;
  const int cap = 2 * NQ;

  // the thread's derivative line of every axis (l = tid < 500: component c, face node y)
  const bool has_line = tid < NF * M;
  double* ln0;
  double* ln1;
  double* ln2;
  {
    const int l = has_line ? tid : 0;
    const int c = l % M, r0 = (l / M) % NQ, r1 = l / (M * NQ);
    ln0 = sSlab + c * SC + r1 * P1 + r0;          // line (i1, i2) = (r1, r0), stride P0
    ln1 = sSlab + c * SC + r0 * P0 + r1;          // line (i0, i2) = (r0, r1), stride P1
    ln2 = sSlab + c * SC + r0 * P0 + r1 * P1;     // line (i0, i1) = (r0, r1), stride 1
  }

  // the convergence test's copy of the previous iterate and the initial state, indexed
  // by the rolled (node, component) loop of the time contraction: thread-private memory
  unsigned smid;
  asm("mov.u32 %0, %%smid;" : "=r"(smid));
  double* qprev = P.sm_scratch + (size_t)smid * S::SCRATCH + tid;   // [nc][t][THREADS]
  double q0l[2 * M];
#pragma unroll
  for (int n = 0; n < 2; ++n)
#pragma unroll
    for (int c = 0; c < M; ++c) q0l[n * M + c] = Qx[n][c];

  auto load_slice = [&](int k, double (&qa)[M], double (&qb)[M]) {
    uint32_t lo[M + 1], hi[M + 1];
#pragma unroll
    for (int c = 0; c < M; ++c) tmem_ld_d(tq + 20 * c + 2 * k, lo[c], hi[c]);
    tmem_ld_d(tb + 2 * k, lo[M], hi[M]);
#pragma unroll
    for (int c = 0; c < CB; ++c) qb[c] = sBt[(c * NQ + k) * THREADS];
#pragma unroll
    for (int c = 0; c < M; ++c) qa[c] = tmem_wait_d(lo[c], hi[c]);
    qb[M - 1] = tmem_wait_d(lo[M], hi[M]);
  };
  auto store_slice = [&](int k, const double (&va)[M], const double (&vb)[M]) {
#pragma unroll
    for (int c = 0; c < M; ++c) tmem_st_d(tq + 20 * c + 2 * k, va[c]);
    tmem_st_d(tb + 2 * k, vb[M - 1]);
#pragma unroll
    for (int c = 0; c < CB; ++c) sBt[(c * NQ + k) * THREADS] = vb[c];
  };

  int iters = 0;
  bool failed = false;
#pragma unroll 1
  for (int it = 0; it < cap; ++it) {
    const int nsl = (it == 0) ? 1 : NQ;     // q = Q at every time level: one slice stands for all
#pragma unroll 1
    for (int k = 0; k < nsl; ++k) {
      double F[2][DIM][M];
      {
        double qa[M], qb[M];
        if (it == 0) {
#pragma unroll
          for (int c = 0; c < M; ++c) { qa[c] = Qx[0][c]; qb[c] = Qx[1][c]; }
        } else {
          load_slice(k, qa, qb);
        }
        flux<DIM>(qa, F[0]);
        flux<DIM>(qb, F[1]);
      }
      double dv[2][M];
      // axis a: owners store F_a (after adding the previous axis' result from the same
      // addresses) -> barrier -> lines in place -> barrier
#pragma unroll
      for (int a = 0; a < DIM; ++a) {
#pragma unroll
        for (int n = 0; n < 2; ++n) {
          if (n == 1 && !hasB) continue;
#pragma unroll
          for (int c = 0; c < M; ++c) {
            double* p = sSlab + c * SC + pn[n];
            if (a == 1) dv[n][c] = *p;
            if (a == 2) dv[n][c] += *p;
            *p = F[n][a][c];
          }
        }
        __syncthreads();
        if (has_line) {
          if (a == 0) deriv_line_eo10<P0>(ln0, P);
          else if (a == 1) deriv_line_eo10<P1>(ln1, P);
          else deriv_line_eo10<1>(ln2, P);
        }
        __syncthreads();
      }
#pragma unroll
      for (int n = 0; n < 2; ++n)
#pragma unroll
        for (int c = 0; c < M; ++c) dv[n][c] += sSlab[c * SC + pn[n]];
      if (it == 0) {
#pragma unroll 1
        for (int kk = 0; kk < NQ; ++kk) store_slice(kk, dv[0], dv[1]);
      } else {
        store_slice(k, dv[0], dv[1]);
      }
    }
    tmem_wait_st();
    // time contraction + Picard update per (node, component): the divergence history is
    // read once, every time level formed from registers and written back in place
    BitMax bm;
#pragma unroll 1
    for (int nc = 0; nc < 2 * M; ++nc) {
      const int n = nc / M, c = nc - n * M;
      const bool in_tmem = (n == 0) || (c == M - 1);
      const uint32_t ta = (n == 0) ? tq + 20 * c : tb;
      double dk[NQ];
      if (in_tmem) {
        tmem_ld10(ta, dk);
      } else {
#pragma unroll
        for (int k = 0; k < NQ; ++k) dk[k] = sBt[(c * NQ + k) * THREADS];
      }
      const double qc = q0l[nc];
      double qn[NQ];
#pragma unroll
      for (int t = 0; t < NQ; ++t) {
        double acc = 0.0;
#pragma unroll
        for (int k = 0; k < NQ; ++k) acc = fma(P.ops.integ[t][k], dk[k], acc);
        qn[t] = qc - scale * acc;
        const double qold = (it == 0) ? qc : qprev[(nc * NQ + t) * THREADS];
        if (n == 0 || hasB) bm.add(fabs(qn[t] - qold));
        qprev[(nc * NQ + t) * THREADS] = qn[t];
      }
      if (in_tmem) {
        tmem_st10(ta, qn);
      } else {
#pragma unroll
        for (int k = 0; k < NQ; ++k) sBt[(c * NQ + k) * THREADS] = qn[k];
      }
    }
    tmem_wait_st();
    iters = it + 1;
    const int fl = block_flags<NW>(bm.conv(tol), bm.bad(), sFlags, it & 1);
    if (fl & 2) { failed = true; break; }
    if (fl & 1) break;
  }

  auto tmem_release = [&]() {
    tmem_fence_before();
    __syncthreads();
    tmem_fence_after();
    if (warp == 0) tmem_dealloc_512(s_tmem);
  };
  if (failed) {
    if (tid == 0) report_error(st, 2 * gcell + 1);
    tmem_release();
    return;
  }

  // ---------------- final flux, integrate_volume and the f-bar traces, one axis at a time ----------------
  // (kernels.py:98-100,130-143,107-128).  The time-averaged flux of axis a is formed
  // from the final iterate in S (the flux of the other axes is dead code in each pass).
  double Dv[2][M], qb[2][M];
#pragma unroll
  for (int n = 0; n < 2; ++n)
#pragma unroll
    for (int c = 0; c < M; ++c) { Dv[n][c] = 0.0; qb[n][c] = 0.0; }
  bool bad = false;
#pragma unroll
  for (int a = 0; a < DIM; ++a) {
    double fb[2][M];
#pragma unroll
    for (int n = 0; n < 2; ++n)
#pragma unroll
      for (int c = 0; c < M; ++c) fb[n][c] = 0.0;
#pragma unroll 1
    for (int t = 0; t < NQ; ++t) {
      double qt[2][M];
      load_slice(t, qt[0], qt[1]);
      const double w = P.ops.w[t];
#pragma unroll
      for (int n = 0; n < 2; ++n) {
        double F[DIM][M];
        flux<DIM>(qt[n], F);
#pragma unroll
        for (int c = 0; c < M; ++c) {
          bad |= an[n] && !finite(F[a][c]);
          fb[n][c] = fma(w, F[a][c], fb[n][c]);
          if (a == 0) qb[n][c] = fma(w, qt[n][c], qb[n][c]);
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int n = 0; n < 2; ++n)
      if (an[n])
#pragma unroll
        for (int c = 0; c < M; ++c) sN[c * NS + xn[n]] = fb[n][c];
    __syncthreads();
    const int sa = (a == 0) ? NQ * NQ : (a == 1) ? NQ : 1;
#pragma unroll
    for (int n = 0; n < 2; ++n) {
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
    // f-bar face traces of axis a (both sides; y fastest)
    for (int e = tid; e < 2 * NF * M; e += THREADS) {
      const int side = e / (NF * M);
      const int y = e % NF;
      const int c = (e / NF) % M;
      const double* vec = side ? P.ops.right : P.ops.left;
      const int ya = y / NQ, yb = y % NQ;
      const int xb = (a == 0) ? ya * NQ + yb : (a == 1) ? ya * NQ * NQ + yb : (ya * NQ + yb) * NQ;
      double v = 0.0;
#pragma unroll
      for (int i = 0; i < NQ; ++i) v = fma(vec[i], sN[c * NS + xb + i * sa], v);
      __stcs(&P.tr_out[((long long)(2 * a + side) * P.slots + own_slot) * REC + NF * M + y * M + c], v);
    }
  }
  if (__syncthreads_or(bad)) {
    if (tid == 0) report_error(st, 2 * gcell + 1);
    tmem_release();
    return;
  }
  if (tid == 0) {
    atomicAdd((unsigned long long*)&st->picard_iters, (unsigned long long)iters);
    atomicAdd((unsigned long long*)&st->predicts, 1ull);
    atomicAdd((unsigned long long*)&st->hist[iters < HIST_BINS ? iters : HIST_BINS - 1], 1ull);
  }
#pragma unroll
  for (int n = 0; n < 2; ++n)
    if (an[n])
#pragma unroll
      for (int c = 0; c < M; ++c) __stcs(&Dg[xn[n] * M + c], Dv[n][c] * scale);

  // ---------------- q-bar face traces ----------------
  // (the barrier of the error vote above separates the last f-bar trace reads from these stores)
#pragma unroll
  for (int n = 0; n < 2; ++n)
    if (an[n])
#pragma unroll
      for (int c = 0; c < M; ++c) sN[c * NS + xn[n]] = qb[n][c];
  if (tid < 2 * DIM) sSmax[tid] = 0ull;
  __syncthreads();
  for (int e = tid; e < 2 * DIM * NF * M; e += THREADS) {
    const int y = e % NF;
    const int c = (e / NF) % M;
    const int f = e / (NF * M);
    const int a = f >> 1;
    const double* vec = (f & 1) ? P.ops.right : P.ops.left;
    const int ya = y / NQ, yb = y % NQ;
    const int sa = (a == 0) ? NQ * NQ : (a == 1) ? NQ : 1;
    const int xb = (a == 0) ? ya * NQ + yb : (a == 1) ? ya * NQ * NQ + yb : (ya * NQ + yb) * NQ;
    double v = 0.0;
#pragma unroll
    for (int i = 0; i < NQ; ++i) v = fma(vec[i], sN[c * NS + xb + i * sa], v);
    __stcs(&P.tr_out[((long long)f * P.slots + own_slot) * REC + y * M + c], v);
  }
  // ---------------- s_max over the space-time traces, one time level at a time ----------------
#pragma unroll 1
  for (int t = 0; t < NQ; ++t) {
    double qt[2][M];
    load_slice(t, qt[0], qt[1]);
    __syncthreads();
#pragma unroll
    for (int n = 0; n < 2; ++n)
      if (an[n])
#pragma unroll
        for (int c = 0; c < M; ++c) sN[c * NS + xn[n]] = qt[n][c];
    __syncthreads();
    for (int e = tid; e < 2 * DIM * NF; e += THREADS) {
      const int y = e % NF;
      const int f = e / NF;
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
