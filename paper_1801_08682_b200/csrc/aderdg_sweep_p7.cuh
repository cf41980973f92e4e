// aderdg_sweep_p7.cuh — the fused 3D sweep at p = 7 (n = 8) with the whole Picard
// state of the cell on chip and the derivatives as exact m8n8k4 DMMA tiles.
//
// One CTA of 512 threads per cell (thread = spatial node), one CTA per SM.
//   * Picard state: the node's time line q[c][t] (40 doubles) and the divergence
//     history dv[c][k] (40 doubles) never touch local memory: q and dv of components
//     0..2 live in tensor memory (128 columns = 64 doubles per thread, tcgen05.ld/st
//     32x32b), dv of components 3, 4 in shared memory ([c][k][tid], conflict free).
//   * derivatives: per time slice three GEMMs Out_a[i][col] = sum_j diff[i][j] F_a[j][col],
//     col = c*64 + (the two other node indices): 40 n-tiles of 8 columns per axis, K = 8
//     = two m8n8k4 DMMAs per tile with no padding.  A = diff (constant fragments), B = the
//     flux from shared memory [j][axis][col]; a tile writes its 8 x 8 outputs back in
//     place (its outputs depend only on its own columns), the node owner sums the axes.
//   * bank layout: row stride 964 == 4 (mod 16) puts the four k rows of a B-fragment load on
//     disjoint bank groups (2 wavefronts, the minimum for 256 bytes); the A rows are
//     permuted (0,2,1,3,4,6,5,7) so that the two output rows a quarter-warp stores as
//     16-byte pairs lie 2 rows = 64 bytes (mod 128) apart (4 wavefronts, the minimum);
//     a half-warp owns a 2 x 2 x 4 node box, so its 8-byte owner stores / loads fall on 16
//     distinct banks along all three axes (the pipe serves 8-byte accesses per half-warp).
//   * time contraction k-outermost over groups of 3 + 2 components: FP64 instructions take
//     no constant operand, so every integ[t][k] fetched feeds 3 (2) FMAs.
//   * software-pipelined slices, one barrier per slice: the interval that runs the tiles
//     of slice k (operand buffer k & 1) also stages the flux of slice k + 1 in the other
//     buffer (its last tile readers passed the previous barrier; an owner reads back and
//     rewrites only its own addresses, in program order).  The flux of the next
//     iteration's slice 0 is staged before the convergence vote, whose barrier
//     publishes it.
//   * the first Picard iteration starts from q_t = Q at every time level, so its eight
//     slices are identical: one is computed and its divergence stored for every k.
//
// Everything else (Riemann, corrector, calc_time_step, final flux, volume integral,
// face traces, s_max) follows sweep_kernel_ho.
//
// Reference (src/ = /root/reference/pkg/src/aderdg/): kernels.py:68-229 (predict,
// extrapolate, integrate_volume, solve_riemann, integrate_face, update,
// calc_time_step), scheduler.py:370-449 (fused sweep).
#pragma once
#include <type_traits>
#include "aderdg_sweep_p5.cuh"   // dmma_nv, TMEM helpers

namespace adg {

struct ShapeP7 {
  static constexpr int DIM = 3, M = 5, NQ = 8;
  static constexpr int NS = 512, NF = 64;
  static constexpr int THREADS = 512, NW = 16;
  static constexpr int REC = 2 * NF * M + 2;
  // DMMA operand arrays [slice parity][j][axis][NCOL] (+ 4 pad doubles per row): tile t of the
  // slice (t = axis * 40 + n-tile) starts at column 8 t of every row
  static constexpr int NCOL = M * NF, NTILE = NCOL / 8;
  static constexpr int STR = DIM * NCOL + 4;
  static constexpr int FBUF = NQ * STR;
  static constexpr int TILES = DIM * NTILE;
  static constexpr int R_PRED = 2 * FBUF;
  static constexpr int CS = 2;                               // dv components in shared memory (3, 4)
  static constexpr int R_DV = CS * NQ * THREADS;
  // node staging of the tail: node (i0, i1, i2) at 72 i0 + 9 i1 + i2 (the face-trace gathers
  // of a half-warp then fall on distinct banks along all three axes)
  static constexpr int T1 = NQ + 1, T0 = NQ * T1, NSP = NQ * T0;
  static constexpr int R_NODE = M * NSP;
  static constexpr int R_FACE = 2 * DIM * NF * M;            // corrector: signed F* per face
  static constexpr int R_RED = 4 * NW + 2 * DIM + 4;         // block_max | s_max | vote flags
  static constexpr int OFF_RED = 0;
  static constexpr int OFF_U = (R_RED + 1) & ~1;
  static constexpr int OFF_DV = OFF_U + R_PRED;
  static constexpr int TOTAL = OFF_DV + R_DV;
  static constexpr size_t SMEM_BYTES = sizeof(double) * TOTAL;
  static_assert(R_PRED >= R_NODE && R_PRED >= R_FACE, "aliased tail / corrector buffers");
  static_assert(NCOL % 16 == 0 && STR % 16 == 4, "operand row layout");
  static_assert(SMEM_BYTES <= 232448, "shared memory per CTA");
};

// eight doubles at 16 consecutive columns: one .x16 access
__device__ __forceinline__ void tmem_ld8(uint32_t a, double (&v)[8]) {
  uint32_t r[16];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(a));
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11]), "+r"(r[12]), "+r"(r[13]), "+r"(r[14]),
                 "+r"(r[15])::"memory");
#pragma unroll
  for (int i = 0; i < 8; ++i) v[i] = __hiloint2double((int)r[2 * i + 1], (int)r[2 * i]);
}
__device__ __forceinline__ void tmem_st8(uint32_t a, const double (&v)[8]) {
  uint32_t r[16];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    r[2 * i] = (uint32_t)__double2loint(v[i]);
    r[2 * i + 1] = (uint32_t)__double2hiint(v[i]);
  }
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};" ::"r"(a),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
      : "memory");
}

// three doubles at 6 consecutive columns (one .x4 and one .x2 access), issue and wait apart
__device__ __forceinline__ void tmem_ld3_issue(uint32_t a, uint32_t (&r)[6]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(a));
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];" : "=r"(r[4]), "=r"(r[5]) : "r"(a + 4));
}
__device__ __forceinline__ void tmem_ld3_wait(uint32_t (&r)[6], double (&v)[3]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5])::"memory");
#pragma unroll
  for (int i = 0; i < 3; ++i) v[i] = __hiloint2double((int)r[2 * i + 1], (int)r[2 * i]);
}
__device__ __forceinline__ void tmem_st3(uint32_t a, double v0, double v1, double v2) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(a),
               "r"((uint32_t)__double2loint(v0)), "r"((uint32_t)__double2hiint(v0)),
               "r"((uint32_t)__double2loint(v1)), "r"((uint32_t)__double2hiint(v1))
               : "memory");
  asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1,%2};" ::"r"(a + 4),
               "r"((uint32_t)__double2loint(v2)), "r"((uint32_t)__double2hiint(v2))
               : "memory");
}

__global__ void __launch_bounds__(ShapeP7::THREADS, 1) sweep_kernel_p7(const SweepParams P) {
  using S = ShapeP7;
  constexpr int DIM = 3, M = 5, NQ = 8, NS = S::NS, NF = S::NF, REC = S::REC, NW = S::NW;
  constexpr int THREADS = S::THREADS, STR = S::STR, NCOL = S::NCOL, FBUF = S::FBUF, CS = S::CS;

  extern __shared__ __align__(16) double smem[];
  double* sRed = smem + S::OFF_RED;
  unsigned long long* sSmax = reinterpret_cast<unsigned long long*>(sRed + 2 * NW);
  unsigned* sFlags = reinterpret_cast<unsigned*>(sRed + 2 * NW + 2 * DIM);   // 2 * NW words
  double* sU = smem + S::OFF_U;         // operand buffers of the Picard loop
  double* sFace = sU;                   // corrector: signed F* per face
  double* sN = sU;                      // [M][NSP] node staging of the tail (padded)
  double* sDv = smem + S::OFF_DV;       // [c - 3][k][tid] divergence history of components 3, 4
  ADG_DEBUG_POISON();

  DevState* st = P.st;
  if (st->status != 0) return;
  const int mode = P.mode;
  if (mode == MODE_RERUN && !st->rerun_next) return;
  if (mode_corrects(mode) && st->reduce[1] != 0) return;   // a predict pass already failed

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // Thread -> node map: a half-warp owns a 2 x 2 x 4 node box (lane bits 0-1: i2 & 3, bit 2:
  // i0 & 1, bit 3: i1 & 1), lane bit 4 selects i2 >= 4, the warp index holds i0 / 2 and
  // i1 / 2.  The shared-memory pipe serves an 8-byte access per half-warp: with the operand
  // rows at bank offsets 4 i_a (STR == 4 mod 16) the 16 owner addresses of a half-warp fall
  // on 16 distinct banks along all three axes (axis 2 with the column map below).
  const int i0 = 2 * (warp >> 2) + ((lane >> 2) & 1);
  const int i1 = 2 * (warp & 3) + ((lane >> 3) & 1);
  const int i2 = (lane & 3) | ((lane >> 4) << 2);
  const int x = (i0 * NQ + i1) * NQ + i2;
  const int xp = i0 * S::T0 + i1 * S::T1 + i2;       // padded node index of the tail staging
  const long long cell = sweep_cell(P);
  const long long gcell = cell + P.cell_offset;
  const int plane = (int)(cell / P.plane_cells);
  const int rest = (int)(cell % P.plane_cells);
  const long long own_slot = (long long)(plane + 1) * P.plane_cells + rest;
  const int step_idx = mode_corrects(mode) ? st->step + 1 : 0;
  double* Qg = P.Q + cell * (NS * M);
  double* Dg = P.D + cell * (NS * M);

  double Qx[M];
#pragma unroll
  for (int c = 0; c < M; ++c) Qx[c] = Qg[x * M + c];

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
    {
      const int i[3] = {i0, i1, i2};
      double Dx[M];
#pragma unroll
      for (int c = 0; c < M; ++c) Dx[c] = Dg[x * M + c];
#pragma unroll
      for (int a = 0; a < DIM; ++a) {
        const int y = (a == 0) ? i1 * NQ + i2 : (a == 1) ? i0 * NQ + i2 : i0 * NQ + i1;
        const double slo = __dmul_rn(scale_old, P.ops.lift_lo[i[a]]);
        const double shi = __dmul_rn(scale_old, P.ops.lift_hi[i[a]]);
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
      for (int c = 0; c < M; ++c) Qg[x * M + c] = Qx[c];
    }
  }

  if (!mode_predict_only(mode)) {
    // ------------- calc_time_step (kernels.py:216-229) -------------
    bool fin = true;
#pragma unroll
    for (int c = 0; c < M; ++c) fin = fin && finite(Qx[c]);
    bool adm = false;
    double lam = max_speed_fast<DIM>(Qx, 0, DIM, adm);
    const bool ok = fin && adm;
    if (!ok) lam = 0.0;
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
    for (int c = 0; c < M; ++c) ok = ok && finite(Qx[c]);
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
  for (int c = 0; c < M; ++c) am = fmax(am, fabs(Qx[c]));
  // (the barriers of block_max publish the TMEM address and retire the corrector's
  //  reads of sFace, which the operand buffers alias)
  const double tol = 1e-10 * (1.0 + block_max<NW>(am, sRed));
  tmem_fence_after();
  // warp w: TMEM lanes 32 (w % 4).., columns 128 (w / 4)..: q[c][t] at column 2 (8c + t),
  // dv[k][c] (c < 3) at column 80 + 2 (3k + c)
  const uint32_t tq = s_tmem + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)((warp >> 2) * 128);
  const uint32_t td = tq + 80;
  double* sDt = sDv + tid;
  const int cap = 2 * NQ;

  // DMMA A fragments: lane = (row << 2) | k holds diff[pi(row)][k], diff[pi(row)][k + 4];
  // pi = (0,2,1,3,4,6,5,7) spreads the output rows of a quarter-warp 64 bytes apart
  const int fr = lane >> 2, fk = lane & 3;
  const int prow = (fr & 4) | ((fr & 1) << 1) | ((fr >> 1) & 1);
  const double a_lo = P.ops.diff[prow][fk];
  const double a_hi = P.ops.diff[prow][fk + 4];
  // lane offsets inside a tile: B rows k / k + 4 at column n = fr; D row pi(fr), columns 2k, 2k + 1
  const int lb0 = fk * STR + fr, lb1 = (fk + 4) * STR + fr, lbd = prow * STR + 2 * fk;
  // owner offsets into one slice buffer: axis a, row i_a, column (other two indices) (+ c * 64)
  // (axis 2: column (i0 & 1) + 2 (i1 & 1) + 4 (i0 / 2) + 16 (i1 / 2) — the GEMM columns are
  //  independent, any bijection of (i0, i1) onto 0..63 will do)
  const int ow[3] = {0 * NCOL + i0 * STR + i1 * NQ + i2, 1 * NCOL + i1 * STR + i0 * NQ + i2,
                     2 * NCOL + i2 * STR + (i0 & 1) + 2 * (i1 & 1) + 4 * (i0 >> 1) + 16 * (i1 >> 1)};

#pragma unroll
  for (int c = 0; c < M; ++c) {
    double qc[NQ];
#pragma unroll
    for (int t = 0; t < NQ; ++t) qc[t] = Qx[c];
    tmem_st8(tq + 16 * c, qc);
  }
  tmem_wait_st();

  auto stage_flux = [&](int k, const double (&qk)[M]) {
    double* B = sU + (k & 1) * FBUF;
    double F[DIM][M];
    flux<DIM>(qk, F);
#pragma unroll
    for (int a = 0; a < DIM; ++a)
#pragma unroll
      for (int c = 0; c < M; ++c) B[ow[a] + c * NF] = F[a][c];
  };
  // Out_a = diff . F_a, in place: warp w takes tiles w, w + 16, ... of the 120 (constant
  // offsets from one base address)
  auto run_tiles = [&](int k) {
    double* base0 = sU + (k & 1) * FBUF + warp * 8;
#pragma unroll
    for (int i = 0; i < (S::TILES + NW - 1) / NW; ++i) {
      if (i * NW + NW > S::TILES && warp + i * NW >= S::TILES) break;
      double* base = base0 + i * NW * 8;
      const double b0 = base[lb0];
      const double b1 = base[lb1];
      double d0, d1;
      dmma_nv(d0, d1, a_lo, b0, 0.0, 0.0);
      dmma_nv(d0, d1, a_hi, b1, d0, d1);
      *reinterpret_cast<double2*>(base + lbd) = make_double2(d0, d1);
    }
  };
  // the node's divergence of slice k: components 0..2 to TMEM, 3..4 to shared memory;
  // the first iteration's slice stands for every k
  auto read_back = [&](int k, bool every_k) {
    const double* B = sU + (k & 1) * FBUF;
    double dvc[M];
#pragma unroll
    for (int c = 0; c < M; ++c) dvc[c] = (B[ow[0] + c * NF] + B[ow[1] + c * NF]) + B[ow[2] + c * NF];
    if (every_k) {
#pragma unroll
      for (int kk = 0; kk < NQ; ++kk) {
        tmem_st3(td + 6 * kk, dvc[0], dvc[1], dvc[2]);
#pragma unroll
        for (int c = M - CS; c < M; ++c) sDt[((c - (M - CS)) * NQ + kk) * THREADS] = dvc[c];
      }
    } else {
      tmem_st3(td + 6 * k, dvc[0], dvc[1], dvc[2]);
#pragma unroll
      for (int c = M - CS; c < M; ++c) sDt[((c - (M - CS)) * NQ + k) * THREADS] = dvc[c];
    }
  };
  // Time contraction + Picard update (kernels.py:86-97) of NC components at a time, k
  // outermost: every integ[t][k] is fetched from the constant bank once per group (FP64
  // instructions take no constant operand), the accumulators become the new time line in
  // place; convergence from the bit patterns of |q_new - q|.
  BitMax bm;
  auto contract = [&](auto c0_, auto nc_) {
    constexpr int C0 = decltype(c0_)::value, NC = decltype(nc_)::value;
    double acc[NC][NQ];
    uint32_t rr[6];
    if (C0 == 0) tmem_ld3_issue(td, rr);
#pragma unroll
    for (int k = 0; k < NQ; ++k) {
      double d[3];
      if (C0 == 0) {
        tmem_ld3_wait(rr, d);
        if (k + 1 < NQ) tmem_ld3_issue(td + 6 * (k + 1), rr);
      } else {
#pragma unroll
        for (int c = 0; c < NC; ++c) d[c] = sDt[((C0 + c - (M - CS)) * NQ + k) * THREADS];
      }
#pragma unroll
      for (int t = 0; t < NQ; ++t) {
        const double g = P.ops.integ[t][k];
#pragma unroll
        for (int c = 0; c < NC; ++c) acc[c][t] = (k == 0) ? g * d[c] : fma(g, d[c], acc[c][t]);
      }
    }
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      double qo[NQ];
      tmem_ld8(tq + 16 * (C0 + c), qo);
#pragma unroll
      for (int t = 0; t < NQ; ++t) {
        acc[c][t] = Qx[C0 + c] - scale * acc[c][t];
        bm.add(fabs(acc[c][t] - qo[t]));
      }
      tmem_st8(tq + 16 * (C0 + c), acc[c]);
    }
  };

  int iters = 0;
  bool failed = false;
  stage_flux(0, Qx);
  __syncthreads();
#pragma unroll 1
  for (int it = 0; it < cap; ++it) {
    if (it == 0) {
      run_tiles(0);
      __syncthreads();
      read_back(0, true);
    } else {
#pragma unroll
      for (int k = 0; k < NQ; ++k) {
        if (k + 1 < NQ) {
          double qk[M];
          tmem_ld_doubles<M>(tq + 2 * (k + 1), 16, qk);
          stage_flux(k + 1, qk);
        }
        run_tiles(k);
        __syncthreads();
        read_back(k, false);
      }
    }
    tmem_wait_st();
    bm = BitMax();
    contract(std::integral_constant<int, 0>(), std::integral_constant<int, 3>());
    contract(std::integral_constant<int, 3>(), std::integral_constant<int, 2>());
    tmem_wait_st();
    iters = it + 1;
    if (it + 1 < cap) {                          // slice 0 of the next iteration
      double q0n[M];
      tmem_ld_doubles<M>(tq, 16, q0n);
      stage_flux(0, q0n);
    }
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

  // final flux: time average fbar and qbar (per node, registers) + finiteness
  double fb[DIM][M], qb[M];
#pragma unroll
  for (int c = 0; c < M; ++c) {
    qb[c] = 0.0;
#pragma unroll
    for (int a = 0; a < DIM; ++a) fb[a][c] = 0.0;
  }
  bool bad = false;
#pragma unroll 2
  for (int t = 0; t < NQ; ++t) {
    double qt[M], F[DIM][M];
    tmem_ld_doubles<M>(tq + 2 * t, 16, qt);
    flux<DIM>(qt, F);
    const double w = P.ops.w[t];
#pragma unroll
    for (int c = 0; c < M; ++c) {
#pragma unroll
      for (int a = 0; a < DIM; ++a) {
        bad |= !finite(F[a][c]);
        fb[a][c] = fma(w, F[a][c], fb[a][c]);
      }
      qb[c] = fma(w, qt[c], qb[c]);
    }
  }
  // (this barrier also retires the last speculative stage_flux stores into sU = sN)
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

  // ---------------- integrate_volume + f-bar traces, one axis at a time ----------------
  // (kernels.py:130-143,107-128)
  double Dv[M];
#pragma unroll
  for (int c = 0; c < M; ++c) Dv[c] = 0.0;
#pragma unroll
  for (int a = 0; a < DIM; ++a) {
    if (a > 0) __syncthreads();
#pragma unroll
    for (int c = 0; c < M; ++c) sN[c * S::NSP + xp] = fb[a][c];
    __syncthreads();
    const int sa = (a == 0) ? S::T0 : (a == 1) ? S::T1 : 1;
    const int ia = (a == 0) ? i0 : (a == 1) ? i1 : i2;
    const int base = xp - ia * sa;
#pragma unroll
    for (int c = 0; c < M; ++c) {
      double s = Dv[c];
#pragma unroll
      for (int j = 0; j < NQ; ++j) s = fma(P.ops.kvol[ia][j], sN[c * S::NSP + base + j * sa], s);
      Dv[c] = s;
    }
    // f-bar face traces of axis a, both sides (side fastest: the two lanes of a pair
    // read the same line)
    for (int e = tid; e < 2 * NF * M; e += THREADS) {
      const int side = e & 1;
      const int y = (e >> 1) % NF;
      const int c = (e >> 1) / NF;
      const double* vec = side ? P.ops.right : P.ops.left;
      const int ya = y / NQ, yb = y % NQ;
      const int xb = (a == 0) ? ya * S::T1 + yb : (a == 1) ? ya * S::T0 + yb : ya * S::T0 + yb * S::T1;
      double v = 0.0;
#pragma unroll
      for (int i = 0; i < NQ; ++i) v = fma(vec[i], sN[c * S::NSP + xb + i * sa], v);
      P.tr_out[((long long)(2 * a + side) * P.slots + own_slot) * REC + NF * M + y * M + c] = v;
    }
  }
#pragma unroll
  for (int c = 0; c < M; ++c) Dg[x * M + c] = Dv[c] * scale;

  // ---------------- q-bar face traces ----------------
  __syncthreads();
#pragma unroll
  for (int c = 0; c < M; ++c) sN[c * S::NSP + xp] = qb[c];
  if (tid < 2 * DIM) sSmax[tid] = 0ull;
  __syncthreads();
  for (int e = tid; e < 2 * DIM * NF * M; e += THREADS) {
    const int y = (e >> 1) % NF;
    const int ca = (e >> 1) / NF;
    const int c = ca % M;
    const int f = 2 * (ca / M) + (e & 1);
    const int a = f >> 1;
    const double* vec = (f & 1) ? P.ops.right : P.ops.left;
    const int ya = y / NQ, yb = y % NQ;
    const int sa = (a == 0) ? S::T0 : (a == 1) ? S::T1 : 1;
    const int xb = (a == 0) ? ya * S::T1 + yb : (a == 1) ? ya * S::T0 + yb : ya * S::T0 + yb * S::T1;
    double v = 0.0;
#pragma unroll
    for (int i = 0; i < NQ; ++i) v = fma(vec[i], sN[c * S::NSP + xb + i * sa], v);
    P.tr_out[((long long)f * P.slots + own_slot) * REC + y * M + c] = v;
  }
  // ---------------- s_max over the space-time traces, one time level at a time ----------------
  double smx = 0.0;                      // this thread's face f = 2 * ((tid >> 1) / NF) + (tid & 1) (tid < 384)
#pragma unroll 1
  for (int t = 0; t < NQ; ++t) {
    double qt[M];
    tmem_ld_doubles<M>(tq + 2 * t, 16, qt);
    __syncthreads();
#pragma unroll
    for (int c = 0; c < M; ++c) sN[c * S::NSP + xp] = qt[c];
    __syncthreads();
    if (tid < 2 * DIM * NF) {
      const int e = tid;
      const int y = (e >> 1) % NF;
      const int f = 2 * ((e >> 1) / NF) + (e & 1);
      const int a = f >> 1;
      const double* vec = (f & 1) ? P.ops.right : P.ops.left;
      const int ya = y / NQ, yb = y % NQ;
      const int sa = (a == 0) ? S::T0 : (a == 1) ? S::T1 : 1;
      const int xb = (a == 0) ? ya * S::T1 + yb : (a == 1) ? ya * S::T0 + yb : ya * S::T0 + yb * S::T1;
      double qs[M];
#pragma unroll
      for (int c = 0; c < M; ++c) {
        double v = 0.0;
#pragma unroll
        for (int i = 0; i < NQ; ++i) v = fma(vec[i], sN[c * S::NSP + xb + i * sa], v);
        qs[c] = v;
      }
      bool adm;
      const double sp = max_speed_fast<DIM>(qs, a, a + 1, adm);
      // NaN must win the max like the reference's np.max: compare bit patterns
      smx = (__double_as_longlong(sp) > __double_as_longlong(smx)) ? sp : smx;
    }
  }
  if (tid < 2 * DIM * NF)
    atomicMax(&sSmax[2 * ((tid >> 1) / NF) + (tid & 1)], (unsigned long long)__double_as_longlong(smx));
  tmem_release();   // (its barrier also orders the s_max atomics)
  if (tid < 2 * DIM) {
    double* rec = P.tr_out + ((long long)tid * P.slots + own_slot) * REC;
    rec[2 * NF * M] = __longlong_as_double((long long)sSmax[tid]);
    rec[2 * NF * M + 1] = record_stamp(P);
  }
}

}  // namespace adg
