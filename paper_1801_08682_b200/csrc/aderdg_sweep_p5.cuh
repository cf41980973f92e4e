// aderdg_sweep_p5.cuh — the fused 3D sweep at p = 5 with the Picard derivatives
// on the FP64 tensor cores.
//
// One CTA per cell, 224 threads (7 warps; thread = spatial node, block_map_p5b), two
// CTAs per SM (128 registers, 104 KB of shared memory, 256 TMEM columns each).  The
// per-node time line q[t][c] and the divergence history dv[k][c] live in tensor memory
// (tcgen05.ld/st 32x32b), so the time contraction (integ) is register-local DFMA work.
// The spatial derivatives of a time slice are three small GEMMs per slice,
//
//     Out_a[i][col] = sum_j diff[i][j] F_a[j][col],   col = c*36 + (other two indices)
//
// (180 columns + 4 zero pad columns = 23 n-tiles of 8), issued as DMMA m8n8k4 with
// diff as the A operand (two constant fragments per lane: k = 0..3 and 4..5, rows
// and columns 6..7 zero) and the flux as the B operand straight from shared memory;
// each tile writes its 6 useful output rows back in place over its own columns
// (a tile's outputs depend only on its own columns), and the node owner sums the
// three axes.
//
// Slice pipeline (one barrier per slice): the operand arrays are double-buffered by
// slice parity; the interval that runs the tiles of slice k also stages the flux of
// slice k + 1, and the first Picard iteration (q_t = Q at every level: six identical
// slices) computes one slice.
//
// Shared-memory layout (the kernel is bound by shared-memory wavefronts: r02 ncu,
// 67 % of the LSU peak at 1.5-2x the ideal wavefront count before this layout): row
// stride 200 with rows 2, 3 shifted by 4 doubles, thread blocks of 2x2x2 nodes per
// quarter-warp grouped into warps by a search (block_map_p5b) — every shared access of
// the Picard loop then takes its minimum number of wavefronts.
//
// The rest (TMA bulk staging of Q, D and the 4d face records, Riemann, corrector,
// calc_time_step, final flux, volume integral, face traces, s_max) follows
// sweep_kernel_p3.
//
// Reference (src/ = /root/reference/pkg/src/aderdg/): kernels.py:68-229 (predict,
// extrapolate, integrate_volume, solve_riemann, integrate_face, update,
// calc_time_step), scheduler.py:370-449 (fused sweep).
#pragma once
#include <type_traits>
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

// six doubles at 12 consecutive columns: one .x8 and one .x4 access (the column
// address needs no alignment to the access width, tools/tmem_align.cu)
__device__ __forceinline__ void tmem_ld6(uint32_t a, double (&v)[6]) {
  uint32_t r[12];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(a));
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11])
               : "r"(a + 8));
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5]), "+r"(r[6]), "+r"(r[7]),
                 "+r"(r[8]), "+r"(r[9]), "+r"(r[10]), "+r"(r[11])::"memory");
#pragma unroll
  for (int i = 0; i < 6; ++i) v[i] = __hiloint2double((int)r[2 * i + 1], (int)r[2 * i]);
}
__device__ __forceinline__ void tmem_st6(uint32_t a, const double (&v)[6]) {
  uint32_t r[12];
#pragma unroll
  for (int i = 0; i < 6; ++i) {
    r[2 * i] = (uint32_t)__double2loint(v[i]);
    r[2 * i + 1] = (uint32_t)__double2hiint(v[i]);
  }
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(a), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};" ::"r"(a + 8), "r"(r[8]), "r"(r[9]),
               "r"(r[10]), "r"(r[11])
               : "memory");
}

// five doubles at 10 consecutive columns: one .x8 and one .x2 store
__device__ __forceinline__ void tmem_st5(uint32_t a, const double (&v)[5]) {
  uint32_t r[10];
#pragma unroll
  for (int i = 0; i < 5; ++i) {
    r[2 * i] = (uint32_t)__double2loint(v[i]);
    r[2 * i + 1] = (uint32_t)__double2hiint(v[i]);
  }
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(a), "r"(r[0]),
               "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
               : "memory");
  asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1,%2};" ::"r"(a + 8), "r"(r[8]), "r"(r[9]) : "memory");
}
// N = 2 or 3 doubles at consecutive columns, issue and wait apart (.x4, + .x2 for the third)
template <int N>
__device__ __forceinline__ void tmem_ldn_issue(uint32_t a, uint32_t (&r)[6]) {
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(a));
  if (N == 3)
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0,%1}, [%2];" : "=r"(r[4]), "=r"(r[5]) : "r"(a + 4));
}
template <int N>
__device__ __forceinline__ void tmem_ldn_wait(uint32_t (&r)[6], double (&v)[3]) {
  if (N == 3)
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3]), "+r"(r[4]), "+r"(r[5])::"memory");
  else
    asm volatile("tcgen05.wait::ld.sync.aligned;" : "+r"(r[0]), "+r"(r[1]), "+r"(r[2]), "+r"(r[3])::"memory");
#pragma unroll
  for (int i = 0; i < N; ++i) v[i] = __hiloint2double((int)r[2 * i + 1], (int)r[2 * i]);
}

// Thread -> node map of the p = 5 kernel.  Eight consecutive lanes own a 2x2x2 node
// block (lane bits 2,1,0 = the i0, i1, i2 offsets); a half-warp owns two of the 27 blocks.
// The shared-memory pipe serves 16-byte accesses per quarter-warp and 8-byte accesses per
// half-warp (r02 ncu: the wavefront counts of the p = 9 line engine match that model
// exactly), so with the operand row offsets below
//   * a 16-byte owner access of a quarter-warp (one block) touches eight distinct
//     16-byte bank groups along all three axes, and
//   * an 8-byte owner access of a half-warp touches 16 distinct banks along all three
//     axes when its two blocks' column bases differ by 4 (mod 8): a maximum matching of the
//     3x3x3 block grid under that condition pairs 22 of the 27 blocks (11 of 14 half-warps).
// Block code = 9 B0 + 3 B1 + B2.
__device__ __forceinline__ void block_map_p5b(int tid, int& i0, int& i1, int& i2, bool& act) {
  constexpr unsigned char kBlock[28] = {0, 8, 1, 10, 2, 6, 3, 12, 4, 13, 5, 14, 7, 16, 9, 17, 11, 15, 18, 26, 20, 24,
                                          19, 22, 21, 23, 25, 0};
  const int blk = tid >> 3;
  act = blk < 27;
  const int code = kBlock[blk];
  i0 = 2 * (code / 9) + ((tid >> 2) & 1);
  i1 = 2 * ((code / 3) % 3) + ((tid >> 1) & 1);
  i2 = 2 * (code % 3) + (tid & 1);
}

struct ShapeP5 {
  static constexpr int DIM = 3, M = 5, NQ = 6;
  static constexpr int NS = 216, NF = 36;
  static constexpr int THREADS = 224, NW = 7;
  static constexpr int REC = 2 * NF * M + 2;
  // DMMA operand arrays [slice parity][j][axis][184]: tile t of the slice (t = axis * 23 +
  // n-tile) starts at column 8 t of every row
  static constexpr int NCOL = 180, NTILE = 23, ACOL = NTILE * 8;
  static constexpr int STR = DIM * ACOL + 16;
  static constexpr int FBUF = NQ * STR;
  // operand row j starts at j * STR + 4 for j = 2, 3: with STR == 8 (mod 16) the rows sit
  // at bank offsets (0, 8, 4, 12, 0, 8) (8-byte banks): the four k rows of a B-fragment
  // load are disjoint (2 wavefronts), rows 4, 5 of the second chunk too (1), and the row
  // pairs (0,1), (2,3), (4,5) that a quarter-warp touches with 16-byte accesses (D store,
  // owner blocks) lie 64 bytes apart (mod 128)
  __host__ __device__ static constexpr int rowoff(int j) { return j * STR + ((j == 2 || j == 3) ? 4 : 0); }
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
  static_assert(STR >= DIM * ACOL + 4 && STR % 16 == 8 && ACOL % 16 == 8, "operand row layout");
};

// tools/p5_timeline.py (A/B build with -DADG_P5_TIMING): thread 0 stamps clock64 / globaltimer
#ifdef ADG_P5_TIMING
#define ADG_P5_STAMP(i)                                                                              \
  do {                                                                                               \
    if (threadIdx.x == 0 && P.sm_scratch != nullptr) P.sm_scratch[blockIdx.x * 8 + (i)] = (double)clock64(); \
  } while (0)
#define ADG_P5_GSTAMP(i)                                                                             \
  do {                                                                                               \
    if (threadIdx.x == 0 && P.sm_scratch != nullptr) {                                               \
      unsigned long long g_;                                                                         \
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_));                                         \
      P.sm_scratch[blockIdx.x * 8 + (i)] = (double)g_;                                               \
    }                                                                                                \
  } while (0)
#else
#define ADG_P5_STAMP(i) ((void)0)
#define ADG_P5_GSTAMP(i) ((void)0)
#endif

__global__ void __launch_bounds__(ShapeP5::THREADS, 2) sweep_kernel_p5(const SweepParams P) {
  using S = ShapeP5;
  ADG_P5_GSTAMP(0);
#ifdef ADG_P5_TIMING
  if (threadIdx.x == 0 && P.sm_scratch != nullptr) {
    unsigned sm_;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm_));
    P.sm_scratch[blockIdx.x * 8 + 6] = (double)sm_;
  }
#endif
  ADG_P5_STAMP(1);
  constexpr int DIM = 3, M = 5, NQ = 6, NS = S::NS, NF = S::NF, REC = S::REC, NW = S::NW;
  constexpr int THREADS = S::THREADS, ACOL = S::ACOL, FBUF = S::FBUF;

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
  block_map_p5b(tid, i0, i1, i2, act);
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
  // lane offsets inside a tile: B fragment rows k / k + 4 at column n, D row r columns 2k, 2k+1
  const int lb0 = S::rowoff(fk) + fr, lb1 = S::rowoff(fk < 2 ? fk + 4 : 4) + fr, lbd = S::rowoff(fr < NQ ? fr : 0) + 2 * fk;
  // owner offsets into one slice buffer: axis a, row i_a, column (other two indices)
  // (columns: components 0,1 interleaved over the 36 positions, then 2,3, then 4:
  //  col = 2o + c | 72 + 2o + (c - 2) | 144 + o, so an owner moves (F_0, F_1) and
  //  (F_2, F_3) with one 16-byte access each)
  const int rb[3] = {0 * ACOL + S::rowoff(i0), 1 * ACOL + S::rowoff(i1), 2 * ACOL + S::rowoff(i2)};
  const int ob[3] = {i1 * NQ + i2, i0 * NQ + i2, i0 * NQ + i1};

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
  for (int e = tid; e < 2 * DIM * NQ * 4; e += THREADS) {   // e = ((buffer * 3 + axis) * 6 + row) * 4 + pad
    const int r = (e >> 2) % NQ, ab = (e >> 2) / NQ;
    sU[(ab / DIM) * FBUF + S::rowoff(r) + (ab % DIM) * ACOL + S::NCOL + (e & 3)] = 0.0;
  }
  // Per-thread time line in tensor memory: 256 columns per CTA (two CTAs per SM fill
  // the 512), warp w on lanes 32*(w%4) and columns (w/4)*128.. : q[t][c] at column
  // 2(6c+t), the slice divergences dv[k][c] at 64 + 2(5k+c)
  __shared__ uint32_t s_tmem;
  ADG_P5_STAMP(2);
  if (warp == 0) tmem_alloc_cols<256>(&s_tmem);
  ADG_P5_STAMP(3);
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
    for (int c = 0; c < M; ++c) tmem_st_d(tq + 12 * c + 2 * t, Qx[c]);
  tmem_wait_st();

  int iters = 0;
  bool failed = false;
  // Software-pipelined slice loop, one barrier per slice.  The interval that runs the
  // DMMA tiles of slice k (operand buffer k & 1) also computes the flux of slice k + 1
  // into the other buffer: that buffer's last tile readers (slice k - 1) passed the
  // previous barrier, and an owner reads back and rewrites only its own addresses, in
  // program order.  Two independent chains (TMEM load -> flux -> stores, operand loads
  // -> DMMA -> stores) share every interval.  The flux of the next iteration's slice 0
  // is staged before the convergence vote, whose barrier publishes it (wasted once,
  // when the vote ends the iteration).
  auto stage_flux = [&](int k, const double (&qk)[M]) {
    double* B = sU + (k & 1) * FBUF;
    double F[DIM][M];
    flux<DIM>(qk, F);
    if (act) {
#pragma unroll
      for (int a = 0; a < DIM; ++a) {
        *reinterpret_cast<double2*>(B + rb[a] + 2 * ob[a]) = make_double2(F[a][0], F[a][1]);
        *reinterpret_cast<double2*>(B + rb[a] + 72 + 2 * ob[a]) = make_double2(F[a][2], F[a][3]);
        B[rb[a] + 144 + ob[a]] = F[a][4];
      }
    }
  };
#ifdef ADG_AB_P5_TILES
  // Out_a = diff . F_a on the tensor cores, in place, tile by tile: warp w takes tiles
  // w, w + 7, ... of the 69 (constant offsets from one base address)
  auto run_tiles = [&](int k) {
    double* base0 = sU + (k & 1) * FBUF + warp * 8;
#pragma unroll
    for (int i = 0; i < (S::TILES + NW - 1) / NW; ++i) {
      if (i * NW + NW > S::TILES && warp + i * NW >= S::TILES) break;
      double* base = base0 + i * NW * 8;
      const double b0 = base[lb0];
      const double b1 = (fk < 2) ? base[lb1] : 0.0;
      double d0, d1;
      dmma_nv(d0, d1, a_lo, b0, 0.0, 0.0);
      dmma_nv(d0, d1, a_hi, b1, d0, d1);
      if (lane < 4 * NQ) *reinterpret_cast<double2*>(base + lbd) = make_double2(d0, d1);
    }
  };
#define ADG_P5_DERIV run_tiles
#else
  // The derivative lines of the slice, one per thread and round on the FP64 pipe, in place
  // (line l = axis * 180 + column; 540 lines over 224 threads), through the even / odd
  // blocks of the centro-antisymmetric diff: e_j = f_j + f_{5-j}, o_j = f_j - f_{5-j},
  // out_i = so_i + se_i, out_{5-i} = so_i - se_i (30 instead of 36 operations per line and
  // none of the 44 % tile padding of the DMMA form: measured 3.94 vs 4.40 ms per sweep).
  auto run_lines = [&](int k) {
    double* B = sU + (k & 1) * FBUF;
#pragma unroll 1
    for (int r = 0; r < 3; ++r) {
      const int l = tid + r * THREADS;
      if (l < DIM * S::NCOL) {
        const int a = (l >= 2 * S::NCOL) ? 2 : (l >= S::NCOL) ? 1 : 0;
        double* ln = B + a * ACOL + (l - a * S::NCOL);
        double e[3], o[3];
#pragma unroll
        for (int j = 0; j < 3; ++j) {
          const double u = ln[S::rowoff(j)], v = ln[S::rowoff(5 - j)];
          e[j] = u + v;
          o[j] = u - v;
        }
#pragma unroll
        for (int i = 0; i < 3; ++i) {
          double se = P.ops.eo_e[i][0] * e[0];
          double so = P.ops.eo_o[i][0] * o[0];
#pragma unroll
          for (int j = 1; j < 3; ++j) {
            se = fma(P.ops.eo_e[i][j], e[j], se);
            so = fma(P.ops.eo_o[i][j], o[j], so);
          }
          ln[S::rowoff(i)] = so + se;
          ln[S::rowoff(5 - i)] = so - se;
        }
      }
    }
  };
#define ADG_P5_DERIV run_lines
#endif
  // the node's divergence of slice k into its TMEM column (idle lanes read a real
  // node's sums and discard them); the first iteration's slice stands for every k
  auto read_back = [&](int k, bool every_k) {
    const double* B = sU + (k & 1) * FBUF;
    double o[DIM][M];
#pragma unroll
    for (int a = 0; a < DIM; ++a) {
      const double2 u = *reinterpret_cast<const double2*>(B + rb[a] + 2 * ob[a]);
      const double2 v = *reinterpret_cast<const double2*>(B + rb[a] + 72 + 2 * ob[a]);
      o[a][0] = u.x; o[a][1] = u.y; o[a][2] = v.x; o[a][3] = v.y;
      o[a][4] = B[rb[a] + 144 + ob[a]];
    }
    double dvc[M];
#pragma unroll
    for (int c = 0; c < M; ++c) dvc[c] = (o[0][c] + o[1][c]) + o[2][c];
    if (every_k) {
#pragma unroll
      for (int kk = 0; kk < NQ; ++kk) tmem_st5(td + 10 * kk, dvc);
    } else {
      tmem_st5(td + 10 * k, dvc);
    }
  };
  auto contract = [&](auto c0_, auto nc_, BitMax& bm, double (&q0n)[M]) {
    constexpr int C0 = decltype(c0_)::value, NC = decltype(nc_)::value;
    double acc[NC][NQ];
    uint32_t rr[6];
    tmem_ldn_issue<NC>(td + 2 * C0, rr);
#pragma unroll
    for (int k = 0; k < NQ; ++k) {
      double d[3];
      tmem_ldn_wait<NC>(rr, d);
      if (k + 1 < NQ) tmem_ldn_issue<NC>(td + 10 * (k + 1) + 2 * C0, rr);
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
      tmem_ld6(tq + 12 * (C0 + c), qo);
      const double qc = sQ[x * M + C0 + c];
#pragma unroll
      for (int t = 0; t < NQ; ++t) {
        acc[c][t] = qc - scale * acc[c][t];
        bm.add(fabs(acc[c][t] - qo[t]));
      }
      q0n[C0 + c] = acc[c][0];
      tmem_st6(tq + 12 * (C0 + c), acc[c]);
    }
  };
  stage_flux(0, Qx);
  __syncthreads();
#pragma unroll 1
  for (int it = 0; it < cap; ++it) {
    if (it == 0) {
      // q_t = Q at every time level: the NQ slices are identical, one is computed
      ADG_P5_DERIV(0);
      __syncthreads();
      read_back(0, true);
    } else {
#pragma unroll
      for (int k = 0; k < NQ; ++k) {
        if (k + 1 < NQ) {
          double qk[M];
          tmem_ld_doubles<M>(tq + 2 * (k + 1), 12, qk);
          stage_flux(k + 1, qk);
        }
        ADG_P5_DERIV(k);
        __syncthreads();
        read_back(k, false);
      }
    }
    tmem_wait_st();
    // time contraction of the divergence history + Picard update (kernels.py:86-97), k
    // outermost over groups of 3 + 2 components (every integ[t][k] fetched from the constant
    // bank feeds 3 (2) FMAs; the accumulators become the new time line in place);
    // convergence from the bit patterns of |q_new - q|
    BitMax bm;
    double q0n[M];
    contract(std::integral_constant<int, 0>(), std::integral_constant<int, 3>(), bm, q0n);
    contract(std::integral_constant<int, 3>(), std::integral_constant<int, 2>(), bm, q0n);
    tmem_wait_st();
    iters = it + 1;
    if (it + 1 < cap) stage_flux(0, q0n);        // slice 0 of the next iteration
    const int fl = block_flags<NW>(!act || bm.conv(tol), act && bm.bad(), sFlags, it & 1);
    if (fl & 2) { failed = true; break; }
    if (fl & 1) break;
  }

  // final flux: time average (fbar) + finiteness, level by level from TMEM; every
  // level of q (for the space-time trace speeds) and qbar into shared memory (the
  // operand buffers are free: the last slice's owner loads precede the convergence
  // barrier)
  double fb[DIM][M], qb[M];
#pragma unroll
  for (int c = 0; c < M; ++c) {
    qb[c] = 0.0;
#pragma unroll
    for (int a = 0; a < DIM; ++a) fb[a][c] = 0.0;
  }
  bool bad = false;
#pragma unroll
  for (int t = 0; t < NQ; ++t) {
    double qt[M];
    tmem_ld_doubles<M>(tq + 2 * t, 12, qt);
    if (!failed) {
      double F[DIM][M];
      flux<DIM>(qt, F);
#pragma unroll
      for (int a = 0; a < DIM; ++a)
#pragma unroll
        for (int c = 0; c < M; ++c) {
          bad |= !finite(F[a][c]);
          fb[a][c] = fma(P.ops.w[t], F[a][c], fb[a][c]);
        }
    }
#pragma unroll
    for (int c = 0; c < M; ++c) {
      if (act) sQt[(t * M + c) * NS + x] = qt[c];
      qb[c] = fma(P.ops.w[t], qt[c], qb[c]);
    }
  }
  tmem_fence_before();
  failed = __syncthreads_or(act && bad) || failed;
  // every TMEM access of the CTA precedes the barrier above: release the columns
  tmem_fence_after();
  ADG_P5_STAMP(4);
  if (warp == 0) tmem_dealloc_cols<256>(s_tmem);
  ADG_P5_STAMP(5);
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

  if (act) {
#pragma unroll
    for (int c = 0; c < M; ++c) {
      sQb[c * NS + x] = qb[c];
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
  ADG_P5_GSTAMP(7);
}

}  // namespace adg
