// aderdg_sweep_v2.cuh — second-generation fused sweep kernel (3D, even p+1).
//
// Changes against sweep_kernel (aderdg_kernels.cuh), driven by the r01 ncu
// profile (12 warps/SM, 168 regs, 30% smem bank conflicts, long-scoreboard
// stalls on the staging loads):
//   * time split: TS threads per spatial node, each owning NQ/TS time levels
//     of the space-time predictor -> TS x more warps, fewer registers.  The
//     time contraction of the Picard update (integ) reads the per-slice
//     divergence of all time levels from shared memory (sDiv).
//   * TMA bulk copies (cp.async.bulk + mbarrier) stage Q, D and the 4d face
//     records of the cell into shared memory in one shot; Q and D go back
//     with bulk stores.
//   * padded flux slices: the axis-0 plane stride is NQ^2 + pad so that the
//     derivative gathers of a warp are bank-conflict free (broadcasts only).
//   * p = 3 (NQ = 4): node index bits i2 sit in lane bits 0-1, so the axis-2
//     derivative is one DMMA.8x8x4 per component with the flux in the A
//     fragment and an interleaved diff^T in B: the result lands in the lane
//     that owns the node (no shared-memory round trip for that axis).
//
// Reference (src/ = /root/reference/pkg/src/aderdg/): same as sweep_kernel —
// kernels.py:68-229 (seven tasks), scheduler.py:370-449 (fused sweep).
#pragma once
#include "aderdg_kernels.cuh"

namespace adg {

__host__ __device__ constexpr int plane_pad(int nq) {
  // smallest pad so that (nq*nq + pad) mod 16 lies in [nq, 16 - nq] (8-byte banks)
  return ((nq * nq) % 16 >= nq && (nq * nq) % 16 <= 16 - nq) ? 0
         : (((nq * nq + 2) % 16 >= nq && (nq * nq + 2) % 16 <= 16 - nq) ? 2
         : (((nq * nq + 4) % 16 >= nq && (nq * nq + 4) % 16 <= 16 - nq) ? 4
         : (((nq * nq + 6) % 16 >= nq && (nq * nq + 6) % 16 <= 16 - nq) ? 6 : 8)));
}

template <int NQ, int TS, bool DMMA, bool ROLLED = (NQ == 4), int MINB_OVERRIDE = 0>
struct ShapeV2 {
  static constexpr int DIM = 3, M = 5;
  static constexpr int NS = NQ * NQ * NQ;
  static constexpr int NF = NQ * NQ;
  static constexpr int NSP = (NS + 31) / 32 * 32;
  static constexpr int THREADS = TS * NSP;
  static constexpr int NWARPS = THREADS / 32;
  static constexpr int TH = NQ / TS;
  // CTAs/SM the register allocation must allow (TS = 1 at NQ = 6 keeps 60 doubles of Picard state)
  // MINB_OVERRIDE 10: axis-1 derivative on the tensor cores through a lane transpose (A1S)
  // MINB_OVERRIDE 16 / 17: A1S with 8 / 7 CTAs per SM forced (<= 128 / 144 registers)
  // MINB_OVERRIDE 20: A1S + A0X (axis 0 from per-warp partial sums: the warp of
  // planes {2w, 2w+1} contracts its own two planes for its nodes and for the other
  // warp's nodes; one shuffle, one store and one load per component replace the
  // four-plane shared-memory gather)
  // MINB_OVERRIDE 30 (PEN, NQ = 6): pencil Picard loop — a thread owns one time
  // level of one i2-pencil (6 nodes); axis 2 is register-local, axes 0/1 and the
  // time contraction are 16-byte broadcast gathers of whole pencils
  static constexpr bool PEN = (MINB_OVERRIDE == 30);
  // MINB_OVERRIDE 31 (BLK, NQ = 6): node-per-thread kernel with warps mapped to node
  // blocks (2x4x4, 4x4x2, ...: every axis sees <= 16 lines per warp) and a flux
  // slice layout i0*73 + i1*12 + i2 that keeps those gathers bank-conflict free
  static constexpr bool BLK = (MINB_OVERRIDE == 31);
  static constexpr bool A0X = (MINB_OVERRIDE == 20);
  // MINB_OVERRIDE 11: A1S with a software-pipelined slice loop (p = 3 default);
  // 14: the same with the axis-1 and axis-2 DMMAs of a slice completed (and the
  // axis-1 result transposed back) in the interval that produces the slice
  static constexpr bool PIPE = (MINB_OVERRIDE == 11 || MINB_OVERRIDE == 14);
  static constexpr bool PIPE2 = (MINB_OVERRIDE == 14);
  static constexpr bool A1S = (MINB_OVERRIDE == 10 || MINB_OVERRIDE == 16 || MINB_OVERRIDE == 17 || A0X || PIPE);
  static constexpr int MINB = (PEN || BLK) ? 1 : (MINB_OVERRIDE == 16) ? 8 : (MINB_OVERRIDE == 17) ? 7 : A0X ? 6
                            : (MINB_OVERRIDE && MINB_OVERRIDE != 9 && !A1S) ? MINB_OVERRIDE : (MINB_OVERRIDE == 9) ? 1
                            : (TS == 1 && NQ >= 6) ? 1
                            : THREADS <= 64 ? 6 : THREADS <= 128 ? 4 : (THREADS <= 256 ? 2 : 1);
  static constexpr int P1 = BLK ? 12 : NQ;             // axis-1 row stride of a flux slice
  static constexpr int P0 = BLK ? 73 : NQ * NQ + plane_pad(NQ);   // padded axis-0 plane stride
  static constexpr int PS = NQ * P0;                   // padded slice size
  static constexpr int DS = DMMA ? (A1S ? 1 : DIM - 1) : DIM;   // axes through shared memory
  static constexpr bool F1T = !A1S && ((NQ == 4) || (NQ == 6 && MINB_OVERRIDE == 9));  // axis-1 flux stored transposed, 16-byte gathers
  static constexpr bool ROLL = ROLLED;                 // rolled slice loop (i-cache); NQ = 6 stays unrolled
  static constexpr int RR = 1;                         // slices per rolled trip
  static constexpr bool DBUF = (TS == 1 && (NQ == 4 || MINB_OVERRIDE == 9));  // double-buffered flux slices
  static constexpr int P1T = NQ * NQ + 2;              // its plane stride (odd number of 16-byte chunks)
  static constexpr int REC = 2 * NF * M + 2;
  // shared memory (doubles), all region sizes even (16-byte alignment)
  static constexpr int R_RED = 3 * NWARPS + 2 * DIM + 4;   // block_max | s_max | convergence flags
  static constexpr int R_Q = NS * M;
  static constexpr int R_REC = 4 * DIM * REC;
  static constexpr int R_F = TS * DS * M * PS;
  static constexpr int R_FB = DIM * M * PS;            // fbar (after the Picard loop)
  static constexpr int R_DIV = (NQ + 1) * M * NSP;     // divergence of all slices / q slices + qbar
  static constexpr int R_PRED0 = (R_F > R_FB ? R_F : R_FB) + R_DIV;
  static constexpr int R_PRED1 = ((ROLL || DBUF) && 2 * R_F > R_PRED0) ? 2 * R_F : R_PRED0;
  // PEN: F0 | F1 | div pencil buffers, row (t, j0, j1) at t*30 + j0*S0 + j1*S1 (strides from a
  // bank-conflict search over the warp blocks below: every 8-byte gather of a warp hits <= 16
  // distinct addresses in distinct bank pairs)
  static constexpr int PB0 = 6 * 1083, PB1 = 6 * 1092, PB2 = 6 * 1083;
  static constexpr int R_PRED = (PEN && PB0 + PB1 + PB2 > R_PRED1) ? PB0 + PB1 + PB2 : R_PRED1;
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
  static_assert((NS * M) % 2 == 0, "bulk copies need 16-byte sizes");
  static_assert(NQ % TS == 0, "time split must divide NQ");
  static_assert(!DMMA || NQ == 4, "DMMA axis-2 path needs i2 in lane bits 0-1");
  static_assert(!A1S || (DMMA && TS == 1 && DBUF), "A1S runs in the double-buffered DMMA slice loop");
  static_assert(!A0X || (NQ == 4 && THREADS == 64), "A0X pairs the two warps of a p = 3 cell");
  static_assert(!(PEN || BLK) || (NQ == 6 && TS == 1 && !DMMA && NSP == 224), "PEN / BLK are p = 5 layouts");
  static_assert(SMEM_BYTES <= 232448, "shared memory per CTA");
};

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

// Node address in the trace-phase q layout.  NQ = 4: Latin-cube swizzle
// 16*i2 + 4*((i0+i2)&3) + ((i1+i2)&3): for every axis, the 16 nodes of a face
// plane hit 16 distinct 8-byte banks, so the face-trace gathers of a
// half-warp are conflict free along all three axes.
template <int NQ>
__device__ __forceinline__ int trace_addr(int i0, int i1, int i2) {
  if (NQ == 4) return 16 * i2 + 4 * ((i0 + i2) & 3) + ((i1 + i2) & 3);
  return (i0 * NQ + i1) * NQ + i2;
}

// p = 5 warp blocks over a 6x6x6 index cube (a, b, c): warps 0-2 take a-pairs x
// b 0-3 x c 0-3; warp 3 a 0-3 x b 0-3 x c 4-5; warp 4 a 0-3 x b 4-5 x c 0-3;
// warp 5 a 4-5 x (b 0-3 x c 4-5 | b 4-5 x c 0-3); warp 6 (24 lanes) a 0-5 x
// b 4-5 x c 4-5.  Every warp's projections onto (a, b), (a, c), (b, c) have at
// most 16 elements, so a gather that varies one index hits <= 16 distinct rows.
// Within a warp each lane quad is a 2x2 block in (b, c) at fixed a: an 8-byte
// shared load costs one wavefront when every quad reads <= 2 distinct doubles
// (measured, tools/smem_wavefronts.cu: 16 bytes per quad per wavefront), so the
// gathers that vary a or b (rows fixed in c or b) are single-wavefront.
__device__ __forceinline__ void block_map_p5(int tid, int& a, int& b, int& c, bool& act) {
  const int w = tid >> 5, l = tid & 31, q = l >> 2, db = (l >> 1) & 1, dc = l & 1;
  act = true;
  if (w < 3) { a = 2 * w + (q >> 2); b = 2 * ((q >> 1) & 1) + db; c = 2 * (q & 1) + dc; }
  else if (w == 3) { a = q >> 1; b = 2 * (q & 1) + db; c = 4 + dc; }
  else if (w == 4) { a = q >> 1; b = 4 + db; c = 2 * (q & 1) + dc; }
  else if (w == 5) {
    const int u = q & 3;
    a = 4 + (u >> 1);
    if (q < 4) { b = 2 * (u & 1) + db; c = 4 + dc; }
    else { b = 4 + db; c = 2 * (u & 1) + dc; }
  } else {
    act = l < 24;
    a = act ? q : 0; b = 4 + db; c = 4 + dc;
  }
}

template <int NQ, int TS, bool DMMA, bool ROLLED = (NQ == 4), int MB = 0>
__global__ void __launch_bounds__(ShapeV2<NQ, TS, DMMA, ROLLED, MB>::THREADS, ShapeV2<NQ, TS, DMMA, ROLLED, MB>::MINB)
sweep_kernel_v2(const SweepParams P) {
  using S = ShapeV2<NQ, TS, DMMA, ROLLED, MB>;
  constexpr int DIM = 3, M = 5, NS = S::NS, NF = S::NF, NSP = S::NSP, REC = S::REC;
  constexpr int THREADS = S::THREADS, NW = S::NWARPS, TH = S::TH, P0 = S::P0, PS = S::PS;
  constexpr int DS = S::DS;

  extern __shared__ __align__(16) double smem[];
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + S::OFF_BAR);
  double* sRed = smem + S::OFF_RED;
  unsigned long long* sSmax = reinterpret_cast<unsigned long long*>(sRed + 2 * NW);
  unsigned* sFlags = reinterpret_cast<unsigned*>(sRed + 2 * NW + 2 * 3);
  double* sQ = smem + S::OFF_Q;
  double* sD = smem + S::OFF_D;
  double* sU = smem + S::OFF_U;
  double* sRec = sU;                                   // corrector phase
  double* sF = sU;                                     // predictor: [TS][DS][M][PS]
  double* sDiv = sU + (S::R_F > S::R_FB ? S::R_F : S::R_FB);   // [NQ][M][NSP]
  double* sFace = smem + S::OFF_FACE;
  ADG_DEBUG_POISON();

  DevState* st = P.st;
  if (st->status != 0) return;
  const int mode = P.mode;
  if (mode == MODE_RERUN && !st->rerun_next) return;
  if (mode_corrects(mode) && st->reduce[1] != 0) return;   // a predict pass already failed

  const int tid = threadIdx.x;
  const int ts = tid / NSP;
  const int x0 = tid % NSP;
  bool act = x0 < NS;
  int x = act ? x0 : 0;
  if constexpr (S::BLK) {
    int b0, b1, b2;
    block_map_p5(tid, b0, b1, b2, act);
    x = (b0 * NQ + b1) * NQ + b2;
  }
  const long long cell = sweep_cell(P);
  const long long gcell = cell + P.cell_offset;
  const int i0 = x / (NQ * NQ), i1 = (x / NQ) % NQ, i2 = x % NQ;
  constexpr int P1 = S::P1;
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
  // derivative rows of the shared-memory axes; DMMA B fragment for axis 2
  double drow[DS][NQ];
  {
    const int idx[3] = {i0, i1, i2};
#pragma unroll
    for (int a = 0; a < DS; ++a)
#pragma unroll
      for (int j = 0; j < NQ; ++j) drow[a][j] = P.ops.diff[idx[a]][j];
  }
  double bfrag = 0.0;
  if (DMMA) {
    const int lane = tid & 31;
    const int g = lane >> 2, t4 = lane & 3;      // B[k=t4][n=g]: n even -> diff[n/2][k]
    bfrag = (g & 1) ? 0.0 : P.ops.diff[g >> 1][t4];
  }
  // A1S: lane sigma(L) swaps lane bits 0-1 (i2) with bits 2-3 (i1).  The DMMA
  // A operand taken from lane sigma(L) has the i1 line in k; the product lands
  // in lane sigma(owner), so one shuffle in and one out replace the axis-1
  // shared-memory gather.
  const int sig = (tid & 16) | ((tid & 3) << 2) | ((tid >> 2) & 3);
  // A0X (NQ = 4, 64 threads): warp w holds planes i0 = 2w + (lane bit 4); the
  // partner lane (lane ^ 16) holds the other plane of the same (i1, i2) line.
  // cl/ch: my output row on the warp's low / high plane; ol/oh: the row of the
  // node in the other warp with the same lane (i0 ^ 2)
  double a0_cl = 0.0, a0_ch = 0.0, a0_ol = 0.0, a0_oh = 0.0;
  if (S::A0X) {
    const int w2 = 2 * (tid >> 5);
    a0_cl = P.ops.diff[i0][w2];
    a0_ch = P.ops.diff[i0][w2 + 1];
    a0_ol = P.ops.diff[i0 ^ 2][w2];
    a0_oh = P.ops.diff[i0 ^ 2][w2 + 1];
  }
  // padded gather bases for the shared-memory axes
  int gbase[DIM], gstr[DIM];
  gbase[0] = px - i0 * P0; gstr[0] = P0;
  gbase[1] = px - i1 * P1; gstr[1] = P1;
  gbase[2] = px - i2;      gstr[2] = 1;
  // F1T: axis-1 flux stored with i1 fastest (plane stride P1T), gathered as
  // 16-byte pairs; 8 distinct 16-byte chunks per warp -> one wavefront.
  const int p1t = i0 * S::P1T + i2 * NQ + i1;
  const int g1t = i0 * S::P1T + i2 * NQ;

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
    if (ts == 0 && act) {
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
    if (ts != 0 || !act) {
#pragma unroll
      for (int c = 0; c < M; ++c) Qx[c] = sQ[x * M + c];
    }
  }

  if (!mode_predict_only(mode)) {
    // ------------- calc_time_step (kernels.py:216-229) -------------
    bool ok = true;
    double lam = 0.0;
    if (ts == 0 && act) {
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
  double absmax;
  {
    double am = 0.0;
#pragma unroll
    for (int c = 0; c < M; ++c) am = fmax(am, fabs(Qx[c]));
    absmax = block_max<NW>(act ? am : 0.0, sRed);
  }
  const double tol = 1e-10 * (1.0 + absmax);
  const int cap = 2 * NQ;

  double q[TH][M];
#pragma unroll
  for (int s = 0; s < TH; ++s)
#pragma unroll
    for (int c = 0; c < M; ++c) q[s][c] = Qx[c];

  double* sFt = sF + ts * (DS * M * PS);
  int iters = 0;
  bool failed = false;
  if constexpr (S::PEN) {
    // Pencil Picard loop (p = 5).  Thread (t, j0, j1) owns time level t of the
    // i2-pencil (j0, j1, 0..5): 30 contiguous doubles [i2][c], the reference's
    // node-major layout.  Per iteration: flux of the 6 nodes; the axis-2
    // derivative from registers; F_0 / F_1 pencils to shared memory; the axis-0
    // (axis-1) derivative reads the 6 pencils (t, j, j1) ((t, j0, j)) that the
    // warp's threads sharing (t, j1) ((t, j0)) read too — 8-byte broadcast
    // gathers; the divergence pencils go back to shared memory and the time
    // contraction reads the 6 pencils (k, j0, j1) the same way.  Warps are
    // (t, j0, j1) blocks (2x4x4, 4x4x2, 4x2x4, ...) so each gather instruction
    // touches <= 16 distinct doubles (one wavefront; 16-byte loads measured
    // ~4 wavefronts each whatever the broadcast).
    constexpr int ROW = NQ * M;                         // one pencil: 30 doubles
    int pt, pj0, pj1;
    bool pact;
    block_map_p5(tid, pt, pj0, pj1, pact);
    double* sP0 = sU;                                   // F_0 pencils
    double* sP1 = sU + S::PB0;                          // F_1 pencils
    double* sPd = sU + S::PB0 + S::PB1;                 // divergence pencils
    double* w0 = sP0 + pt * ROW + pj0 * 180 + pj1 * 1083;
    double* w1 = sP1 + pt * ROW + pj0 * 181 + pj1 * 1092;
    double* wd = sPd + pt * ROW + pj0 * 180 + pj1 * 1083;
    const double* r0 = sP0 + pt * ROW + pj1 * 1083;    // + j * 180: rows (t, j, j1)
    const double* r1 = sP1 + pt * ROW + pj0 * 181;     // + j * 1092: rows (t, j0, j)
    const double* rd = sPd + pj0 * 180 + pj1 * 1083;   // + k * ROW: rows (k, j0, j1)
    const double* rq = sQ + (pj0 * NQ + pj1) * ROW;
    double d0[NQ], d1[NQ], ig[NQ];
#pragma unroll
    for (int j = 0; j < NQ; ++j) {
      d0[j] = P.ops.diff[pj0][j];
      d1[j] = P.ops.diff[pj1][j];
      ig[j] = P.ops.integ[pt][j];
    }
    double qp[NQ][M];
#pragma unroll
    for (int e = 0; e < ROW; ++e) qp[e / M][e % M] = rq[e];
#pragma unroll 1
    for (int it = 0; it < cap; ++it) {
      double dv[NQ][M];
#pragma unroll
      for (int o = 0; o < NQ; ++o)
#pragma unroll
        for (int c = 0; c < M; ++c) dv[o][c] = 0.0;
#pragma unroll
      for (int i2 = 0; i2 < NQ; ++i2) {
        double F[DIM][M];
        flux<DIM>(qp[i2], F);
        if (pact) {
#pragma unroll
          for (int c = 0; c < M; ++c) {
            w0[i2 * M + c] = F[0][c];
            w1[i2 * M + c] = F[1][c];
          }
        }
#pragma unroll
        for (int o = 0; o < NQ; ++o)
#pragma unroll
          for (int c = 0; c < M; ++c) dv[o][c] = fma(P.ops.diff[o][i2], F[2][c], dv[o][c]);
      }
      __syncthreads();
#pragma unroll
      for (int j = 0; j < NQ; ++j)
#pragma unroll
        for (int e = 0; e < ROW; ++e) dv[e / M][e % M] = fma(d0[j], r0[j * 180 + e], dv[e / M][e % M]);
#pragma unroll
      for (int j = 0; j < NQ; ++j)
#pragma unroll
        for (int e = 0; e < ROW; ++e) dv[e / M][e % M] = fma(d1[j], r1[j * 1092 + e], dv[e / M][e % M]);
      if (pact) {
#pragma unroll
        for (int e = 0; e < ROW; ++e) wd[e] = dv[e / M][e % M];
      }
      __syncthreads();
      // time contraction of the divergence pencils (k = 0..5) + Picard update
      double acc[NQ][M];
#pragma unroll
      for (int k = 0; k < NQ; ++k)
#pragma unroll
        for (int e = 0; e < ROW; ++e)
          acc[e / M][e % M] = (k == 0) ? ig[0] * rd[e] : fma(ig[k], rd[k * ROW + e], acc[e / M][e % M]);
      BitMax bm;
#pragma unroll
      for (int e = 0; e < ROW; ++e) {
        const double qn = rq[e] - scale * acc[e / M][e % M];
        bm.add(fabs(qn - qp[e / M][e % M]));
        qp[e / M][e % M] = qn;
      }
      iters = it + 1;
      const int fl = block_flags<NW>(!pact || bm.conv(tol), pact && bm.bad(), sFlags, it & 1);
      if (fl & 2) { failed = true; break; }
      if (fl & 1) break;
    }
    if (!failed) {
      // publish the final iterate in the trace layout; continue in the node view
      double* sQt = sDiv;
      if (pact) {
#pragma unroll
        for (int i2 = 0; i2 < NQ; ++i2)
#pragma unroll
          for (int c = 0; c < M; ++c) sQt[(pt * M + c) * NSP + trace_addr<NQ>(pj0, pj1, i2)] = qp[i2][c];
      }
      __syncthreads();
      const int qa = trace_addr<NQ>(i0, i1, i2);
#pragma unroll
      for (int s = 0; s < TH; ++s)
#pragma unroll
        for (int c = 0; c < M; ++c) q[s][c] = sQt[(s * M + c) * NSP + qa];
    }
  } else if constexpr (TS == 1 && S::ROLL) {
    // Rolled slice loop (keeps the Picard loop inside the instruction cache):
    // each trip processes RR slices from register slots 0..RR-1, then the
    // time line rotates by RR slots (back in order after NQ slices).
#pragma unroll 1
    for (int it = 0; it < cap; ++it) {
      double acc[NQ][M];
#pragma unroll
      for (int t = 0; t < NQ; ++t)
#pragma unroll
        for (int c = 0; c < M; ++c) acc[t][c] = 0.0;
      // one barrier per slice: the flux slice is double-buffered by slice
      // parity, and the time-contraction update of slice k is applied while
      // slice k+1's flux stores drain (hides the DMMA -> FMA latency)
      double dvp[M];
#pragma unroll
      for (int c = 0; c < M; ++c) dvp[c] = 0.0;
#pragma unroll 1
      for (int k = 0; k < NQ; ++k) {
        double* sFk = sF + (k & 1) * (DS * M * PS);
        double F[DIM][M];
        flux<DIM>(q[0], F);
        if (act) {
#pragma unroll
          for (int a = 0; a < DS; ++a)
#pragma unroll
            for (int c = 0; c < M; ++c)
              sFk[(a * M + c) * PS + ((S::F1T && a == 1) ? p1t : px)] = F[a][c];
        }
        if (k > 0) {
#pragma unroll
          for (int t = 0; t < NQ; ++t) {
            const double ic = P.ops.integ[t][k - 1];
#pragma unroll
            for (int c = 0; c < M; ++c) acc[t][c] = fma(ic, dvp[c], acc[t][c]);
          }
        }
#pragma unroll
        for (int c = 0; c < M; ++c) {
          const double q0 = q[0][c];
#pragma unroll
          for (int t = 0; t + 1 < NQ; ++t) q[t][c] = q[t + 1][c];
          q[NQ - 1][c] = q0;
        }
        __syncthreads();
#pragma unroll
        for (int c = 0; c < M; ++c) {
          double part[DS];
#pragma unroll
          for (int a = 0; a < DS; ++a) {
            double v = 0.0;
            if (S::F1T && a == 1) {
              const double2* b2 = reinterpret_cast<const double2*>(sFk + (a * M + c) * PS + g1t);
#pragma unroll
              for (int jj = 0; jj < NQ / 2; ++jj) {
                const double2 w2 = b2[jj];
                v = fma(drow[a][2 * jj], w2.x, v);
                v = fma(drow[a][2 * jj + 1], w2.y, v);
              }
            } else {
              const double* b = sFk + (a * M + c) * PS + gbase[a];
#pragma unroll
              for (int j = 0; j < NQ; ++j) v = fma(drow[a][j], b[j * gstr[a]], v);
            }
            part[a] = v;
          }
          double sum = part[0];
#pragma unroll
          for (int a = 1; a < DS; ++a) sum += part[a];
          dvp[c] = sum;
        }
        if (DMMA) {
#pragma unroll
          for (int c = 0; c < M; ++c) {
            double d1;
            dmma_8x8x4(dvp[c], d1, F[2][c], bfrag, dvp[c], 0.0);
          }
        }
      }
#pragma unroll
      for (int t = 0; t < NQ; ++t) {
        const double ic = P.ops.integ[t][NQ - 1];
#pragma unroll
        for (int c = 0; c < M; ++c) acc[t][c] = fma(ic, dvp[c], acc[t][c]);
      }
      // Picard update; max |q_new - q| via the bit patterns of non-negative
      // doubles (NaN/inf patterns sort above every finite value)
      // converged iff every |q_new - q| <= tol; a running sum carries inf/NaN
      BitMax bm;
#pragma unroll
      for (int t = 0; t < NQ; ++t)
#pragma unroll
        for (int c = 0; c < M; ++c) {
          const double qn = Qx[c] - scale * acc[t][c];
          bm.add(fabs(qn - q[t][c]));
          q[t][c] = qn;
        }
      iters = it + 1;
      const int fl = block_flags<NW>(!act || bm.conv(tol), act && bm.bad(), sFlags, it & 1);
      if (fl & 2) { failed = true; break; }
      if (fl & 1) break;
    }
  } else if constexpr (S::PIPE) {
    // Software-pipelined slice loop (p = 3, A1S): the interval after the barrier
    // that publishes slice s also computes the flux of slice s+1 — its axis-0 flux
    // goes to the other buffer, whose readers (slice s-1) all passed this barrier —
    // and issues its axis-1 DMMA, so two independent dependency chains share every
    // barrier interval.  PIPE2 also issues the slice's axis-2 DMMA (C = 0) there and
    // transposes the axis-1 result back, leaving only the axis-0 gather after the barrier.
    auto produce = [&](int sl, double (&f2)[M], double (&d1)[M]) {
      double F[DIM][M];
      flux<DIM>(q[sl], F);
      double* sFn = sF + (sl & 1) * (DS * M * PS);
      if (act) {
#pragma unroll
        for (int c = 0; c < M; ++c) sFn[c * PS + px] = F[0][c];
      }
#pragma unroll
      for (int c = 0; c < M; ++c) {
        const double a1 = __shfl_sync(0xffffffffu, F[1][c], sig);
        double z1;
        dmma_8x8x4(d1[c], z1, a1, bfrag, 0.0, 0.0);
        if (S::PIPE2) dmma_8x8x4(f2[c], z1, F[2][c], bfrag, 0.0, 0.0);
        else f2[c] = F[2][c];
      }
    };
    auto finish_produce = [&](double (&d1)[M]) {
      if (S::PIPE2) {
#pragma unroll
        for (int c = 0; c < M; ++c) d1[c] = __shfl_sync(0xffffffffu, d1[c], sig);
      }
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
        for (int j = 0; j < NQ; ++j) v = fma(drow[0][j], b[j * gstr[0]], v);
        double dv = S::PIPE2 ? (v + d1c[c]) + F2c[c] : v + __shfl_sync(0xffffffffu, d1c[c], sig);
        if (!S::PIPE2) {
          double d1;
          dmma_8x8x4(dv, d1, F2c[c], bfrag, dv, 0.0);
        }
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
      const int fl = block_flags<NW>(!act || bm.conv(tol), act && bm.bad(), sFlags, 0);
      if (fl & 2) failed = true;
      first_done = fl != 0;
    }
#pragma unroll 1
    for (int it = 1; it < cap && !first_done; ++it) {
      double accr[NQ][M];
      double dvp[M];
      double F2c[M], d1c[M];           // current slice: axis-2 flux (A operand) / PIPE2: axis-2 result,
                                       // axis-1 DMMA result (PIPE2: transposed back)
      produce(0, F2c, d1c);
      finish_produce(d1c);
#pragma unroll
      for (int s = 0; s < NQ; ++s) {
        __syncthreads();
        const double* sFs = sF + (s & 1) * (DS * M * PS);
        double dv[M];
#pragma unroll
        for (int c = 0; c < M; ++c) {
          const double* b = sFs + c * PS + gbase[0];
          double v = 0.0;
#pragma unroll
          for (int j = 0; j < NQ; ++j) v = fma(drow[0][j], b[j * gstr[0]], v);
          dv[c] = S::PIPE2 ? (v + d1c[c]) + F2c[c] : v + __shfl_sync(0xffffffffu, d1c[c], sig);
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
        for (int c = 0; c < M; ++c) {
          if (!S::PIPE2) {
            double d1;
            dmma_8x8x4(dv[c], d1, F2c[c], bfrag, dv[c], 0.0);
          }
          dvp[c] = dv[c];
        }
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
      const int fl = block_flags<NW>(!act || bm.conv(tol), act && bm.bad(), sFlags, it & 1);
      if (fl & 2) { failed = true; break; }
      if (fl & 1) break;
    }
  } else {
  for (int it = 0; it < cap; ++it) {
    double accr[TS == 1 ? NQ : 1][M];            // register time contraction (TS == 1)
    double dvp[M];                               // pending slice (DBUF: deferred contraction)
#pragma unroll
    for (int s = 0; s < TH; ++s) {
      const int k = ts * TH + s;
      // TS == 1: flux slices alternate between two buffers, so the barrier
      // that publishes slice k also retires the reads of slice k-2's buffer
      double* sFs = (TS == 1 && S::DBUF) ? sF + (k & 1) * (DS * M * PS) : sFt;
      double F[DIM][M];
      flux<DIM>(q[s], F);
      double own0[M];                            // A0X: this warp's two planes, my row
      if (S::A0X) {
        const bool hi = (tid & 16) != 0;         // my plane is the warp's high plane
#pragma unroll
        for (int c = 0; c < M; ++c) {
          const double pf = __shfl_xor_sync(0xffffffffu, F[0][c], 16);
          const double flo = hi ? pf : F[0][c], fhi = hi ? F[0][c] : pf;
          own0[c] = fma(a0_ch, fhi, a0_cl * flo);
          // the other warp's node on this lane: its row (i0 ^ 2) over my two planes
          sFs[c * NSP + (tid ^ 32)] = fma(a0_oh, fhi, a0_ol * flo);
        }
      }
      if (act && !S::A0X) {
#pragma unroll
        for (int a = 0; a < DS; ++a)
#pragma unroll
          for (int c = 0; c < M; ++c)
            sFs[(a * M + c) * PS + ((S::F1T && a == 1) ? p1t : px)] = F[a][c];
      }
      double d1t[M];                             // A1S: axis-1 derivative, transposed lane
      if (S::A1S) {
#pragma unroll
        for (int c = 0; c < M; ++c) {
          const double a1 = __shfl_sync(0xffffffffu, F[1][c], sig);
          double z1;
          dmma_8x8x4(d1t[c], z1, a1, bfrag, 0.0, 0.0);
        }
      }
      if (TS == 1 && S::DBUF && s > 0) {
        // time contraction of the previous slice, deferred past its DMMA latency
#pragma unroll
        for (int t = 0; t < (TS == 1 ? NQ : 1); ++t)
#pragma unroll
          for (int c = 0; c < M; ++c)
            accr[t][c] = (k == 1) ? P.ops.integ[t][0] * dvp[c] : fma(P.ops.integ[t][k - 1], dvp[c], accr[t][c]);
      }
      __syncthreads();
      double dv[M];
#pragma unroll
      for (int c = 0; c < M; ++c) {
        double part[DS];
#pragma unroll
        for (int a = 0; a < DS; ++a) {
          double v = 0.0;
          if (S::A0X && a == 0) {
            v = own0[c] + sFs[c * NSP + tid];    // + the other warp's two planes
          } else if (S::F1T && a == 1) {
            const double2* b2 = reinterpret_cast<const double2*>(sFs + (a * M + c) * PS + g1t);
#pragma unroll
            for (int jj = 0; jj < NQ / 2; ++jj) {
              const double2 w2 = b2[jj];
              v = fma(drow[a][2 * jj], w2.x, v);
              v = fma(drow[a][2 * jj + 1], w2.y, v);
            }
          } else {
            const double* b = sFs + (a * M + c) * PS + gbase[a];
#pragma unroll
            for (int j = 0; j < NQ; ++j) v = fma(drow[a][j], b[j * gstr[a]], v);
          }
          part[a] = v;
        }
        double sum = part[0];
#pragma unroll
        for (int a = 1; a < DS; ++a) sum += part[a];
        if (S::A1S) sum += __shfl_sync(0xffffffffu, d1t[c], sig);
        dv[c] = sum;
      }
      if (DMMA) {
#pragma unroll
        for (int c = 0; c < M; ++c) {
          double d1;
          dmma_8x8x4(dv[c], d1, F[2][c], bfrag, dv[c], 0.0);
        }
      }
      if (TS == 1 && S::DBUF) {
#pragma unroll
        for (int c = 0; c < M; ++c) dvp[c] = dv[c];
      } else if (TS == 1) {
#pragma unroll
        for (int t = 0; t < (TS == 1 ? NQ : 1); ++t)
#pragma unroll
          for (int c = 0; c < M; ++c)
            accr[t][c] = (k == 0) ? P.ops.integ[t][0] * dv[c] : fma(P.ops.integ[t][k], dv[c], accr[t][c]);
      } else if (act) {
#pragma unroll
        for (int c = 0; c < M; ++c) sDiv[(k * M + c) * NSP + x] = dv[c];
      }
      if (!(TS == 1 && S::DBUF)) __syncthreads();
    }
    if (TS == 1 && S::DBUF) {
#pragma unroll
      for (int t = 0; t < (TS == 1 ? NQ : 1); ++t)
#pragma unroll
        for (int c = 0; c < M; ++c) accr[t][c] = fma(P.ops.integ[t][NQ - 1], dvp[c], accr[t][c]);
    }
    BitMax bm;
#pragma unroll
    for (int c = 0; c < M; ++c) {
      double dvk[NQ];
      if (TS > 1) {
#pragma unroll
        for (int k = 0; k < NQ; ++k) dvk[k] = sDiv[(k * M + c) * NSP + x];
      }
#pragma unroll
      for (int s = 0; s < TH; ++s) {
        const int t = ts * TH + s;
        double acc = 0.0;
        if (TS == 1) {
          acc = accr[TS == 1 ? s : 0][c];
        } else {
#pragma unroll
          for (int k = 0; k < NQ; ++k) acc = fma(P.ops.integ[t][k], dvk[k], acc);
        }
        const double qn = Qx[c] - scale * acc;
        bm.add(fabs(qn - q[s][c]));
        q[s][c] = qn;
      }
    }
    iters = it + 1;
    const int fl = block_flags<NW>(!act || bm.conv(tol), act && bm.bad(), sFlags, it & 1);
    if (fl & 2) { failed = true; break; }
    if (fl & 1) break;
  }
  }

  // final flux: time average of the owned levels (partial fbar) + finiteness
  double fb[DIM][M];
#pragma unroll
  for (int a = 0; a < DIM; ++a)
#pragma unroll
    for (int c = 0; c < M; ++c) fb[a][c] = 0.0;
  if (!failed) {
    bool bad = false;
#pragma unroll
    for (int s = 0; s < TH; ++s) {
      const int t = ts * TH + s;
      double F[DIM][M];
      flux<DIM>(q[s], F);
#pragma unroll
      for (int a = 0; a < DIM; ++a)
#pragma unroll
        for (int c = 0; c < M; ++c) {
          bad |= !finite(F[a][c]);
          fb[a][c] = fma(P.ops.w[t], F[a][c], fb[a][c]);
        }
    }
    failed = __syncthreads_or(act && bad);
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

  // all time levels of q into sDiv's region: [t][c][NSP] in the trace layout
  double* sQt = sDiv;
  double* sQb = sDiv + NQ * M * NSP;                   // qbar [c][NSP] (trace layout)
  double* sFb = sF;                                    // [DIM][M][PS] total fbar
  const int qax = trace_addr<NQ>(i0, i1, i2);
  if (act) {
#pragma unroll
    for (int s = 0; s < TH; ++s)
#pragma unroll
      for (int c = 0; c < M; ++c) sQt[((ts * TH + s) * M + c) * NSP + qax] = q[s][c];
  }
  // fbar = sum over the TS partial time averages
  if (TS > 1) {
    if (ts == 1 && act) {
#pragma unroll
      for (int a = 0; a < DIM; ++a)
#pragma unroll
        for (int c = 0; c < M; ++c) sFb[(a * M + c) * PS + px] = fb[a][c];
    }
    __syncthreads();
    if (ts == 0 && act) {
#pragma unroll
      for (int a = 0; a < DIM; ++a)
#pragma unroll
        for (int c = 0; c < M; ++c) fb[a][c] += sFb[(a * M + c) * PS + px];
    }
    __syncthreads();
#pragma unroll
    for (int r = 2; r < TS; ++r) {
      if (ts == r && act) {
#pragma unroll
        for (int a = 0; a < DIM; ++a)
#pragma unroll
          for (int c = 0; c < M; ++c) sFb[(a * M + c) * PS + px] = fb[a][c];
      }
      __syncthreads();
      if (ts == 0 && act) {
#pragma unroll
        for (int a = 0; a < DIM; ++a)
#pragma unroll
          for (int c = 0; c < M; ++c) fb[a][c] += sFb[(a * M + c) * PS + px];
      }
      __syncthreads();
    }
  }
  if (ts == 0 && act) {
#pragma unroll
    for (int a = 0; a < DIM; ++a)
#pragma unroll
      for (int c = 0; c < M; ++c) sFb[(a * M + c) * PS + px] = fb[a][c];
  }
  if (tid < 2 * DIM) sSmax[tid] = 0ull;
  __syncthreads();

  // ---------------- integrate_volume (kernels.py:130-143) ----------------
  if (ts == 0 && act) {
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
  if (ts == 0 && act) {
#pragma unroll
    for (int c = 0; c < M; ++c) {
      double v = 0.0;
#pragma unroll
      for (int t = 0; t < NQ; ++t) v = fma(P.ops.w[t], sQt[(t * M + c) * NSP + qax], v);
      sQb[c * NSP + qax] = v;
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
      // (NQ = 4 keeps y fastest: its Latin-cube trace layout is conflict-free per face plane)
      const int side = (NQ == 4) ? e / (NQ * NF) : e & 1;
      const int y = (NQ == 4) ? e % NF : (e >> 1) % NF;
      const int t = (NQ == 4) ? (e / NF) % NQ : (e >> 1) / NF;
      const double* vec = side ? P.ops.right : P.ops.left;
      const int ya = y / NQ, yb = y % NQ;
      double qs[M];
#pragma unroll
      for (int c = 0; c < M; ++c) qs[c] = 0.0;
#pragma unroll
      for (int i = 0; i < NQ; ++i) {
        const int ad = (a == 0) ? trace_addr<NQ>(i, ya, yb)
                     : (a == 1) ? trace_addr<NQ>(ya, i, yb) : trace_addr<NQ>(ya, yb, i);
        const double v = vec[i];
#pragma unroll
        for (int c = 0; c < M; ++c) qs[c] = fma(v, sQt[(t * M + c) * NSP + ad], qs[c]);
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
      // side fastest at NQ != 4 (lane pairs share loads); NQ = 4 keeps y fastest
      const int side = (NQ == 4) ? e / (M * NF) : e & 1;
      const int y = (NQ == 4) ? e % NF : (e >> 1) % NF;
      const int c = (NQ == 4) ? (e / NF) % M : (e >> 1) / NF;
      const double* vec = side ? P.ops.right : P.ops.left;
      const int ya = y / NQ, yb = y % NQ;
      const int pxb = (a == 0) ? ya * P1 + yb : (a == 1) ? ya * P0 + yb : ya * P0 + yb * P1;
      double vq = 0.0, vf = 0.0;
#pragma unroll
      for (int i = 0; i < NQ; ++i) {
        const int ad = (a == 0) ? trace_addr<NQ>(i, ya, yb)
                     : (a == 1) ? trace_addr<NQ>(ya, i, yb) : trace_addr<NQ>(ya, yb, i);
        vq = fma(vec[i], sQb[c * NSP + ad], vq);
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
