// aderdg_limiter.cuh — a-posteriori subcell finite-volume limiter on sm_100a.
//
// The reference's SubcellLimiter (src/limiter.py:26-234) inside its
// straightforward driver (src/scheduler.py:239-309), src/ =
// /root/reference/pkg/src/aderdg/.  Per step, after the corrector pass:
//
//   lim_detect_kernel   one CTA per cell: troubled |= !admissible(Q) ||
//                       !admissible(P^d Q) || relaxed DMP against the
//                       prev_Q of the cell and its 2d face neighbours
//                       (limiter.py:138-160); troubled cells are listed.
//   lim_apply_kernel    persistent CTAs over the list: project prev_Q to
//                       (2p+1)^d subcells (or nearest-node samples), freeze
//                       the neighbours' projected boundary layers as halo,
//                       Rusanov FV sub-steps over dt, least-squares lift back
//                       with the cell mean restored, admissibility fallback
//                       to subcell samples (limiter.py:164-234); lambda of
//                       the new state (calc_time_step, kernels.py:216-229).
//   lim_lambda_kernel   max of the per-cell lambdas -> DevState (dt_adm).
//
// Traversal semantics (changes results, kept from the reference): prev_Q is
// refreshed cell by cell along the traversal inside Kernels.update and the
// DMP test of a cell runs right after its own update, so a neighbour at or
// before the cell in the traversal contributes Q^n (`cur`), a later one
// Q^(n-1) (`old`; zeros before the first update, mesh.py:90-96).
//
// This path is robustness, not throughput: troubled cells are few, so the
// apply kernel keeps its patches in per-CTA global scratch (L1/L2 resident)
// and runs scalar FP64 at any p; detection is one CTA per cell with the
// separable projection staged in shared memory.
#pragma once

#include "aderdg_kernels.cuh"

namespace adg {

struct LimParams {
  SweepParams sp;            // PDE plug-in parameters (advection velocity), ops.w
  const double* P;           // [ns][n]  subcell averages of the Lagrange basis (limiter.py:26-34)
  const double* R;           // [n][ns]  least-squares lift (P^T P)^-1 P^T (limiter.py:99)
  const int* nearest;        // [ns]     node nearest to each subcell centre (limiter.py:105-108)
  const int* sample;         // [n]      subcell holding each node (limiter.py:227-228)
  const int* rank;           // [cells]  traversal rank of each cell
  double* Q;                 // [cells][N][M]
  const double* cur;         // prev_Q written by this step's corrector (Q^n)
  const double* old;         // prev_Q of the previous step (Q^(n-1))
  unsigned char* troubled;   // [cells]
  int* list;                 // [cells]  troubled cells of this step
  double* lam;               // [cells]
  double* scratch;           // apply: per-CTA patches
  long long scratch_cta;     // doubles per CTA
  DevState* st;
  int n, ns, K, n_cells;
  int outflow;               // boundary faces have no neighbour (mesh.py:139-146 -> None)
  double h_sub, cfl;
};

__device__ __forceinline__ long long ipow_ll(int b, int e) {
  long long r = 1;
  for (int i = 0; i < e; ++i) r *= b;
  return r;
}

// neighbour of `cell` across face f (axis f/2, low side for even f): periodic,
// or -1 across an outflow boundary (Grid.cell_neighbors -> None)
template <int DIM>
__device__ __forceinline__ int face_neighbour(int cell, int f, int K, int outflow) {
  const int a = f >> 1;
  int st = 1;
  for (int b = DIM - 1; b > a; --b) st *= K;
  const int ia = (cell / st) % K;
  if (outflow && ((f & 1) ? ia == K - 1 : ia == 0)) return -1;
  const int ja = (f & 1) ? (ia + 1) % K : (ia + K - 1) % K;
  return cell + (ja - ia) * st;
}

// y = Mat applied along `axis` of x: x has extents ext[0..DIM-1] then M
// components (C-order), Mat is rows x ext[axis]; y has ext[axis] -> rows.
template <int DIM, int M>
__device__ void apply_axis(const double* __restrict__ x, double* __restrict__ y, const int (&ext)[DIM],
                           int axis, const double* __restrict__ Mat, int rows) {
  int inner = M;
  for (int b = DIM - 1; b > axis; --b) inner *= ext[b];
  int outer = 1;
  for (int b = 0; b < axis; ++b) outer *= ext[b];
  const int kx = ext[axis];
  const int total = outer * rows * inner;
  for (int e = threadIdx.x; e < total; e += blockDim.x) {
    const int i = e % inner;
    const int r = (e / inner) % rows;
    const int o = e / (inner * rows);
    const double* xs = x + (long long)o * kx * inner + i;
    double acc = 0.0;
    for (int k = 0; k < kx; ++k) acc = fma(Mat[r * kx + k], xs[(long long)k * inner], acc);
    y[e] = acc;
  }
}

// admissibility of `count` states (pde.py:59-67); block-uniform result
template <class PDE>
__device__ bool block_admissible(const double* x, int count, const SweepParams& sp) {
  bool ok = true;
  for (int s = threadIdx.x; s < count; s += blockDim.x) {
    double q[PDE::M];
#pragma unroll
    for (int c = 0; c < PDE::M; ++c) q[c] = x[(long long)s * PDE::M + c];
    double lam = 0.0;
    ok = ok && PDE::node_lambda(q, lam, sp);
  }
  return __syncthreads_and(ok) != 0;
}

// max signal speed over `count` states and all axes (kernels.py:224-226); NaN-free inputs
template <class PDE, int DIM>
__device__ double block_lambda(const double* x, int count, const SweepParams& sp, double* red) {
  double lam = 0.0;
  for (int s = threadIdx.x; s < count; s += blockDim.x) {
    double q[PDE::M];
#pragma unroll
    for (int c = 0; c < PDE::M; ++c) q[c] = x[(long long)s * PDE::M + c];
#pragma unroll
    for (int a = 0; a < DIM; ++a) lam = fmax(lam, PDE::trace_speed(q, a, sp));
  }
  for (int o = 16; o > 0; o >>= 1) lam = fmax(lam, __shfl_xor_sync(0xffffffffu, lam, o));
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = lam;
  __syncthreads();
  double r = 0.0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) r = fmax(r, red[w]);
  __syncthreads();
  return r;
}

// per-component min / max over `count` states into lo[M] / hi[M] (combined)
template <int M>
__device__ void block_minmax(const double* x, int count, double* lo, double* hi, double* red) {
  double mn[M], mx[M];
#pragma unroll
  for (int c = 0; c < M; ++c) { mn[c] = INFINITY; mx[c] = -INFINITY; }
  for (int s = threadIdx.x; s < count; s += blockDim.x) {
#pragma unroll
    for (int c = 0; c < M; ++c) {
      const double v = x[(long long)s * M + c];
      mn[c] = fmin(mn[c], v);
      mx[c] = fmax(mx[c], v);
    }
  }
  const int nw = blockDim.x >> 5, w = threadIdx.x >> 5;
#pragma unroll
  for (int c = 0; c < M; ++c) {
    for (int o = 16; o > 0; o >>= 1) {
      mn[c] = fmin(mn[c], __shfl_xor_sync(0xffffffffu, mn[c], o));
      mx[c] = fmax(mx[c], __shfl_xor_sync(0xffffffffu, mx[c], o));
    }
  }
  __syncthreads();
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int c = 0; c < M; ++c) { red[(2 * c) * nw + w] = mn[c]; red[(2 * c + 1) * nw + w] = mx[c]; }
  }
  __syncthreads();
  if (threadIdx.x < M) {
    const int c = threadIdx.x;
    double a = lo[c], b = hi[c];
    for (int k = 0; k < nw; ++k) { a = fmin(a, red[(2 * c) * nw + k]); b = fmax(b, red[(2 * c + 1) * nw + k]); }
    lo[c] = a;
    hi[c] = b;
  }
  __syncthreads();
}

// ---------------------------------------------------------------------------
// detection (limiter.py:138-160, scheduler.py:282-284): one CTA per cell.
// shared: [A | B/Qstage] with A = ns*n^(d-1)*M, B = max(n^d, ns^2 n^(d-2)) * M,
// + reductions.
template <class PDE, int DIM>
__global__ void __launch_bounds__(256) lim_detect_kernel(const LimParams L) {
  constexpr int M = PDE::M;
  extern __shared__ double sm[];
  ADG_DEBUG_POISON();
  DevState* st = L.st;
  if (st->status != 0 || st->reduce[1] != 0) return;
  const int cell = blockIdx.x;
  const int n = L.n, ns = L.ns;
  const int N = (int)ipow_ll(n, DIM);
  const long long NM = (long long)N * M;
  if (L.troubled[cell]) {                       // bool(cell.troubled) or ... (short-circuit)
    if (threadIdx.x == 0) L.list[atomicAdd((unsigned long long*)&st->lim_count, 1ull)] = cell;
    return;
  }
  const int szA = ns * (int)ipow_ll(n, DIM - 1) * M;
  double* A = sm;
  double* B = A + szA;
  const int szB = (int)((DIM == 3 ? (long long)ns * ns * n : (long long)n * n) * M);
  const int szB2 = (int)(NM > szB ? NM : szB);
  double* red = B + szB2;                        // 2*M*8 doubles + 8 + 4M
  double* lo = red + 2 * M * 8;
  double* hi = lo + M;
  double* clo = hi + M;
  double* chi = clo + M;
  const double* Qg = L.Q + (long long)cell * NM;
  for (int e = threadIdx.x; e < NM; e += blockDim.x) B[e] = Qg[e];
  __syncthreads();
  bool troubled = !block_admissible<PDE>(B, N, L.sp);
  if (threadIdx.x < M) {
    lo[threadIdx.x] = INFINITY; hi[threadIdx.x] = -INFINITY;
    clo[threadIdx.x] = INFINITY; chi[threadIdx.x] = -INFINITY;
  }
  __syncthreads();
  if (!troubled) {
    block_minmax<M>(B, N, clo, chi, red);        // min/max of the nodal Q
    // separable projection P^d Q, last axis streamed
    int ext[DIM];
    for (int a = 0; a < DIM; ++a) ext[a] = n;
    apply_axis<DIM, M>(B, A, ext, 0, L.P, ns);   // axis 0: B (Q) -> A
    __syncthreads();
    ext[0] = ns;
    const double* last = A;
    if (DIM == 3) {
      apply_axis<DIM, M>(A, B, ext, 1, L.P, ns); // axis 1: A -> B (Q no longer needed)
      __syncthreads();
      ext[1] = ns;
      last = B;
    }
    // final axis: each thread one subcell, all M components
    const int nsub = (int)ipow_ll(ns, DIM);
    bool ok = true;
    double mn[M], mx[M];
#pragma unroll
    for (int c = 0; c < M; ++c) { mn[c] = INFINITY; mx[c] = -INFINITY; }
    for (int s = threadIdx.x; s < nsub; s += blockDim.x) {
      const int sl = s % ns, head = s / ns;
      double q[M];
#pragma unroll
      for (int c = 0; c < M; ++c) {
        double acc = 0.0;
        for (int k = 0; k < n; ++k) acc = fma(L.P[sl * n + k], last[((long long)head * n + k) * M + c], acc);
        q[c] = acc;
        mn[c] = fmin(mn[c], acc);
        mx[c] = fmax(mx[c], acc);
      }
      double lam = 0.0;
      ok = ok && PDE::node_lambda(q, lam, L.sp);
    }
    troubled = !__syncthreads_and(ok);
    if (!troubled) {
      // combine the patch min/max into clo/chi (reuse block_minmax's reduction)
      const int nw = blockDim.x >> 5, w = threadIdx.x >> 5;
#pragma unroll
      for (int c = 0; c < M; ++c)
        for (int o = 16; o > 0; o >>= 1) {
          mn[c] = fmin(mn[c], __shfl_xor_sync(0xffffffffu, mn[c], o));
          mx[c] = fmax(mx[c], __shfl_xor_sync(0xffffffffu, mx[c], o));
        }
      if ((threadIdx.x & 31) == 0)
#pragma unroll
        for (int c = 0; c < M; ++c) { red[(2 * c) * nw + w] = mn[c]; red[(2 * c + 1) * nw + w] = mx[c]; }
      __syncthreads();
      if (threadIdx.x < M) {
        const int c = threadIdx.x;
        for (int k = 0; k < nw; ++k) {
          clo[c] = fmin(clo[c], red[(2 * c) * nw + k]);
          chi[c] = fmax(chi[c], red[(2 * c + 1) * nw + k]);
        }
      }
      __syncthreads();
      // relaxed DMP range: own prev_Q (= Q^n) and the 2d face neighbours
      block_minmax<M>(L.cur + (long long)cell * NM, N, lo, hi, red);
      const int r0 = L.rank[cell];
      for (int f = 0; f < 2 * DIM; ++f) {
        const int nb = face_neighbour<DIM>(cell, f, L.K, L.outflow);
        if (nb < 0) continue;                    // limiter.py:150-151
        const double* src = (L.rank[nb] <= r0) ? L.cur : L.old;
        block_minmax<M>(src + (long long)nb * NM, N, lo, hi, red);
      }
      bool viol = false;
      if (threadIdx.x < M) {
        const int c = threadIdx.x;
        const double delta = 1e-3 + 1e-2 * (hi[c] - lo[c]);      // DMP_ABS + DMP_REL (hi - lo)
        viol = (clo[c] < lo[c] - delta) || (chi[c] > hi[c] + delta);
      }
      troubled = __syncthreads_or(viol) != 0;
    }
  }
  if (troubled && threadIdx.x == 0) {
    L.troubled[cell] = 1;
    L.list[atomicAdd((unsigned long long*)&st->lim_count, 1ull)] = cell;
  }
}

// project a nodal block (n^d x M) to subcells (ns^d x M): x -> y via t1/t2
template <int DIM, int M>
__device__ void project_full(const double* x, double* y, double* t1, double* t2, const double* Pm, int n,
                             int ns) {
  int ext[DIM];
  for (int a = 0; a < DIM; ++a) ext[a] = n;
  const double* src = x;
  for (int a = 0; a < DIM; ++a) {
    double* dst = (a == DIM - 1) ? y : ((a & 1) ? t2 : t1);
    apply_axis<DIM, M>(src, dst, ext, a, Pm, ns);
    __syncthreads();
    ext[a] = ns;
    src = dst;
  }
}

// src/limiter.py:164-175 — exact projection when physical, else nearest-node samples
template <class PDE, int DIM>
__device__ void start_patch(const double* Qn, double* y, double* t1, double* t2, const LimParams& L) {
  constexpr int M = PDE::M;
  project_full<DIM, M>(Qn, y, t1, t2, L.P, L.n, L.ns);
  const int nsub = (int)ipow_ll(L.ns, DIM);
  if (block_admissible<PDE>(y, nsub, L.sp)) return;
  for (int e = threadIdx.x; e < nsub * M; e += blockDim.x) {
    const int c = e % M;
    int s = e / M, node = 0, mul = 1;
    for (int a = DIM - 1; a >= 0; --a) {
      node += L.nearest[s % L.ns] * mul;
      mul *= L.n;
      s /= L.ns;
    }
    y[e] = Qn[(long long)node * M + c];
  }
  __syncthreads();
}

// Rusanov flux between states l and r along axis a (limiter.py:72-78)
template <class PDE, int DIM>
__device__ __forceinline__ void fv_flux(const double (&l)[PDE::M], const double (&r)[PDE::M], int a,
                                        const SweepParams& sp, double (&out)[PDE::M]) {
  constexpr int M = PDE::M;
  double Fl[DIM][M], Fr[DIM][M];
  PDE::flux(l, Fl, sp);
  PDE::flux(r, Fr, sp);
  const double alpha = fmax(PDE::trace_speed(l, a, sp), PDE::trace_speed(r, a, sp));
#pragma unroll
  for (int c = 0; c < M; ++c)
    out[c] = __dsub_rn(__dmul_rn(0.5, __dadd_rn(Fl[a][c], Fr[a][c])),
                       __dmul_rn(__dmul_rn(0.5, alpha), __dsub_rn(r[c], l[c])));
}

// ---------------------------------------------------------------------------
// apply (limiter.py:196-234 + scheduler.py:306-309): persistent CTAs over the list.
// scratch per CTA: A, B (patch ping-pong), Y (projection output), T1, T2
// (separable intermediates), each ns^d * M, then H = 2d * ns^(d-1) * M.
constexpr int LIM_SCRATCH_PATCHES = 5;

template <class PDE, int DIM>
__global__ void __launch_bounds__(256) lim_apply_kernel(const LimParams L) {
  constexpr int M = PDE::M;
  constexpr int NWMAX = 8;
  __shared__ double red[2 * M * NWMAX + NWMAX];
  DevState* st = L.st;
  if (st->status != 0 || st->reduce[1] != 0) return;
  const int count = (int)st->lim_count;
  const double dt = st->dt_new;                  // the step's dt (straightforward: dt = tc.dt_new)
  const int n = L.n, ns = L.ns;
  const int N = (int)ipow_ll(n, DIM);
  const long long NM = (long long)N * M;
  const int nsub = (int)ipow_ll(ns, DIM);
  const int nlay = nsub / ns;
  const long long SZ = (long long)nsub * M;
  double* const base = L.scratch + blockIdx.x * L.scratch_cta;
  double* Y = base + 2 * SZ;
  double* T1 = base + 3 * SZ;
  double* T2 = base + 4 * SZ;
  double* H = base + 5 * SZ;                     // [2d][ns^(d-1)][M]
  const double h_sub = L.h_sub;
  const int nw = blockDim.x >> 5, wid = threadIdx.x >> 5;
  for (int li = blockIdx.x; li < count; li += gridDim.x) {
    const int cell = L.list[li];
    double* A = base;
    double* B = base + SZ;
    // ---- rollback patch and frozen halo (limiter.py:177-194) ----
    start_patch<PDE, DIM>(L.cur + (long long)cell * NM, A, T1, T2, L);
    for (int f = 0; f < 2 * DIM; ++f) {
      const int a = f >> 1;
      const int nb = face_neighbour<DIM>(cell, f, L.K, L.outflow);
      const double* Ysrc = A;                    // boundary: zero-gradient copy of the own edge
      int lay = (f & 1) ? ns - 1 : 0;
      if (nb >= 0) {
        start_patch<PDE, DIM>(L.cur + (long long)nb * NM, Y, T1, T2, L);
        Ysrc = Y;
        lay = (f & 1) ? 0 : ns - 1;              // low face: neighbour's last layer; high: its first
      }
      int inner = 1;
      for (int b = DIM - 1; b > a; --b) inner *= ns;
      for (int e = threadIdx.x; e < nlay * M; e += blockDim.x) {
        const int c = e % M, t = e / M;
        const int i = t % inner, o = t / inner;
        H[(long long)f * nlay * M + e] = Ysrc[(((long long)o * ns + lay) * inner + i) * M + c];
      }
      __syncthreads();
    }
    // ---- FV sub-steps over dt (limiter.py:203-217, rusanov_fv_step :41-84) ----
    bool failed = false;
    double remaining = dt;
    while (remaining > 1e-15 * dt) {
      const double lam = block_lambda<PDE, DIM>(A, nsub, L.sp, red);
      double dt_sub = remaining;
      if (!(lam <= 0.0)) dt_sub = fmin(remaining, __ddiv_rn(__dmul_rn(L.cfl, h_sub), __dmul_rn((double)DIM, lam)));
      const double cf = __ddiv_rn(dt_sub, h_sub);
      for (int s = threadIdx.x; s < nsub; s += blockDim.x) {
        double q[M], out[M];
#pragma unroll
        for (int c = 0; c < M; ++c) { q[c] = A[(long long)s * M + c]; out[c] = q[c]; }
        int idx[DIM];
        {
          int rest = s;
          for (int a = DIM - 1; a >= 0; --a) { idx[a] = rest % ns; rest /= ns; }
        }
        int st_a = nsub;
        for (int a = 0; a < DIM; ++a) {
          st_a /= ns;
          int lin = 0;                           // position inside the layer perpendicular to a
          for (int b = 0; b < DIM; ++b)
            if (b != a) lin = lin * ns + idx[b];
          double lft[M], rgt[M], fl[M], fh[M];
#pragma unroll
          for (int c = 0; c < M; ++c) {
            lft[c] = (idx[a] > 0) ? A[(long long)(s - st_a) * M + c] : H[((long long)(2 * a) * nlay + lin) * M + c];
            rgt[c] = (idx[a] < ns - 1) ? A[(long long)(s + st_a) * M + c]
                                       : H[((long long)(2 * a + 1) * nlay + lin) * M + c];
          }
          fv_flux<PDE, DIM>(lft, q, a, L.sp, fl);
          fv_flux<PDE, DIM>(q, rgt, a, L.sp, fh);
#pragma unroll
          for (int c = 0; c < M; ++c) out[c] = __dsub_rn(out[c], __dmul_rn(cf, __dsub_rn(fh[c], fl[c])));
        }
#pragma unroll
        for (int c = 0; c < M; ++c) B[(long long)s * M + c] = out[c];
      }
      __syncthreads();
      if (!block_admissible<PDE>(B, nsub, L.sp)) {          // limiter.py:213-216
        if (threadIdx.x == 0)
          report_error(st, SUBCELL_KEY | ((long long)L.rank[cell] << SUBCELL_CELL_BITS) | (long long)cell);
        failed = true;
        break;
      }
      double* t = A; A = B; B = t;
      remaining = __dsub_rn(remaining, dt_sub);
    }
    if (failed) break;
    // ---- reconstruct (limiter.py:119-134): R along every axis, cell mean restored ----
    {
      int ext[DIM];
      for (int a = 0; a < DIM; ++a) ext[a] = ns;
      const double* src = A;
      for (int a = 0; a < DIM; ++a) {
        double* dst = (a == DIM - 1) ? B : ((a & 1) ? T2 : T1);
        apply_axis<DIM, M>(src, dst, ext, a, L.R, n);
        __syncthreads();
        ext[a] = n;
        src = dst;
      }
    }
    {
      double ps[M], qs[M];
#pragma unroll
      for (int c = 0; c < M; ++c) { ps[c] = 0.0; qs[c] = 0.0; }
      for (int s = threadIdx.x; s < nsub; s += blockDim.x)
#pragma unroll
        for (int c = 0; c < M; ++c) ps[c] += A[(long long)s * M + c];
      for (int x = threadIdx.x; x < N; x += blockDim.x) {
        int idx[DIM];
        int r = x;
        for (int a = DIM - 1; a >= 0; --a) { idx[a] = r % n; r /= n; }
        double w = 1.0;                          // mean_weights: prod_a w[i_a] (limiter.py:101-104)
        for (int a = 0; a < DIM; ++a) w = w * L.sp.ops.w[idx[a]];
#pragma unroll
        for (int c = 0; c < M; ++c) qs[c] += w * B[(long long)x * M + c];
      }
#pragma unroll
      for (int c = 0; c < M; ++c)
        for (int o = 16; o > 0; o >>= 1) {
          ps[c] += __shfl_xor_sync(0xffffffffu, ps[c], o);
          qs[c] += __shfl_xor_sync(0xffffffffu, qs[c], o);
        }
      if ((threadIdx.x & 31) == 0)
#pragma unroll
        for (int c = 0; c < M; ++c) { red[c * NWMAX + wid] = ps[c]; red[(M + c) * NWMAX + wid] = qs[c]; }
      __syncthreads();
      if (threadIdx.x < M) {                     // fixed summation order (deterministic)
        const int c = threadIdx.x;
        double a = 0.0, b = 0.0;
        for (int k = 0; k < nw; ++k) { a += red[c * NWMAX + k]; b += red[(M + c) * NWMAX + k]; }
        red[c * NWMAX] = __dsub_rn(__ddiv_rn(a, (double)nsub), b);
      }
      __syncthreads();
      for (int e = threadIdx.x; e < NM; e += blockDim.x) B[e] = __dadd_rn(B[e], red[(e % M) * NWMAX]);
      __syncthreads();
    }
    bool ok = block_admissible<PDE>(B, N, L.sp);
    if (ok) {
      project_full<DIM, M>(B, Y, T1, T2, L.P, n, ns);
      ok = block_admissible<PDE>(Y, nsub, L.sp);
    }
    double* Qg = L.Q + (long long)cell * NM;
    if (ok) {
      for (int e = threadIdx.x; e < NM; e += blockDim.x) Qg[e] = B[e];
    } else {
      // raw subcell means sampled at the nodes (limiter.py:225-233)
      for (int e = threadIdx.x; e < NM; e += blockDim.x) {
        const int c = e % M;
        int x = e / M, sub = 0, mul = 1;
        for (int a = DIM - 1; a >= 0; --a) {
          sub += L.sample[x % n] * mul;
          mul *= ns;
          x /= n;
        }
        Qg[e] = A[(long long)sub * M + c];
      }
    }
    __syncthreads();
    // calc_time_step of the limited cell (scheduler.py:307-309)
    {
      bool adm = true;
      double lam = 0.0;
      for (int x = threadIdx.x; x < N; x += blockDim.x) {
        double q[M];
#pragma unroll
        for (int c = 0; c < M; ++c) q[c] = Qg[(long long)x * M + c];
        adm = PDE::node_lambda(q, lam, L.sp) && adm;
      }
      const bool all = __syncthreads_and(adm) != 0;
      for (int o = 16; o > 0; o >>= 1) lam = fmax(lam, __shfl_xor_sync(0xffffffffu, lam, o));
      if ((threadIdx.x & 31) == 0) red[2 * M * NWMAX + wid] = lam;
      __syncthreads();
      if (threadIdx.x == 0) {
        double r = 0.0;
        for (int w = 0; w < nw; ++w) r = fmax(r, red[2 * M * NWMAX + w]);
        L.lam[cell] = all ? r : 0.0;
        L.troubled[cell] = ok ? 0 : 1;
      }
      __syncthreads();
    }
  }
}

// dt_adm = min over cells (inf for inadmissible ones) == max of lambda
__global__ void __launch_bounds__(256) lim_lambda_kernel(const double* lam, int n_cells, DevState* st) {
  if (st->status != 0 || st->reduce[1] != 0) return;
  double v = 0.0;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n_cells; i += gridDim.x * blockDim.x)
    v = fmax(v, lam[i]);
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) atomicMax(&st->reduce[0], __double_as_longlong(v));
}

}  // namespace adg
