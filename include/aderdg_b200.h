/* aderdg_b200.h — C ABI of the B200-native fused ADER-DG Euler step.
 *
 * This library replaces the reference's *driver seam* for the fused,
 * single-touch, optimistic time stepping of compressible Euler on a periodic
 * Cartesian grid.  One call advances whole grid sweeps on the GPU; there is no
 * per-cell or per-task call.  Each entry point names the reference interface
 * it stands in for (paths relative to /root/reference/pkg/src/aderdg/):
 *
 *   adg_create            Driver.__init__ + build_grid + Kernels.__init__ +
 *                         TimeControl.__init__      (scheduler.py:44-55,92-131;
 *                         mesh.py:167-243; kernels.py:46-60)
 *   adg_set_operators     make_basis(p) arrays consumed by Kernels.__init__
 *                         (basis.py:91-122; kernels.py:53-60)
 *   adg_load_state        filling grid.cells[i].Q   (tests/conftest.py:20-22)
 *   adg_store_state       reading grid.cells[i].Q   (tests/conftest.py:77-79)
 *   adg_seed              Driver._seed_time_control (scheduler.py:135-155)
 *   adg_step              Driver.step, fused mode   (scheduler.py:190-208,
 *                         370-449, incl. priming sweep and optimistic rerun)
 *   adg_run               Driver.run(steps=N)       (scheduler.py:210-218)
 *   adg_step_records      Driver.step_records       (scheduler.py:459-481)
 *   adg_error_info /      exception classes NumericalError /
 *   adg_last_error        PredictorFailureError(cell_index) (errors.py:28-39)
 *
 * Multi-GPU (x-slab decomposition, one process per GPU) uses the phase API
 * (adg_phase_*) plus adg_buffer() so that the host can run the halo exchange
 * and the lambda/error all-reduce with NCCL between phases.
 *
 * Conventions: all arrays are fp64, host pointers are borrowed for the
 * duration of the call, device buffers/streams belong to the handle.  State
 * layout = the reference's stack([c.Q for c in grid.cells]):
 * [cell (C-order over the cell multi-index)][i_0..i_{d-1}][component].
 * A handle is driven by one host thread.  Calls return an adg_status.
 */
#ifndef ADERDG_B200_H
#define ADERDG_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  ADG_OK = 0,
  ADG_ERR_CONFIG = 2,      /* ConfigurationError / ResourceBudgetError  */
  ADG_ERR_NUMERICAL = 3,   /* NumericalError                             */
  ADG_ERR_RUNTIME = 4,     /* CUDA runtime failure                        */
  ADG_ERR_PREDICTOR = 5    /* PredictorFailureError(cell_index)          */
} adg_status;

/* Numerical error kinds reported by adg_error_info (kind field). */
typedef enum {
  ADG_EK_NONE = 0,
  ADG_EK_INIT_INADMISSIBLE = 1, /* "initial data inadmissible in cell {c}"   scheduler.py:146-148 */
  ADG_EK_NO_INITIAL_STEP = 2,   /* "no admissible initial step (got {adm})"  scheduler.py:153-154 */
  ADG_EK_INADMISSIBLE = 3,      /* "inadmissible state in cell {c} at step {s}" scheduler.py:429-432 */
  ADG_EK_PREDICTOR = 4,         /* PredictorFailureError(c)                   kernels.py:80-100 */
  ADG_EK_DEGENERATE = 5,        /* "admissible step degenerated to {dt_adm}"  scheduler.py:81-82 */
  ADG_EK_SUBCELL = 6,           /* "subcell update left cell {c} inadmissible" limiter.py:214-216 */
  ADG_EK_STALE = 7,             /* debug library: a face record with the wrong sweep stamp was read
                                   (the reference's stale-hull checks, kernels.py:158-170,196-200) */
  ADG_EK_BOUNDS = 8             /* debug library: cell / record slot index out of bounds */
} adg_error_kind;

typedef struct {
  int d;                 /* 2 or 3                                         */
  int p;                 /* polynomial order, 0..9                         */
  int L;                 /* refinement depth: 3^L cells per axis, h = 3^-L */
  double cfl;            /* Kernels(cfl=0.9)                               */
  double c_dt;           /* TimeControl(c_dt=0.99)                         */
  int creeping;          /* TimeControl(averaging="creeping") if nonzero   */
  double forced_dt;      /* TimeControl(forced_dt=...); NaN = off          */
  int inject_rerun;      /* Driver(inject_rerun=True)                      */
  int spike_step;        /* Driver(spike_step=...); <0 = off               */
  double spike_factor;   /* Driver(spike_factor=3.0)                       */
  int device;            /* CUDA device ordinal                            */
  int rank;              /* slab index (0 for a single GPU)                */
  int world;             /* number of slabs along axis 0 (1 = periodic in place) */
  int halo_mode;         /* 0: halo slots iff world > 1; 1: always (world = 1 then exchanges with itself) */
  int driver_mode;       /* 0: fused single-touch (scheduler.py:370-449); 1: straightforward
                            (scheduler.py:230-313: predict pass, then Riemann/corrector pass,
                            dt = dt_new, no priming, no rerun)                               */
  int system;            /* PDE plug-in (pde.py:16-102): 0 EulerSystem(d), m = d+2;
                            1 AdvectionSystem(d, velocity), m = 1                            */
  double velocity[3];    /* AdvectionSystem velocity (first d used)        */
  int boundary;          /* build_grid(boundary=...) (mesh.py:167-231): 0 periodic; 1 outflow
                            (zero-gradient ghost traces, kernels.py:124-127; one slab)     */
} adg_config;

typedef struct {
  int step;              /* realisation step (1-based)                     */
  int reruns;            /* rerun passes booked on this step (0/1)         */
  double T;
  double dt_old;
  double dt_new;
  double dt_adm;
  long long picard_iters;  /* Picard iterations summed over all predicts of the step */
  long long predicts;      /* number of cell predictions in the step        */
  long long troubled;      /* cells handed to the subcell limiter (Driver.troubled_by_step,
                              scheduler.py:301-305); 0 without limiter      */
} adg_step_record;

typedef struct adg_handle adg_handle;

/* which buffer adg_buffer() returns */
typedef enum {
  ADG_BUF_Q = 0,         /* local state, [local cells][nodes][m]            */
  ADG_BUF_D = 1,         /* volume/face update D_h                           */
  ADG_BUF_TRACE0 = 2,    /* face-trace records, parity 0                     */
  ADG_BUF_TRACE1 = 3,    /* face-trace records, parity 1                     */
  ADG_BUF_REDUCE = 4     /* int64[2] = {lambda bits (max), INT64_MAX-err key (max)} */
} adg_buffer_id;

/* Layout queries for the halo exchange (multi-GPU). */
typedef struct {
  int n_cells_global;    /* 3^(d L)                                         */
  int n_cells_local;     /* cells of this slab                              */
  int cell_offset;       /* global index of the first local cell            */
  int planes_local;      /* axis-0 planes of this slab                      */
  int plane_cells;       /* 3^(L(d-1))                                      */
  int record_doubles;    /* doubles per face-side record                     */
  int faces_per_cell;    /* 2d                                               */
  size_t state_doubles;  /* n_cells_local * (p+1)^d * m                      */
} adg_layout;

adg_status adg_create(const adg_config* cfg, adg_handle** out);
void       adg_destroy(adg_handle* h);
adg_status adg_set_operators(adg_handle* h, const double* nodes, const double* weights,
                             const double* diff, const double* integ,
                             const double* left, const double* right);
/* Launch stream: a cudaStream_t (NULL = the legacy default stream).  Until this
 * is called the handle uses its own non-blocking stream. */
adg_status adg_set_stream(adg_handle* h, void* cuda_stream);
/* Back to the state right after adg_create: time control, counters, D and the
 * face records are cleared (Q is kept; load a new one with adg_load_state and
 * call adg_seed).  Used to restart an episode from the initial data. */
adg_status adg_reset(adg_handle* h);
adg_status adg_load_state(adg_handle* h, const double* Q, size_t n_doubles);
adg_status adg_store_state(adg_handle* h, double* Q, size_t n_doubles);
adg_status adg_seed(adg_handle* h);
adg_status adg_step(adg_handle* h, adg_step_record* out);
adg_status adg_run(adg_handle* h, int steps, adg_step_record* out);
/* records of steps first..first+count-1 (1-based; the last 4096 steps are kept) */
adg_status adg_step_records(adg_handle* h, int first, int count, adg_step_record* out);
adg_status adg_sync(adg_handle* h);
/* tc.dt_new = value before the next step (straightforward run(final_time) clamp,
 * scheduler.py:223-226) */
adg_status adg_set_dt_new(adg_handle* h, double value);
int        adg_step_count(const adg_handle* h);
int        adg_rerun_count(const adg_handle* h);
int        adg_sweep_count(const adg_handle* h);
adg_status adg_time_control(const adg_handle* h, double* T, double* dt_old,
                            double* dt_new, double* dt_adm);
adg_status adg_picard_histogram(const adg_handle* h, long long* hist, int n_bins);
adg_status adg_error_info(const adg_handle* h, int* kind, long long* cell, int* step, double* value);
const char* adg_last_error(const adg_handle* h);
adg_status adg_layout_info(const adg_handle* h, adg_layout* out);

/* SubcellLimiter(system, basis, grid, cfl) attached to a straightforward driver
 * (limiter.py:87-108, scheduler.py:100-102,239-309), one slab.  P [ns][n] =
 * subcell_average_matrix(basis), R [n][ns] = solve(P^T P, P^T), nearest [ns] =
 * node nearest to each subcell centre, sample [n] = min(int(nodes*ns), ns-1),
 * ns = 2p+1; traversal = the driver's cell order (NULL = lexicographic), which
 * fixes whose prev_Q the DMP test sees.  Call before the first step. */
adg_status adg_set_limiter(adg_handle* h, const double* P, const double* R, const int* nearest,
                           const int* sample, const long long* traversal, double cfl);
/* Cell.troubled of every local cell (mesh.py:39). */
adg_status adg_troubled_flags(adg_handle* h, unsigned char* out, size_t n);
adg_status adg_buffer(adg_handle* h, int which, void** dev_ptr, size_t* bytes);

/* Phase API (one process per GPU; the host drives NCCL between phases).
 * A realisation step is: rerun -> [halo exchange of the current parity] ->
 * sweep -> [all-reduce ADG_BUF_REDUCE with MAX] -> finish.  The priming sweep
 * (first step) is sweep(priming) -> [all-reduce] -> finish(priming). */
adg_status adg_phase_seed(adg_handle* h);      /* seed pass: fills ADG_BUF_REDUCE   */
adg_status adg_phase_seed_finish(adg_handle* h);
adg_status adg_phase_rerun(adg_handle* h);     /* device-conditional rerun predict  */
adg_status adg_phase_sweep(adg_handle* h);     /* priming on the first call          */
adg_status adg_phase_finish(adg_handle* h);    /* time control + step record         */
/* Overlapped slab step (the paper's transfer hiding):
 * rerun -> { halo exchange  ||  sweep_part(INTERIOR) } -> sweep_part(BOUNDARY)
 * -> all-reduce -> finish.  Interior planes (1..P-2) read no halo slot and
 * write no record a neighbour receives, so they run while the exchange of the
 * parity the sweep reads is in flight; the two boundary planes follow.  Both
 * parts (or ALL) must be enqueued before adg_phase_finish; the priming sweep
 * is ALL only.  The cells are independent, so split = whole sweep bitwise. */
typedef enum { ADG_PART_ALL = 0, ADG_PART_INTERIOR = 1, ADG_PART_BOUNDARY = 2 } adg_sweep_part;
adg_status adg_phase_sweep_part(adg_handle* h, int part);
int        adg_trace_parity(const adg_handle* h); /* parity the next sweep reads      */

/* Driver.step with the state in host memory: uploads Q_in, advances one
 * realisation step (fused driver, one slab), downloads the result into Q_out
 * (both [cells][nodes][m]; Q_in == Q_out allowed; pin them for overlap).  The
 * H2D, the sweep and the D2H are pipelined over chunks of cell planes, so the
 * transfers overlap the compute (a step with the priming sweep or a rerun
 * uploads all of Q first).  Synchronous at return. */
adg_status adg_step_host(adg_handle* h, const double* Q_in, double* Q_out, adg_step_record* out);

/* Timing helpers for bench.py: launches on the handle's stream. */
adg_status adg_flush_l2(adg_handle* h);
/* Enqueue `steps` realisation steps (single GPU) with CUDA events around the
 * whole segment and around every sweep-kernel launch; synchronises once.
 * out[0] = elapsed ms of the segment, out[1] = summed ms of the sweep-kernel
 * launches (rerun pass + sweep), both measured on the handle's stream. */
adg_status adg_run_timed(adg_handle* h, int steps, double* out);

/* adg_run_timed with options: flags & ADG_TIMED_KERNEL_EVENTS records CUDA events
 * around every rerun / sweep launch (out[1] = their summed ms; without it out[1] = 0
 * and the segment carries only its two bracketing events, which is what the
 * throughput number is measured on).  adg_run_timed = flags ADG_TIMED_KERNEL_EVENTS. */
#define ADG_TIMED_KERNEL_EVENTS 1
adg_status adg_run_timed_ex(adg_handle* h, int steps, int flags, double* out);

/* Multi-GPU steps enqueued from C (no per-step Python): the library opens its own
 * NCCL communicator (libnccl.so.2, resolved at run time) over the slab ranks.
 * adg_nccl_unique_id fills 128 bytes on rank 0 (ncclGetUniqueId); the host
 * broadcasts them; every rank calls adg_nccl_init.  adg_run_timed_mgpu then
 * enqueues `steps` overlapped slab steps (rerun -> { grouped ncclSend/ncclRecv of
 * the boundary face records on the comm stream || interior planes } -> boundary
 * planes -> ncclAllReduce MAX of ADG_BUF_REDUCE -> finish) with the same events
 * and outputs as adg_run_timed.  world = 1 with halo_mode = 1 exchanges with
 * itself (the single-GPU test of this path).  Replaces the Python per-step loop
 * of parallel.SlabDriver.enqueue_step. */
adg_status adg_nccl_unique_id(unsigned char* out128);
adg_status adg_nccl_init(adg_handle* h, const unsigned char* id128, int rank, int world);
adg_status adg_run_timed_mgpu(adg_handle* h, int steps, double* out);
/* adg_run_timed_mgpu with adg_run_timed_ex's flags. */
adg_status adg_run_timed_mgpu_ex(adg_handle* h, int steps, int flags, double* out);

/* In-process multi-GPU group: the reference's parallel driver seam
 * Driver(grid, kernels, tc, mode, parallel=True, n_workers=N) (src/scheduler.py:92-95,
 * 126-130, thread pool over cells) as N x-slab handles of one grid on N GPUs of one
 * process.  The caller creates handle i with cfg.rank = i, cfg.world = N and its own
 * cfg.device; adg_group_init opens one NCCL clique over them (ncclCommInitAll);
 * adg_group_seed / adg_group_run drive every handle from its own host thread with the
 * step sequence of adg_run_timed_mgpu (halo exchange hidden behind the interior
 * planes, MAX all-reduce of the step reduction).  out[k] = rank 0's records with the
 * Picard counts summed over ranks. */
adg_status adg_group_init(adg_handle** hs, int n);
adg_status adg_group_seed(adg_handle** hs, int n);
adg_status adg_group_run(adg_handle** hs, int n, int steps, adg_step_record* out);
/* Visible CUDA devices (0 without a driver / GPU). */
int adg_device_count(void);

/* Per-handle launch options (defaults in brackets):
 * ADG_OPT_GRAPH [1]       adg_run / adg_run_timed* capture their steps into one CUDA graph
 * ADG_OPT_COND_RERUN [1]  the rerun pass is a conditional graph node
 * ADG_OPT_HOST_CHUNKS [16] wave-aligned cell chunks of adg_step_host (1..81)
 * ADG_OPT_FUSE_FINISH [1] kernels that can (2D p = 3) run the step's time control in the last
 *                         CTA of the sweep launch instead of a separate launch (one slab)
 * ADG_OPT_PERSISTENT [1]  kernels that can (2D p = 3) run the step sequences of adg_run /
 *                         adg_run_timed in ONE cooperative launch with a grid barrier per step
 *                         (needs ADG_OPT_GRAPH 1; falls back to the step graph when the device
 *                         refuses the cooperative launch) */
#define ADG_OPT_GRAPH 1
#define ADG_OPT_COND_RERUN 2
#define ADG_OPT_HOST_CHUNKS 3
#define ADG_OPT_FUSE_FINISH 4
#define ADG_OPT_PERSISTENT 5
adg_status adg_set_option(adg_handle* h, int option, int value);

#ifdef __cplusplus
}
#endif
#endif /* ADERDG_B200_H */
