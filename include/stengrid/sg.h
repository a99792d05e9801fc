/*
 * stengrid/sg.h — the C ABI of the B200-native stencil engine
 * (libstengrid_b200.so). Plain pointers and sizes only; no torch or C++
 * types cross this boundary. Every entry point returns sg_status; on error
 * sg_last_error() holds a thread-local message (and, for SG_ERR_PENTA_SOLVE,
 * the failing system index).
 *
 * Each function names the reference interface it replaces
 * (/root/reference/proj/...). The reference is a C++ library with no FFI of
 * its own; this ABI is what its C++ API (re-implemented on top of it by the
 * headers in include/stengrid) and any ctypes/cffi binding call.
 *
 * Memory: grids are dense row-major (entry (i, j) at j*nx + i, grid.hpp:11-49).
 * A plan binds either HOST buffers (the plan owns device mirrors and moves
 * data according to the residency argument of sg_plan_compute) or DEVICE
 * buffers (zero-copy; kernels read/write them directly).
 */
#ifndef STENGRID_SG_H
#define STENGRID_SG_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SG_ABI_VERSION 1

typedef enum sg_status {
  SG_OK = 0,
  SG_ERR_INVALID_ARGUMENT = 1, /* std::invalid_argument (stencil.cpp:128-161,206-207) */
  SG_ERR_LOGIC = 2,            /* std::logic_error: destroyed plan (stencil.cpp:198,203) */
  SG_ERR_PENTA_SOLVE = 3,      /* PentaSolveError{system} (penta.hpp:51-55) */
  SG_ERR_DOMAIN = 4,           /* std::domain_error (cahn_hilliard.cpp:186,209) */
  SG_ERR_CUDA = 5,             /* CUDA runtime failure */
  SG_ERR_NO_DEVICE = 6         /* no CUDA device: there is no CPU fallback */
} sg_status;

typedef enum sg_direction { SG_DIR_X = 0, SG_DIR_Y = 1, SG_DIR_XY = 2 } sg_direction; /* stencil.hpp:35 */
typedef enum sg_boundary { SG_PERIODIC = 0, SG_NONPERIODIC = 1 } sg_boundary;         /* grid.hpp:64 */
typedef enum sg_dtype { SG_F64 = 0, SG_F32 = 1 } sg_dtype;
typedef enum sg_residency { SG_RESIDENCY_HOST = 0, SG_RESIDENCY_DEVICE = 1 } sg_residency; /* stencil.hpp:37-38 */
typedef enum sg_memory { SG_MEM_HOST = 0, SG_MEM_DEVICE = 1 } sg_memory;

/* Device twins of the reference's window functions (the reference passes a
 * host function pointer, stencil.hpp:20-25, which cannot run on a GPU). */
typedef enum sg_function {
  SG_FN_NONE = 0,                 /* weight stencil */
  SG_FN_CH_NONLINEAR = 1,         /* ch_nonlinear_window, cahn_hilliard.cpp:36-47 (3x3, 9 coe) */
  SG_FN_CENTRAL_DIFFERENCE = 2,   /* central_difference_window, tools/main.cpp:47-49 (3x1, 1 coe) */
  SG_FN_CENTER = 3,               /* fn_center, tests/test_stencil.cpp:68 (>=2x2, 0 coe) */
  SG_FN_CENTRAL_SECOND = 4,       /* fn_central_second, tests/test_stencil.cpp:70-77 (3x1, 1 coe) */
  SG_FN_LAP_CUBE_DIFF_FIRST = 5,  /* fn_lap_cube_diff_first, tests/test_stencil.cpp:79-85 (3x3, 2 coe) */
  SG_FN_WEIGHTED_3X3 = 6,         /* fn_weighted_3x3, tests/test_stencil.cpp:88-93 (3x3, 9 coe) */
  SG_FN_COUNT = 7,
  SG_FN_JIT_BASE = 1000           /* functions registered from source: 1000, 1001, ... */
} sg_function;

typedef struct sg_extents { int left, right, top, bottom; } sg_extents; /* grid.hpp:53-62 */

typedef struct sg_plan_s* sg_plan_t;

/* ---------------------------------------------------------------- library */
int sg_abi_version(void);
const char* sg_last_error(void);
int sg_last_error_system(void);
/* Number of kernels this library has launched in this process (all entry
 * points); used by bench.py to report gpu_launches. */
uint64_t sg_launch_count(void);
/* Initialise the CUDA context on `device` (cudaSetDevice); SG_ERR_NO_DEVICE
 * when no GPU is visible. */
sg_status sg_init(int device);
/* Minimum coefficient count a device window function reads; -1 if unknown. */
int sg_function_min_coe(int fn);
/* Name of a device window function ("ch_nonlinear_window", ...). */
const char* sg_function_name(int fn);
/* Register a window function from CUDA C++ SOURCE — the reference's
 * StencilFunction is arbitrary user code (stencil.hpp:20-25), which a GPU
 * cannot call through a host pointer. `body` is the body of
 *     template <typename T> T fn(const T* window, const T* coe, int rowStride)
 * (T = double, or float for FP32 plans; entry (p, q) of the window is
 * window[q*rowStride + p], exactly the reference's contract), e.g.
 *     "return (window[0] - 2.0 * window[1] + window[2]) * coe[0];"
 * It is compiled at run time by NVRTC for sm_100a with --fmad=false (the
 * reference's -ffp-contract=off) into the library's own stencil kernels,
 * once per (dtype, window shape, kernel) on first use; FP64 results equal a
 * host evaluation of the same expression bitwise. *fnId receives the id
 * (>= SG_FN_JIT_BASE) to pass as sg_plan_create's fn; any window is accepted
 * (the function must not read outside it, as in the reference), with up to
 * 256 coefficients. A body that does not compile returns
 * SG_ERR_INVALID_ARGUMENT with the compiler log in sg_last_error(). */
sg_status sg_register_function_source(const char* name, const char* body, int* fnId);

/* ----------------------------------------------------------- grid helpers */
/* wrap(i, n): grid.cpp:42-47. SG_ERR_INVALID_ARGUMENT if n <= 0. */
sg_status sg_wrap(int64_t i, int n, int* out);
/* make_tiles(ny, numTiles): grid.cpp:62-82; begins/ends hold numTiles ints. */
sg_status sg_make_tiles(int ny, int numTiles, int* begins, int* ends);

/* ---------------------------------------------------------- stencil plans
 * Replaces create_plan (stencil.hpp:90-92, stencil.cpp:152-184). fn ==
 * SG_FN_NONE selects a weight stencil with `count` weights (row-major W*H,
 * stencil.hpp:12-18); otherwise `values` is the coefficient array of the
 * device window function (FunctionStencil::coe, stencil.hpp:29-33).
 * numTiles keeps make_tiles validation (1 <= numTiles <= ny) and is the
 * y-slab count; numWorkers must be >= 1 (SPEC maps workers to devices).
 * Validation and error classes follow stencil.cpp:128-161 exactly. */
sg_status sg_plan_create(sg_direction dir, sg_boundary mode, sg_extents ext, sg_function fn,
                         const double* values, size_t count, sg_dtype dtype, void* in, void* out,
                         int nx, int ny, sg_memory memory, int numTiles, int numWorkers,
                         sg_plan_t* plan);
/* HOST grids whose two device mirrors would not fit in free device memory
 * (or any host plan with SG_STREAM_PLANS=1 in the environment at creation;
 * SG_STREAM_ROWS sets the chunk height) get a STREAMED plan: no mirrors,
 * every compute streams the grid through a ring of three row-chunk buffers
 * (chunk rows + halo rows; H2D, kernels and D2H overlapped on three
 * streams), so grids larger than HBM work — the reason for the paper's
 * tiling. Such a plan is always host-coherent and
 * synchronous (DEVICE residency behaves as HOST). */
/* compute (stencil.cpp:202-235). HOST residency: host grids are
 * authoritative — the input is uploaded, the output downloaded. DEVICE
 * residency: the input is uploaded only if its device copy is stale, the
 * output stays on the device until sg_plan_sync_to_host. `stream` is a
 * cudaStream_t (NULL = the plan's own stream, a blocking stream: it is
 * ordered after work queued on the legacy default stream, so device inputs
 * produced there are complete); `synchronize` != 0 blocks until the result
 * is complete (the reference's compute is synchronous). */
sg_status sg_plan_compute(sg_plan_t plan, sg_residency residency, void* stream, int synchronize);
/* swap_plan (stencil.cpp:197-200): exchange input and output bindings. */
sg_status sg_plan_swap(sg_plan_t plan);
/* destroy_plan (stencil.cpp:186-195): idempotent, never touches the grids;
 * *plan is set to NULL. */
sg_status sg_plan_destroy(sg_plan_t* plan);
/* Copy any device-resident bound grid back to its host buffer. */
sg_status sg_plan_sync_to_host(sg_plan_t plan);
/* Mark a host-bound grid as modified on the host (which = 0 input, 1 output). */
sg_status sg_plan_mark_host_dirty(sg_plan_t plan, int which);
/* Current bindings (which = 0 input, 1 output): host/device pointers. */
sg_status sg_plan_binding(sg_plan_t plan, int which, void** host_ptr, void** device_ptr);
/* 1 if the plan is valid (not destroyed). */
int sg_plan_valid(sg_plan_t plan);
/* Which kernel the plan dispatches to: 1 = register-strip fast path, 0 =
 * generic one-point-per-thread path. */
int sg_plan_kernel_kind(sg_plan_t plan);

/* numWorkers -> GPUs (SPEC.md:12 maps cuSten's deviceNum onto the workers).
 * A plan over HOST grids created with numWorkers = G > 1 splits the rows
 * into make_tiles(ny, G) y-slabs (grid.cpp:62-82), one per worker, each on
 * its own GPU with its own stream; every slab holds top/bottom halo rows.
 * compute() uploads each worker's rows plus halo rows straight from the
 * host grid (Residency::Host) or, for device-resident inputs, refreshes the
 * halos from the neighbouring workers by peer copies over NVLink; results
 * are bitwise those of one GPU. Device grids always run on their device.
 * Mode 0 ("clip", default): G = min(numWorkers, visible GPUs). Mode 1
 * ("modulo"): G = numWorkers, worker w on GPU w % visible GPUs (several
 * workers per GPU: exercises the multi-GPU path on a one-GPU box).
 * SG_DEVICE_MAP=modulo in the environment selects mode 1 at load. */
sg_status sg_set_device_map(int mode);
int sg_get_device_map(void);
/* Workers of a plan: count, and for the first `capacity` the GPU and the
 * global row range [rowBegin, rowEnd) each owns (1 worker for a one-GPU
 * plan). Any output pointer may be NULL. */
sg_status sg_plan_workers(sg_plan_t plan, int* workers, int* devices, int* rowBegins, int* rowEnds,
                          int capacity);

/* --------------------------------------------------------- slab launches
 * Stateless device launch used by the multi-GPU y-slab decomposition (and
 * internally by plans). Computes output rows [row0, row1) and columns
 * [col0, col1) of `out` (row pitch nx). Output row j reads input rows
 * j + inShift - top + q (q = 0..H-1), wrapped modulo inRows when wrapY,
 * from `in` (row pitch nx, inRows rows); columns wrap modulo nx when wrapX.
 * A slab stored with `h` halo rows above its own rows uses inShift = h. */
typedef struct sg_slab_desc {
  int nx;
  int inRows;
  int inShift;
  int row0, row1;
  int col0, col1;
  int wrapX, wrapY;
} sg_slab_desc;
sg_status sg_stencil_launch(const sg_slab_desc* desc, sg_extents ext, sg_function fn,
                            const double* values, size_t count, sg_dtype dtype, const void* in,
                            void* out, void* stream);
/* Same launch, fused with the halo exchange of the NEXT application: output
 * rows j < upRows are also stored to peerUp + j*nx (the up neighbour's
 * bottom halo rows, in its output buffer), rows j >= dnRow0 to
 * peerDn + (j - dnRow0)*nx (the down neighbour's top halo) — peer device
 * memory over NVLink (sg_ipc_*). NULL peers are skipped. The caller orders
 * the peers' writes with a barrier between applications. */
sg_status sg_stencil_launch_p2p(const sg_slab_desc* desc, sg_extents ext, sg_function fn, const double* values,
                                size_t count, sg_dtype dtype, const void* in, void* out, void* peerUp, int upRows,
                                void* peerDn, int dnRow0, void* stream);

/* --------------------------------------------------------- WENO5 advection
 * weno_advect (weno.cpp:50-94): out = -(u dphi/dx + v dphi/dy) with
 * fifth-order WENO upwind derivatives on a periodic grid, bitwise identical
 * to the reference. All four fields nx*ny row-major in `memory`; nx, ny >= 7. */
sg_status sg_weno_advect(const double* phi, const double* u, const double* v, int nx, int ny, double dx,
                         double dy, double* out, sg_memory memory, void* stream);

/* ---------------------------------------------------- pentadiagonal batch
 * PentaFactor / PeriodicPentaFactor (penta.hpp:57-100, penta.cpp:93-295) on
 * the device. Bands are interleaved (r*B + b, penta.hpp:12-20), `memory`
 * says where they live. The factorization runs on the device, one system per
 * thread; a zero pivot returns SG_ERR_PENTA_SOLVE with the system index. */
typedef struct sg_penta_s* sg_penta_t;
sg_status sg_penta_create(int batchCount, int n, int periodic, const double* secondSub,
                          const double* sub, const double* diag, const double* super,
                          const double* secondSuper, sg_memory memory, sg_penta_t* factor);
/* solve_in_place (penta.cpp:199-202, 289-295) on an interleaved rhs batch. */
sg_status sg_penta_solve(sg_penta_t factor, double* rhs, sg_memory memory, void* stream,
                         int synchronize);
sg_status sg_penta_destroy(sg_penta_t* factor);

/* ----------------------------------------------------- Cahn-Hilliard ADI
 * CHParams (cahn_hilliard.hpp:23-39) + CHStepper (:104-137). */
typedef struct sg_ch_params {
  double D, gamma, lx, ly, dt, T, icAmplitude;
  int nx, ny;
  uint64_t seed;
  int nonlinearEnabled;
} sg_ch_params;
typedef struct sg_ch_s* sg_ch_t;
/* CHParams defaults (D=1, gamma=0.01, 512^2, 2*pi box, seed 1, amp 0.1). */
void sg_ch_default_params(sg_ch_params* p);
/* CHParams::validate (cahn_hilliard.cpp:56-66). */
sg_status sg_ch_validate(const sg_ch_params* p);
/* CHStepper ctor (cahn_hilliard.cpp:213-241): initial condition generated on
 * the device from SplitMix64, C^{n-1} := C^n, factors built. */
sg_status sg_ch_create(const sg_ch_params* p, int numTiles, int numWorkers, sg_ch_t* ch);
/* numWorkers -> GPUs (as for plans, sg_set_device_map): with G > 1 the
 * stepper runs config 5's distributed step over G GPUs from this process —
 * y-slabs of ny/G rows; RHS + x-sweep on the rows each GPU owns; both
 * all-to-all transposes and the halo rows stored by the sweeps / combine
 * straight into the peers' buffers (peer access over NVLink), or moved by
 * peer copies when the sweep stage does not divide the slab. G is the
 * largest power of two <= the mapped worker count with >= 2 rows per slab.
 * Results are bitwise those of one GPU. field() gathers the slabs;
 * sg_ch_device_field returns a gathered copy on worker 0's GPU. */
sg_status sg_ch_workers(sg_ch_t ch, int* workers, int* p2p);
/* Extension (opt-in, single GPU): partitioned sweeps. With segments = P >= 2
 * every x / y system's unknowns are split into P segments solved as
 * independent chains (SPIKE-type: local solves with the segment factor,
 * a 4P x 4P interface system per system, a rank-4 correction per segment),
 * so the sequential recurrence per CTA is n / P rows instead of n — the
 * latency bound of the bitwise sweeps on grids with few systems per SM.
 * NOT bitwise equal to the reference (different operation order); the
 * deviation is measured in tests/test_ch_partition_gpu.py and DESIGN.md
 * against the north-star bar (1e-9 relative L2 after 100 steps).
 * segments = 0 or 1 restores the bitwise default. Needs nx % 64 == 0 and
 * segment lengths n / P that are multiples of 64. */
sg_status sg_ch_set_partition(sg_ch_t ch, int segments);
/* Block until every queued step is complete. */
sg_status sg_ch_synchronize(sg_ch_t ch);
/* `steps` calls of CHStepper::step (cahn_hilliard.cpp:260-328). */
sg_status sg_ch_step(sg_ch_t ch, int steps);
/* set_state (cahn_hilliard.cpp:251-258): host arrays nx*ny; resets step/time. */
sg_status sg_ch_set_state(sg_ch_t ch, const double* curr, const double* prev, sg_memory memory);
/* field() / previous_field(): which = 0 C^n, 1 C^{n-1}; copies nx*ny doubles. */
sg_status sg_ch_get_field(sg_ch_t ch, int which, double* out, sg_memory memory);
sg_status sg_ch_device_field(sg_ch_t ch, int which, const double** dptr);
sg_status sg_ch_status(sg_ch_t ch, int* step, double* time);
/* Restore the step counter (time = step*dt) after set_state, for exact
 * checkpoint resume; set_state itself resets it to 0 like the reference. */
sg_status sg_ch_set_step(sg_ch_t ch, int step);
sg_status sg_ch_destroy(sg_ch_t* ch);
/* CHStepper::diagnostics (cahn_hilliard.cpp:330-340) on the device-resident
 * C^n: t, s = s_metric, k1Inv = 1/k1_metric (0 for an all-zero field).
 * SG_ERR_DOMAIN when the mixture is saturated (s_metric throws). */
sg_status sg_ch_diagnostics(sg_ch_t ch, double* t, double* s, double* k1Inv);

/* ------------------------------------------------------ field diagnostics
 * simpson_mean (cahn_hilliard.cpp:161-177; square != 0: mean of v^2) and
 * s_metric (:179-188) — bitwise identical to the reference — and k1_metric
 * (:190-211; cuFFT + deterministic reduction, ~1e-13 relative). Fields are
 * row-major nx*ny in host or device memory. */
sg_status sg_simpson_mean(const double* field, int nx, int ny, int square, sg_memory memory, double* out);
sg_status sg_s_metric(const double* field, int nx, int ny, sg_memory memory, double* out);
sg_status sg_k1_metric(const double* field, int nx, int ny, double dx, double dy, sg_memory memory, double* out);

/* ------------------------------------- distributed Cahn-Hilliard (y-slabs)
 * One process per GPU; rank r owns rows [r*ny/world, (r+1)*ny/world) of both
 * time levels, stored as "ext" slabs with 2 halo rows above and below
 * ((own + 4) x nx, row-major). Per step the host (ch_dist.py) runs:
 *   halo exchange of both ext slabs (2 rows each way, periodic ring)
 *   sg_chd_phase_x   fused RHS + x-sweep + Woodbury-corrected transpose into
 *                    `send`, packed as world blocks of (own x nx/world)
 *   all-to-all       send -> ycol: rank q receives columns [q*nxq,(q+1)*nxq)
 *                    of every row, i.e. the (ny x nxq) y-sweep batch
 *   sg_chd_phase_y   y-sweep (nxq periodic systems of ny unknowns) in place
 *   all-to-all       ycol -> recv (packed like send)
 *   sg_chd_combine   C^{n+1} = (2C^n - C^{n-1}) + v over C^{n-1}; roles swap.
 * Replaces CHStepper::step (cahn_hilliard.cpp:260-328) across GPUs; the
 * arithmetic is identical, so fields are bitwise independent of world. */
typedef struct sg_chd_s* sg_chd_t;
sg_status sg_chd_create(const sg_ch_params* p, int world, int rank, sg_chd_t* h);
sg_status sg_chd_geometry(sg_chd_t h, int* own, int* nxq, int* r0);
sg_status sg_chd_init(sg_chd_t h, double* currExt, double* prevExt, void* stream);
sg_status sg_chd_phase_x(sg_chd_t h, const double* currExt, const double* prevExt, double* send, void* stream);
sg_status sg_chd_phase_y(sg_chd_t h, double* ycol, void* stream);
sg_status sg_chd_combine(sg_chd_t h, const double* currExt, double* prevExt, const double* recv, void* stream);
sg_status sg_chd_destroy(sg_chd_t* h);

/* P2P form of the same step: the two all-to-alls are fused into the sweeps.
 * Each sweep kernel TMA-stores every finished stage of its backward pass
 * straight into the buffer of the rank that consumes it (peer memory over
 * NVLink: IPC-mapped device pointers, sg_ipc_*), and writes its Woodbury
 * coefficients to every rank, so the exchange overlaps the recurrence; the
 * receiving sweep reads its input transposed with the x correction on load,
 * and the combine applies the y correction. Per step:
 *   halo exchange; sg_chd_phase_x_p2p; barrier (all ranks);
 *   sg_chd_phase_y_p2p; barrier; sg_chd_combine_p2p.
 * The barriers order the peers' writes (e.g. a one-element NCCL all-reduce
 * on the compute stream). Bitwise identical to the single-GPU stepper.
 * sg_chd_p2p_buffers returns this rank's receive buffers (to export);
 * sg_chd_set_peers takes every rank's, in rank order, and reports whether
 * the path can run (needs nx % 64 == 0, own and nx/world multiples of the
 * sweep stage height, world <= 8). */
sg_status sg_chd_p2p_buffers(sg_chd_t h, double** recvX, double** recvY, double** y4xAll, double** y4yAll);
sg_status sg_chd_set_peers(sg_chd_t h, double* const* recvX, double* const* recvY, double* const* y4xAll,
                           double* const* y4yAll, int* enabled);
sg_status sg_chd_phase_x_p2p(sg_chd_t h, const double* currExt, const double* prevExt, void* stream);
sg_status sg_chd_phase_y_p2p(sg_chd_t h, void* stream);
/* peerUpPrev / peerDnPrev (may be NULL): the up / down neighbours' ext slab
 * of the time level being written (their prevExt). The first 2 rows of
 * C^{n+1} also go into the up neighbour's bottom halo, the last 2 into the
 * down neighbour's top halo — the next step needs no halo exchange. */
sg_status sg_chd_combine_p2p(sg_chd_t h, const double* currExt, double* prevExt, double* peerUpPrev,
                             double* peerDnPrev, void* stream);

/* CUDA IPC (peer device memory across processes): a handle is 64 bytes and
 * names the allocation containing devPtr; *offset is devPtr's byte offset in
 * it (add it to the pointer sg_ipc_open_handle returns). */
sg_status sg_ipc_get_handle(const void* devPtr, void* handle64, size_t* offset);
sg_status sg_ipc_open_handle(const void* handle64, void** devPtr);
sg_status sg_ipc_close(void* devPtr);

#ifdef __cplusplus
}
#endif

#endif /* STENGRID_SG_H */
