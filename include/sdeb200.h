/* sdeb200 -- C ABI of the B200-native ensemble SDE integrator.
 *
 * The reference (sdebatch, pure Python/numpy) has no C ABI or plugin
 * registry: its hot path sits behind Python functions.  Each entry point
 * below names the reference interface it replaces (paths relative to
 * /root/reference/pkg/src/sdebatch).  The Python package
 * paper_1908_03869_b200 binds this ABI with ctypes.
 *
 * Conventions
 *  - Plain pointers and sizes only; no torch or Python types cross the ABI.
 *  - Host arrays are C-order float64 / uint32 / uint64 / int64 owned by the
 *    caller.  "_device" entry points take device pointers plus a cudaStream_t
 *    passed as void*.
 *  - Status codes: SDB_OK, or an error whose message sdb_last_error(ctx)
 *    returns (ctx may be NULL for context-free calls; the message is then
 *    thread-local).  Per-orbit solver failures are data (fail_step), not errors.
 *  - A context is used by one host thread at a time.
 */
#ifndef SDEB200_H
#define SDEB200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SDB_ABI_VERSION 2

typedef enum sdb_status {
    SDB_OK = 0,
    SDB_ERR_CONFIG = 1,      /* maps to ConfigError (engine.py:40) */
    SDB_ERR_UNSUPPORTED = 2, /* maps to NotImplementedError */
    SDB_ERR_CUDA = 3,        /* maps to RuntimeError */
    SDB_ERR_ARGUMENT = 4     /* maps to ValueError */
} sdb_status;

enum { SDB_MODEL_KURAMOTO = 1,                   /* model.py:188-220 */
       SDB_MODEL_EXPRESSION = 2 };               /* model_from_dsl, model.py:291-309 */
enum { SDB_SOLVER_EM = 0, SDB_SOLVER_EULER = 1, SDB_SOLVER_RK4 = 2 }; /* solvers.py:369-375 */
enum { SDB_STREAM_PHILOX = 0, SDB_STREAM_SFC64 = 1, SDB_STREAM_XOSHIRO256PP = 2 };
/* How the coupling sum S_i = sum_j sin(y_j - y_i) (model.py:193-195) is evaluated:
 * MEANFIELD: S_i = cos(y_i) * sum_j sin(y_j) - sin(y_i) * sum_j cos(y_j)  (O(n));
 * PAIRWISE : every term sin(fl(y_j - y_i)) as the reference rounds it (O(n^2)). */
enum { SDB_COUPLING_MEANFIELD = 0, SDB_COUPLING_PAIRWISE = 1 };

typedef struct sdb_ctx sdb_ctx;
typedef struct sdb_model sdb_model;

/* One integration run: the fields of EngineConfig (engine.py:44-64) that the
 * device needs, after the host has validated them (engine.py:66-80,
 * 192-208) and computed chunks = iteration_count(...) (engine.py:126-142). */
typedef struct sdb_desc {
    int32_t model;        /* SDB_MODEL_KURAMOTO, or SDB_MODEL_EXPRESSION for sdb_run_model */
    int32_t nequat;       /* n oscillators */
    int32_t nparams;      /* row length of params: (K, omega_1..n[, s_1..n, ...]) */
    int32_t nnoise;       /* n (stochastic) or 0 (ODE) */
    int32_t solver;       /* SDB_SOLVER_* */
    int32_t stream;       /* SDB_STREAM_* (ignored unless solver=EM and nnoise>0) */
    int32_t coupling;     /* SDB_COUPLING_* */
    int32_t lanes;        /* lanes per orbit (power of two, <= 32); 0 = autotune */
    uint64_t seed;        /* EngineConfig.seed reduced mod 2**64 (rng.py:145-147) */
    double dt;
    int64_t ksteps;       /* steps per chunk; one sample per chunk (engine.py:231-262) */
    int64_t chunks;       /* k; samples = k + 1 */
    int64_t orbits;       /* rows in this call */
    int64_t orbit_offset; /* global orbit id of row 0 (noise is keyed by it) */
} sdb_desc;

int sdb_abi_version(void);
int sdb_device_count(void);

/* Context over a list of devices; orbits of one run are sharded across them
 * in contiguous ranges (the analogue of partition_orbits + the worker pool,
 * engine.py:145-150, 265-274).  A device id may repeat (two shards on one GPU). */
sdb_status sdb_open(const int* devices, int ndevices, sdb_ctx** out);
void sdb_close(sdb_ctx* ctx);
const char* sdb_last_error(const sdb_ctx* ctx);

/* Replaces run_batch's integration (engine.py:184-277).
 * init:   [orbits][nequat]   params: [orbits][nparams]
 * values: [orbits][chunks+1][nequat], caller-allocated; sample 0 is written
 *         as a verbatim copy of init (engine.py:214), samples 1..k by the device.
 * fail_step: [orbits]; absolute step index of the orbit's first non-finite
 *         state (engine.py:244-261) or -1.  Rows of failed orbits are NaN from
 *         that step on. */
sdb_status sdb_run(sdb_ctx* ctx, const sdb_desc* desc, const double* init,
                   const double* params, double* values, int64_t* fail_step);

/* Same integration on device-resident buffers on the context's FIRST device
 * (benchmarks: inputs already in HBM).  d_values: [orbits][chunks][nequat]
 * (samples 1..k only).  Launches on `stream` (a cudaStream_t); asynchronous. */
sdb_status sdb_run_device(sdb_ctx* ctx, const sdb_desc* desc, const double* d_init,
                          const double* d_params, double* d_values, int64_t* d_fail_step,
                          void* stream);

/* Number of kernel launches the last sdb_run/sdb_run_device issued (all devices). */
int64_t sdb_last_launch_count(const sdb_ctx* ctx);
/* Lanes-per-orbit layout chosen by the last run (after autotune). */
int32_t sdb_last_lanes(const sdb_ctx* ctx);
/* Full layout of the last run: lanes per orbit, persistent work-pulling grid
 * (0/1), resident CTAs per SM it ran at, register-capped kernel variant (0/1),
 * and the orbit tiles the host-buffer pipeline used (0 for sdb_run_device).
 * SDEB200_LAYOUT="lanes,persistent,ctas,variant" in the environment pins the
 * layout (profiling); SDEB200_TILES / SDEB200_PIECE_KB / SDEB200_HOST_THREADS
 * override the host pipeline's tiling, transfer piece size and copy threads.
 * Any pointer may be NULL. */
void sdb_last_layout(const sdb_ctx* ctx, int32_t* lanes, int32_t* persistent,
                     int32_t* ctas_per_sm, int32_t* variant, int32_t* tiles);
/* Oscillators per lane (J) of the last Kuramoto launch: next_pow2(n) / lanes,
 * or n itself for the exact one-lane layouts of non-power-of-two n <= 16
 * (meanfield);
 * SDEB200_LAYOUT's optional 5th field pins it ("1,1,0,0,5"). */
int32_t sdb_last_lane_width(const sdb_ctx* ctx);
/* Microseconds the last call spent choosing launch layouts (autotune probes;
 * 0 when the layout came from the in-memory or on-disk cache, or was pinned).
 * The probe is budgeted at ~10% of the predicted run; its decisions persist in
 * SDEB200_TUNE_CACHE (default ~/.cache/sdeb200/layouts-v2.tsv; "" disables),
 * keyed by GPU, driver, build and launch shape. */
int64_t sdb_last_tune_us(const sdb_ctx* ctx);

/* ---- noise streams (rng.py) ------------------------------------------------ */

/* Philox-4x32-10 blocks: in [count][6] = (k0, k1, c0, c1, c2, c3), out [count][4].
 * Replaces rng._philox_words / philox_block (rng.py:74-118). */
sdb_status sdb_philox_words(sdb_ctx* ctx, const uint32_t* in, int64_t count, uint32_t* out);

/* Standard normals for one step of a group of orbits: out [count][m].
 * Replaces rng.normals_for_orbits (rng.py:150-188) for stream=PHILOX
 * (chunk/step are the two free counter words).  For SFC64/XOSHIRO256PP the
 * draws are those of step index (chunk<<32 | step) of the per-(orbit, block)
 * stream. */
sdb_status sdb_normals(sdb_ctx* ctx, int32_t stream, uint64_t seed, const uint32_t* orbits,
                       int64_t count, uint32_t chunk, uint32_t step, int32_t m, double* out);

/* Raw 64-bit outputs of one per-(orbit, block) SFC64/XOSHIRO256PP stream. */
sdb_status sdb_stream_raw(sdb_ctx* ctx, int32_t stream, uint64_t seed, uint64_t orbit,
                          uint64_t block, int64_t count, uint64_t* out);

/* Reserved-tag sampling uniforms on [0,1): out [count][ncols].
 * Replaces rng.sampling_uniforms (rng.py:200-222). */
sdb_status sdb_sampling_uniforms(sdb_ctx* ctx, uint64_t seed, const uint32_t* orbits,
                                 int64_t count, int32_t ncols, double* out);

/* Kuramoto batch sampler: init [count][n], params [count][2n+1].
 * Replaces model.sample_kuramoto_batch (model.py:242-270). */
sdb_status sdb_sample_kuramoto(sdb_ctx* ctx, int32_t n, uint64_t seed, const uint32_t* orbits,
                               int64_t count, double omega_lo, double omega_hi,
                               double noise_lo, double noise_hi, double coupling,
                               double* init, double* params);

/* ---- per-step API (solvers.py / model.py) --------------------------------- */

/* Kuramoto drift f(y, p) for count rows: replaces model.drift_eval with the
 * native _kuramoto_drift (model.py:142-157, 188-196). */
sdb_status sdb_drift(sdb_ctx* ctx, int32_t n, int32_t nparams, int32_t coupling, int64_t count,
                     const double* y, const double* p, double* f);

/* One step of solver for count rows with explicit noise [count][n] (EM only;
 * may be NULL otherwise): replaces euler_maruyama_step / euler_step / rk4_step
 * (solvers.py:63-88) for the Kuramoto model. */
sdb_status sdb_step(sdb_ctx* ctx, int32_t solver, int32_t n, int32_t nparams, int32_t nnoise,
                    int32_t coupling, int64_t count, double dt, const double* y,
                    const double* p, const double* noise, double* out);

/* ---- measurement --------------------------------------------------------- */

/* FP64 pipe peak of the context's first device: a DFMA-throughput kernel
 * (ILP 8, one wave of resident CTAs per SM).  Writes FP64 lane-operations per
 * second (one DFMA = one op = 2 flops) and the kernel time in ms.  This is the
 * roofline denominator bench.py reports (MEASURED_PEAKS.json has no FP64 figure). */
sdb_status sdb_fp64_peak(sdb_ctx* ctx, double* ops_per_s, double* ms);

/* Evaluate one of the stepper's device math routines element-wise (accuracy
 * tests): func 0 = sin, 1 = cos (the stepper's sincos), 2 = log (Box-Muller
 * radius), 3 = sqrt, 4 = sin / 5 = cos / 6 = log of libdevice for comparison,
 * 7 = sin / 8 = cos of the Box-Muller angle 2*pi*(w+1)*2^-32 with x = the word w. */
sdb_status sdb_math_probe(sdb_ctx* ctx, int32_t func, const double* x, int64_t count,
                          double* out);

/* ---- streaming store writer (storage.py:108-131) -------------------------------- */

/* run_batch straight into an SDB1 binary store file (storage.py write_store_bin):
 * the caller has written the header and the sample times; the value section,
 * [orbits][chunks+1][nequat] little-endian float64 rows of [initial state |
 * samples 1..k], starts at byte `offset` of the existing file `path`.  Each
 * output piece is written with pwrite as it drains from the GPU, so the store
 * is never held in host memory.  model: NULL for the Kuramoto stepper, else an
 * expression-template model (desc->model = SDB_MODEL_EXPRESSION).  fail_step
 * as sdb_run. */
sdb_status sdb_run_to_file(sdb_ctx* ctx, sdb_model* model, const sdb_desc* desc,
                           const double* init, const double* params, const char* path,
                           int64_t offset, int64_t* fail_step);

/* ---- analysis (analysis.py:72-186) -------------------------------------------- */

/* run_batch fused with coherence_series (analysis.py:98-101): the Kuramoto
 * integration of sdb_run, but each sample is the orbit's order parameter
 * r e^{i Phi} = mean_j e^{i theta_j} computed in the kernel (r = min(|z|, 1),
 * Phi = wrap_phase(arg z), Phi = 0 at r = 0; analysis.py:77-82) -- the phases
 * never leave the GPU.  r_phi: [orbits][2][chunks+1] (per orbit the r series then
 * the Phi series), sample 0 = the initial state's.  fail_step as sdb_run;
 * failed orbits give NaN. */
sdb_status sdb_run_coherence(sdb_ctx* ctx, const sdb_desc* desc, const double* init,
                             const double* params, double* r_phi, int64_t* fail_step);
/* The same on device buffers (first device, asynchronous on `stream`). */
sdb_status sdb_run_coherence_device(sdb_ctx* ctx, const sdb_desc* desc, const double* d_init,
                                    const double* d_params, double* d_r_phi, int64_t* d_fail_step,
                                    void* stream);
/* Order parameter of `rows` populations of n phases each (phases [rows][n]),
 * e.g. a stored trajectory viewed as [orbits * samples][n]
 * (_order_parameter_arrays, analysis.py:77-82). */
sdb_status sdb_order_parameter(sdb_ctx* ctx, int32_t n, int64_t rows, const double* phases,
                               double* r, double* phi);

/* ---- expression-template models (dsl.py / model.py:291-323) -----------------
 *
 * The reference evaluates a model's drift and diffusion templates with a numpy
 * interpreter (dsl.py:441-571, via drift_eval/diffusion_eval, model.py:142-182).
 * Here the template text is compiled: parsed, turned into CUDA device functions
 * and built by NVRTC for sm_100a into a one-thread-per-orbit stepper with the
 * same fused noise streams (the paper's runtime kernel generation,
 * PAPER.md:88-113).  Grammar: dsl.py:12-19 (numbers; t, N, i; y[.], p[.], n[.];
 * + - * / ^; sin cos tan exp ln sqrt abs; sum(j, body)).  The caller validates
 * the templates against the dimensions first (dsl.validate, dsl.py:353-408) and
 * checks that every index stays in range (the reference raises DomainError at
 * evaluation time, dsl.py:516-531); the device does not bounds-check. */

/* Parse both templates and generate their device code (no GPU needed).
 * Errors: SDB_ERR_ARGUMENT with "drift|diffusion: line L, column C: ..." in
 * sdb_last_error(NULL).  Programs are compiled lazily on first use. */
sdb_status sdb_model_create(int32_t nequat, int32_t nparams, int32_t nnoise, const char* drift,
                            const char* diffusion, sdb_model** out);
void sdb_model_free(sdb_model* model);
/* Generated CUDA source of program `kind` (0..9, see sdeb_dsl_args.h DslKind;
 * + 256: the meanfield form sdb_run_model uses when desc->coupling is
 * SDB_COUPLING_MEANFIELD -- sum(j, sin|cos(A_j - B)) factored by the addition
 * formulas into two equation-independent sums; sums that do not depend on the
 * equation are always computed once per evaluation):
 * copies at most cap-1 bytes + NUL into buf (may be NULL) and returns the full
 * length, or -1. */
int64_t sdb_model_source(const sdb_model* model, int32_t kind, char* buf, int64_t cap);
/* NVRTC-compile program `kind` without loading it (no GPU needed); the compile
 * log / error is in sdb_last_error(NULL) on failure. */
sdb_status sdb_model_build(sdb_model* model, int32_t kind);

/* run_batch (engine.py:184-277) for an expression-template model: desc->model
 * = SDB_MODEL_EXPRESSION, dimensions equal to the model's; buffers as sdb_run. */
sdb_status sdb_run_model(sdb_ctx* ctx, sdb_model* model, const sdb_desc* desc,
                         const double* init, const double* params, double* values,
                         int64_t* fail_step);
/* The same on device buffers (first device, asynchronous on `stream`), as
 * sdb_run_device. */
sdb_status sdb_run_model_device(sdb_ctx* ctx, sdb_model* model, const sdb_desc* desc,
                                const double* d_init, const double* d_params, double* d_values,
                                int64_t* d_fail_step, void* stream);
/* drift_eval (which=0) / diffusion_eval (which=1) at time t over `count` rows
 * (model.py:142-182; strict=False semantics: domain errors give inf/NaN).
 * y [count][nequat], p [count][nparams], noise [count][nnoise] (diffusion),
 * out [count][nequat]. */
sdb_status sdb_model_eval(sdb_ctx* ctx, sdb_model* model, int32_t which, double t, int64_t count,
                          const double* y, const double* p, const double* noise, double* out);
/* One em / euler / rk4 step at time t (solvers.py:63-88) with caller-given
 * noise for em on a noisy model. */
sdb_status sdb_model_step(sdb_ctx* ctx, sdb_model* model, int32_t solver, double t, double dt,
                          int64_t count, const double* y, const double* p, const double* noise,
                          double* out);

/* Page-locked host memory for run inputs (cudaHostAlloc, portable across the
 * context's devices).  When init and params of a host-buffer run lie in such
 * memory, sdb_run / sdb_run_coherence / sdb_run_to_file DMA them straight to
 * the device instead of copying them through the library's pinned staging
 * slots (the host copy is what bounds the input leg of large runs).  The
 * reference has no counterpart (its arrays are ordinary numpy buffers);
 * ordinary pageable buffers keep working unchanged. */
sdb_status sdb_host_alloc(int64_t bytes, void** out);
void sdb_host_free(void* ptr);

#ifdef __cplusplus
}
#endif
#endif /* SDEB200_H */
