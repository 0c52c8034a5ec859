// Launch arguments of the NVRTC-compiled expression-template programs
// (sdeb_dsl_kernel.cuh).  Plain POD shared by the nvcc-built host runtime
// (sdeb_dsl.cu) and the runtime-compiled device code, so both sides agree on
// the layout byte for byte.
#pragma once
#include "sdeb_cstdint.cuh"

namespace sdeb {

// What one compiled program does (baked in as SDB_KIND).
enum DslKind : int {
    DK_RUN_PHILOX = 0,   // run_batch loop, em, Philox normals (rng.py:150-188)
    DK_RUN_SFC64 = 1,    // run_batch loop, em, per-(orbit, block) sfc64 streams
    DK_RUN_XOSHIRO = 2,  // run_batch loop, em, per-(orbit, block) xoshiro256++ streams
    DK_RUN_EULER = 3,    // run_batch loop, euler (or em on a noise-free model)
    DK_RUN_RK4 = 4,      // run_batch loop, rk4
    DK_STEP_EM = 5,      // one em step with caller-given noise (solvers.py:63-71)
    DK_STEP_EULER = 6,   // one euler step (solvers.py:74-77)
    DK_STEP_RK4 = 7,     // one rk4 step (solvers.py:80-88)
    DK_EVAL_DRIFT = 8,   // drift_eval (model.py:142-157)
    DK_EVAL_DIFFUSION = 9,  // diffusion_eval (model.py:160-182)
    DK_COUNT = 10
};

struct DslArgs {
    const double* state_in;   // [rows][N]: init / y
    const double* params;     // [rows][NP]
    const double* noise;      // [rows][NN] caller-given normals (STEP_EM, EVAL_DIFFUSION)
    double* state_out;        // [rows][N]: state at chunk_end / stepped y (may be null for runs)
    double* values;           // runs: sample of chunk c -> values[(r*vstride + c-chunk_begin)*N + i];
                              // eval: [rows][N]
    int64_t* fail_step;       // [rows] first non-finite absolute step or -1 (runs)
    uint64_t* rng_state;      // [rows][ceil(NN/4)][4] stateful streams (runs)
    double* scratch;          // SDB_GLOBAL_STATE programs: [N + 4*ceil(NN/4)][rows]
    int64_t rows, orbit_offset, vstride;
    int64_t ksteps, chunk_begin, chunk_end;
    uint64_t seed;
    double dt, sqrt_dt, t;    // t: STEP / EVAL time
    int32_t fresh;            // runs: 1 = start (fail=-1, seed streams); 0 = resume
    int32_t pad_;
};

}  // namespace sdeb
