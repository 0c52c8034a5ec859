// Runtime code generation for expression-template models (host side).
//
// The reference evaluates drift/diffusion templates with a numpy tree-walking
// interpreter (dsl.py:441-571).  Here the template text (the grammar of
// dsl.py:12-19, in the canonical form dsl.to_source prints) is parsed once,
// turned into CUDA device functions, spliced into sdeb_dsl_kernel.cuh and
// compiled by NVRTC for sm_100a -- the paper's own mechanism of generating
// the system's GPU source at run time.  Programs are cached
// per (model, kind).
#pragma once
#include <cuda_runtime.h>

#include <map>
#include <memory>
#include <mutex>
#include <string>

#include "sdeb_dsl_args.h"

struct sdb_model {
    int32_t nequat = 0, nparams = 0, nnoise = 0;
    std::string drift_text, diffusion_text;  // as given
    std::string drift_cu[2], diffusion_cu[2];  // generated device functions: [literal, factored]
    int drift_h[2] = {1, 1}, diffusion_h[2] = {1, 1};  // hoisted values per evaluation
    std::string error;                       // last compile / launch error
    bool eq_sum[2] = {false, false};         // [literal, factored]: a sum stays per equation
    std::mutex mu;
    struct Program {
        cudaLibrary_t lib = nullptr;
        cudaKernel_t kernel = nullptr;
        std::string log;
    };
    std::map<int, Program> programs;  // by kind + 64 * lanes + 4096 * factor
    ~sdb_model();
};

namespace sdeb_dsl {

// Parse both templates and generate their device code.  On failure returns
// false with `err` = "drift: line L, column C: message" style text.
bool generate(sdb_model* m, std::string* err);

// Full CUDA source of one program kind (for inspection / tests).  factor:
// the meanfield form (sum(j, sin|cos(A_j - B)) via the addition formulas).
std::string program_source(const sdb_model* m, int kind, int lanes, bool factor);

// NVRTC compile only (no device needed); the log lands in m->error.
cudaError_t compile_only(sdb_model* m, int kind, int lanes, bool factor, std::string* err);

// The compiled kernel of one (kind, lanes) (compiled on first use, thread-safe).
cudaError_t kernel_for(sdb_model* m, int kind, int lanes, bool factor, cudaKernel_t* out,
                       std::string* err);

// Launch one program over `a.rows` orbits (lanes_for(m) threads each); the
// caller provides a.scratch of scratch_doubles() when global_state().
cudaError_t launch(sdb_model* m, int kind, const sdeb::DslArgs& a, cudaStream_t st,
                   std::string* err, bool factor = false);

constexpr int kBlock = 128;      // threads per CTA = 128 / lanes orbit slots
constexpr int kSmemMax = 96 * 1024;
constexpr size_t kTableSmem = 16 * (1024 + 512);  // sincos + log tables staged by the program
constexpr int kUnrollWork = 32;  // unroll equation loops while (N / lanes) x evaluations <= this

// Doubles per orbit in the shared column: y + one step's normals.
int state_words(const sdb_model* m);
// Lanes per orbit (power of two <= 32): ~4 equations per lane for templates
// with sums (O(N) work per equation), ~16 without, or SDEB200_DSL_LANES.
// Results do not depend on it.
int lanes_for(const sdb_model* m, bool factor);
// True when the program stages the math tables in shared memory.
bool stage_tables(const sdb_model* m, bool factor);
// True when the columns go to global scratch instead of shared memory.
bool global_state(const sdb_model* m, int lanes);
// Doubles of global scratch a launch over `rows` orbits needs (0 = none).
size_t scratch_doubles(const sdb_model* m, int lanes, int64_t rows);

}  // namespace sdeb_dsl
