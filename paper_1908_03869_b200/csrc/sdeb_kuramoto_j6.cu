// Instantiates the fused stepper for J = 6 oscillators per lane (the exact one-lane layout of n = 6).
// the stepper reads the sincos / log tables from shared memory (sdeb_math.cuh)
#define SDEB_SMEM_TABLES 1
#include "sdeb_kuramoto_inst.cuh"

namespace sdeb {
template cudaError_t launch_kuramoto_j<6>(const RunArgs&, int, int, int, int, cudaStream_t);
template cudaError_t occupancy_kuramoto_j<6>(int, int, int, int, size_t, int*);
}  // namespace sdeb
