// Instantiates the fused stepper for J = 9 oscillators per lane (the exact one-lane layout of n = 9).
// the stepper reads the sincos / log tables from shared memory (sdeb_math.cuh)
#define SDEB_SMEM_TABLES 1
#include "sdeb_kuramoto_inst.cuh"

namespace sdeb {
template cudaError_t launch_kuramoto_j<9>(const RunArgs&, int, int, int, int, cudaStream_t);
template cudaError_t occupancy_kuramoto_j<9>(int, int, int, int, size_t, int*);
}  // namespace sdeb
