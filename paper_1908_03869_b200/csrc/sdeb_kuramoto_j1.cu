// Instantiates the fused stepper for J = 1 oscillators per lane.
#include "sdeb_kuramoto_inst.cuh"

namespace sdeb {
template cudaError_t launch_kuramoto_j<1>(const RunArgs&, int, int, int, cudaStream_t);
}  // namespace sdeb
