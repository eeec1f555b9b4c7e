// Kernel (b), tensor-core path: placeholder until the tcgen05 scorer lands.
#include "route.cuh"

namespace fepll {

int select_level_tc(Plan* p, const LevelArgs& a, const float* Z32, const double* Z64,
                    const double* sq, double guard, cudaStream_t st) {
  (void)p; (void)a; (void)Z32; (void)Z64; (void)sq; (void)guard; (void)st;
  set_error("tcgen05 scoring path not built yet");
  return kDataError;
}

}  // namespace fepll
