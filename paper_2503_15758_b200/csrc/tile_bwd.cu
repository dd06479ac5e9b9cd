#include "kernels.h"
namespace a2d {
int launch_tile_bwd(const a2d_tile_bwd_args&, const CUtensorMap&, const CUtensorMap&,
                    const CUtensorMap&, const CUtensorMap&, cudaStream_t) {
  return set_error(A2D_EUNSUPPORTED, "tile backward not built yet");
}
}  // namespace a2d
