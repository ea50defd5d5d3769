// SIPG kernels (cell + face terms).  Placeholder until the element-centric kernel lands.
#include "device_common.cuh"

namespace fem {

void launch_dg_apply(fem_ctx*, const Level&, const double*, double*) {
  throw Error{FEM_E_ARG, "SIPG operator not built yet"};
}
void launch_dg_diagonal(fem_ctx*, Level&) { throw Error{FEM_E_ARG, "SIPG operator not built yet"}; }
void launch_dg_face_geometry(fem_ctx*, Level&) {}

}  // namespace fem
