// Kernel instantiations for the Euler law with the Roe numerical flux and for Euler (LLF) on
// meshes with slip walls (GPU-only extensions).
#include "eval_impl.cuh"

namespace strom_host {
int eval_euler_roe(strom_handle* h, const EvalArgs& a) { return dispatch_shape<strom::EulerRoe>(h, a); }
int eval_euler_wall(strom_handle* h, const EvalArgs& a) { return dispatch_shape<strom::EulerWall>(h, a); }
}  // namespace strom_host
