// Kernel instantiations for the LinAdvMS law (linear advection with a manufactured solution).
#include "eval_impl.cuh"

namespace strom_host {
int eval_linadv_ms(strom_handle* h, const EvalArgs& a) { return dispatch_shape<strom::LinAdvMS>(h, a); }
}  // namespace strom_host
