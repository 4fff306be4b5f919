// Kernel instantiations for the Euler law.
#include "eval_impl.cuh"

namespace strom_host {
int eval_euler(strom_handle* h, const EvalArgs& a) { return dispatch_shape<strom::Euler>(h, a); }
}  // namespace strom_host
