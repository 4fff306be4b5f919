// Kernel instantiations for the BurgersStrip law.
#include "eval_impl.cuh"

namespace strom_host {
int eval_strip(strom_handle* h, const EvalArgs& a) { return dispatch_shape<strom::BurgersStrip>(h, a); }
}  // namespace strom_host
