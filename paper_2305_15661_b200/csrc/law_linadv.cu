// Kernel instantiations for the LinAdv law.
#include "eval_impl.cuh"

namespace strom_host {
int eval_linadv(strom_handle* h, const EvalArgs& a) { return dispatch_shape<strom::LinAdv>(h, a); }
}  // namespace strom_host
