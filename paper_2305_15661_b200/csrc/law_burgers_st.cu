// Kernel instantiations for the BurgersST law.
#include "eval_impl.cuh"

namespace strom_host {
int eval_burgers_st(strom_handle* h, const EvalArgs& a) { return dispatch_shape<strom::BurgersST>(h, a); }
}  // namespace strom_host
