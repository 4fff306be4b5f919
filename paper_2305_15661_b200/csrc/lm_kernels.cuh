// Batched Levenberg-Marquardt (placeholder until the LM milestone).
#pragma once
namespace strom {
struct LmWork { void* dummy = nullptr; };
inline void lm_free(LmWork&) {}
}
