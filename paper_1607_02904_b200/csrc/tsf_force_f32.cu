// f32 instantiation of the force path (Real = float, Acc = float).
#include "tsf_force_impl.cuh"

namespace tsf {
void compute_f32(Ctx& c, std::uint32_t flags) { compute_t<float, float>(c, flags); }
}  // namespace tsf
