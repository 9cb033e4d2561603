// mixed instantiation of the force path (Real = float, Acc = double).
#include "tsf_force_impl.cuh"

namespace tsf {
void compute_mixed(Ctx& c, std::uint32_t flags) { compute_t<float, double>(c, flags); }
}  // namespace tsf
