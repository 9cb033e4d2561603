// f64 instantiation of the force path (Real = double, Acc = double).
#include "tsf_force_impl.cuh"

namespace tsf {
void compute_f64(Ctx& c, std::uint32_t flags) { compute_t<double, double>(c, flags); }
}  // namespace tsf
