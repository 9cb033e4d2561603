// Force-path entry points: parameter upload and precision dispatch.  The
// kernels live in tsf_force_impl.cuh and are instantiated per precision in
// tsf_force_{f64,mixed,f32}.cu so the three compile in parallel.
#include "tsf_force_impl.cuh"

namespace tsf {

void compute_f64(Ctx& c, std::uint32_t flags);
void compute_mixed(Ctx& c, std::uint32_t flags);
void compute_f32(Ctx& c, std::uint32_t flags);

void upload_params(Ctx& c) {
  const int s = c.params.species_count();
  if (s > kMaxSpecies)
    throw ConfigError("at most " + std::to_string(kMaxSpecies) + " species are supported");
  std::vector<Row<double>> r64;
  std::vector<Row<float>> r32;
  std::vector<double> cut;
  for (int i = 0; i < s; ++i)
    for (int j = 0; j < s; ++j)
      for (int k = 0; k < s; ++k) {
        const Entry& e = c.params.entry(i, j, k);
        r64.push_back(make_row<double>(e));
        r32.push_back(make_row<float>(e));
        const double cc = e.cutoff();
        cut.push_back(cc * cc);
      }
  c.rows_f64.reserve(r64.size());
  c.rows_f32.reserve(r32.size());
  c.cutsq.reserve(cut.size());
  TSF_CUDA(cudaMemcpyAsync(c.rows_f64.get(), r64.data(), sizeof(Row<double>) * r64.size(),
                           cudaMemcpyHostToDevice, c.stream));
  TSF_CUDA(cudaMemcpyAsync(c.rows_f32.get(), r32.data(), sizeof(Row<float>) * r32.size(),
                           cudaMemcpyHostToDevice, c.stream));
  TSF_CUDA(cudaMemcpyAsync(c.cutsq.get(), cut.data(), sizeof(double) * cut.size(),
                           cudaMemcpyHostToDevice, c.stream));
  TSF_CUDA(cudaStreamSynchronize(c.stream));
  c.hoist_ramp = c.params.ramp_depends_on_ik_only();
}

void compute(Ctx& c, Precision prec, std::uint32_t flags) {
  switch (prec) {
    case Precision::F64: compute_f64(c, flags); break;
    case Precision::Mixed: compute_mixed(c, flags); break;
    case Precision::F32: compute_f32(c, flags); break;
  }
}

}  // namespace tsf
