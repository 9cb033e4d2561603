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

namespace {
// Diagnostics of the device math (tsf_math_probe): the constant-bank exp/log
// against libdevice, and the bond order's series and log-space paths.
__global__ void k_math_probe(int fn, int n, const double* __restrict__ x, Row<double> rd,
                             Row<float> rf, double* __restrict__ out) {
  const int q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= n) return;
  const double v = x[q];
  double a = 0, b = 0;
  switch (fn) {
    case 0: a = exp_cb(v); break;
    case 1: a = log_cb(v); break;
    case 2: a = exp(v); break;
    case 3: a = log(v); break;
    case 4: bond_order<double>(v, rd, a, b); break;
    case 5: {
      float bf, dbf;
      bond_order<float>(float(v), rf, bf, dbf);
      a = bf;
      b = dbf;
      break;
    }
    case 8: Fn<double>::sincospi_half(v, &a, &b); break;   // the cutoff ramp's (|x| <= 1/2)
    case 9: sincospi(v, &a, &b); break;
    case 7: {    // which path the double bond order takes: a = 1 series, b = ln u
      const double xb = rd.beta * v;
      b = rd.eta * log_cb(xb);
      double bb, dbb;
      a = (v > 0 && xb >= 0x1p-1000 && bond_order_series(b, rd, v, bb, dbb)) ? 1.0 : 0.0;
      break;
    }
    default: {   // the reference's pow form (potential.hpp:107-120), double
      if (v > 0) {
        const double u = pow(rd.beta * v, rd.eta);
        a = pow(1.0 + u, -0.5 / rd.eta);
        b = -0.5 * a * (u / (1.0 + u)) / v;
      } else {
        a = 1.0;
      }
    }
  }
  out[2 * q] = a;
  out[2 * q + 1] = b;
}
}  // namespace

void math_probe(const Params& p, int fn, std::int64_t n, const double* x, double* out) {
  if (fn < 0 || fn > 9) throw ConfigError("unknown probe function");
  if (n <= 0) return;
  double *dx = nullptr, *dy = nullptr;
  TSF_CUDA(cudaMalloc(&dx, sizeof(double) * n));
  TSF_CUDA(cudaMalloc(&dy, sizeof(double) * 2 * n));
  TSF_CUDA(cudaMemcpy(dx, x, sizeof(double) * n, cudaMemcpyHostToDevice));
  k_math_probe<<<int((n + 255) / 256), 256>>>(fn, int(n), dx, make_row<double>(p.entry(0, 0, 0)),
                                              make_row<float>(p.entry(0, 0, 0)), dy);
  const cudaError_t e = cudaMemcpy(out, dy, sizeof(double) * 2 * n, cudaMemcpyDeviceToHost);
  cudaFree(dx);
  cudaFree(dy);
  TSF_CUDA(e);
}

void compute(Ctx& c, Precision prec, std::uint32_t flags) {
  switch (prec) {
    case Precision::F64: compute_f64(c, flags); break;
    case Precision::Mixed: compute_mixed(c, flags); break;
    case Precision::F32: compute_f32(c, flags); break;
  }
}

}  // namespace tsf
