// TEST INFRASTRUCTURE ONLY.  The reference's own verification battery
// (tmd::run_verification, proj/src/verify.cpp:822-845) driven through the B200
// drop-in (integration/potential_b200.cpp): every evaluate_forces call of the
// battery — and of the Engine it runs — goes to the GPU.  Prints one line per
// check: PASS|FAIL <name> <detail>.  Exit code: number of failed checks.
#include <cstdio>
#include <fstream>
#include <sstream>

#include "tmd/params.hpp"
#include "tmd/verify.hpp"

int main(int argc, char** argv) {
  tmd::ParamTable params = tmd::builtin_silicon();
  if (argc > 1) {
    std::ifstream in(argv[1]);
    std::stringstream ss;
    ss << in.rdbuf();
    params = tmd::parse_param_text(ss.str(), argv[1]);
  }
  int failed = 0;
  for (const tmd::CheckResult& r : tmd::run_verification(params)) {
    std::printf("%s %s %s\n", r.pass ? "PASS" : "FAIL", r.name.c_str(), r.detail.c_str());
    failed += r.pass ? 0 : 1;
  }
  return failed;
}
