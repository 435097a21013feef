// verify_gpu.cpp -- TEST INFRASTRUCTURE: the reference's own property suite
// (apmm::run_verify, src/verify.cpp:413-463) with the B200 kernel plugged into its KernelFn
// seam (verify.hpp:23-24) through include/apmm_b200.hpp, plus the reference's mutation
// idea (tests/test_verify.cpp:47-86): a corrupted GPU kernel must be caught.
//
//   _ref/verify_gpu [seed] [cases]     exit 0 iff every property passes AND the mutant fails
#include <cstdio>
#include <cstdlib>
#include <string>

#include "apmm/verify.hpp"
#include "apmm_b200.hpp"

int main(int argc, char** argv) {
  apmm::VerifyOptions opt;
  opt.seed = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 1;
  opt.cases = argc > 2 ? std::atoi(argv[2]) : 1000;
  int rc = 0;
  try {
    const apmm::VerifyReport rep = apmm::run_verify(opt, apmm::b200::kernel_fn());
    for (const auto& p : rep.properties) {
      if (p.passed) {
        std::printf("PASS %s (%d cases)\n", p.name.c_str(), p.cases);
      } else {
        std::printf("FAIL %s\n  %s\n", p.name.c_str(), p.detail.c_str());
        rc = 1;
      }
    }
    std::printf("gpu kernel: %s (seed %llu)\n", rep.all_passed() ? "all properties passed" : "FAILED",
                static_cast<unsigned long long>(opt.seed));
    // mutation: flip one output entry of the GPU result; the suite must catch it
    const apmm::KernelFn mutant = [](const apmm::PackedBitPlanes& w, const apmm::PackedBitPlanes& x,
                                     const apmm::TileConfig& c) {
      apmm::AccumMatrix y = apmm::b200::matmul_ap(w, x, c);
      if (y.rows * y.cols > 3) y.data[y.data.size() / 2] += 2;
      return y;
    };
    apmm::VerifyOptions mopt = opt;
    mopt.cases = 50;
    const apmm::VerifyReport bad = apmm::run_verify(mopt, mutant);
    const bool caught = !bad.properties[0].passed;
    std::printf("mutant kernel %s\n", caught ? "caught by kernel-vs-oracle" : "NOT caught");
    if (!caught) rc = 1;
  } catch (const std::exception& e) {
    std::printf("exception: %s\n", e.what());
    rc = 2;
  }
  return rc;
}
