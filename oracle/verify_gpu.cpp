// verify_gpu.cpp -- TEST INFRASTRUCTURE: the reference's own property suite
// (apmm::run_verify, src/verify.cpp:413-463) with the B200 kernel plugged into its KernelFn
// seam (verify.hpp:23-24) through include/apmm_b200.hpp, plus the reference's mutation
// idea (tests/test_verify.cpp:47-86): a corrupted GPU kernel must be caught.
//
//   _ref/verify_gpu [seed] [cases]     exit 0 iff every property passes AND the mutant fails
#include <cstdio>
#include <cstdlib>
#include <random>
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
    // the debug/property path on the device: compute_plane_products + recover against the
    // reference's own functions (kernel.cpp:146-181), and recover's error behaviour
    std::mt19937_64 gen(opt.seed);
    int pp_bad = 0;
    for (int c = 0; c < 100; ++c) {
      const std::size_t m = 1 + gen() % 24, n = 1 + gen() % 24, k = 1 + gen() % 300;
      const int nw = 1 + static_cast<int>(gen() % 8), nx = 1 + static_cast<int>(gen() % 8);
      std::vector<std::uint8_t> wb(m * k), xb(n * k);
      for (auto& v : wb) v = static_cast<std::uint8_t>(gen() % (1u << nw));
      for (auto& v : xb) v = static_cast<std::uint8_t>(gen() % (1u << nx));
      const auto w = apmm::decompose_and_pack(apmm::CodeMatrix(m, k, apmm::BitWidth(nw), wb));
      const auto x = apmm::decompose_and_pack(apmm::CodeMatrix(n, k, apmm::BitWidth(nx), xb));
      const auto ref = apmm::compute_plane_products(w, x);
      const auto got = apmm::b200::compute_plane_products(w, x);
      for (int i = 0; i < nw; ++i) {
        for (int j = 0; j < nx; ++j) {
          if (!(got.product(i, j) == ref.product(i, j))) ++pp_bad;
        }
      }
      if (!(apmm::b200::recover(got) == apmm::recover(ref))) ++pp_bad;
    }
    std::printf("%s compute_plane_products + recover on the device (100 cases)\n",
                pp_bad ? "FAIL" : "PASS");
    if (pp_bad) rc = 1;
    {  // recover must throw Overflow exactly like the reference (kernel.cpp:172-176)
      std::vector<apmm::IntMatrix> prods(64, apmm::IntMatrix(1, 1));
      for (auto& p : prods) p.data[0] = 40000;
      const apmm::PlaneProductStack big(apmm::BitWidth(8), apmm::BitWidth(8), 40000, prods);
      bool ref_threw = false, gpu_threw = false;
      try { apmm::recover(big); } catch (const apmm::Overflow&) { ref_threw = true; }
      try { apmm::b200::recover(big); } catch (const apmm::Overflow&) { gpu_threw = true; }
      std::printf("%s recover overflow (reference %d, device %d)\n",
                  ref_threw == gpu_threw && gpu_threw ? "PASS" : "FAIL", ref_threw, gpu_threw);
      if (!(ref_threw && gpu_threw)) rc = 1;
    }
    {  // dot_1bit_xor / matmul_plane_pair through the drop-in (kernel.hpp:61-69): the
       // xor_identity property (verify.cpp:142-157) on the device, plus the error classes
      int bad = 0;
      for (int c = 0; c < 200; ++c) {
        const std::size_t k = 1 + gen() % 2000, words = (k + 31) / 32;
        std::vector<std::uint32_t> a(words), b(words);
        for (auto& v : a) v = static_cast<std::uint32_t>(gen());
        for (auto& v : b) v = static_cast<std::uint32_t>(gen());
        if (k % 32) {
          a.back() &= (1u << (k % 32)) - 1u;
          b.back() &= (1u << (k % 32)) - 1u;
        }
        if (apmm::b200::dot_1bit_xor(a, b, k) != apmm::dot_1bit_xor(a, b, k)) ++bad;
      }
      bool len_ok = false, k_ok = false;
      const std::vector<std::uint32_t> one(1), two(2);
      try { apmm::b200::dot_1bit_xor(one, two, 32); } catch (const apmm::LengthMismatch&) { len_ok = true; }
      try { apmm::b200::dot_1bit_xor(one, one, 0); } catch (const apmm::OutOfRange&) { k_ok = true; }
      for (int c = 0; c < 20; ++c) {
        const std::size_t m = 1 + gen() % 30, n = 1 + gen() % 30, k = 1 + gen() % 400;
        const int nw = 1 + static_cast<int>(gen() % 8), nx = 1 + static_cast<int>(gen() % 8);
        std::vector<std::uint8_t> wb(m * k), xb(n * k);
        for (auto& v : wb) v = static_cast<std::uint8_t>(gen() % (1u << nw));
        for (auto& v : xb) v = static_cast<std::uint8_t>(gen() % (1u << nx));
        const auto w = apmm::decompose_and_pack(apmm::CodeMatrix(m, k, apmm::BitWidth(nw), wb));
        const auto x = apmm::decompose_and_pack(apmm::CodeMatrix(n, k, apmm::BitWidth(nx), xb));
        const unsigned i = static_cast<unsigned>(gen() % nw), j = static_cast<unsigned>(gen() % nx);
        if (!(apmm::b200::matmul_plane_pair(w, i, x, j) == apmm::matmul_plane_pair(w, i, x, j))) ++bad;
      }
      const bool ok = bad == 0 && len_ok && k_ok;
      std::printf("%s xor_identity / dot_1bit_xor / matmul_plane_pair through the drop-in "
                  "(200 dots, 20 plane pairs, errors %d%d)\n", ok ? "PASS" : "FAIL", len_ok, k_ok);
      if (!ok) rc = 1;
    }
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
