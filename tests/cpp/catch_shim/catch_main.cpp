// Runner for the Catch2-compatible shim: runs every registered test case,
// once per flat SECTION, prints a summary, exits non-zero on any failure.
#include <chrono>
#include <cstdio>
#include <exception>
#include <string>

#include "catch2/catch_amalgamated.hpp"

int main(int argc, char** argv) {
  const std::string filter = argc > 1 ? argv[1] : "";
  int cases = 0, runs = 0, failed = 0;
  const auto t0 = std::chrono::steady_clock::now();
  for (const shim::TestCaseInfo& tc : shim::registry()) {
    if (!filter.empty() && std::string(tc.name).find(filter) == std::string::npos) continue;
    ++cases;
    shim::SectionState& s = shim::sections();
    s.target = 0;
    bool ok = true;
    do {
      s.seen = 0;
      ++runs;
      try {
        tc.fn();
      } catch (const shim::Failure& f) {
        std::printf("FAILED: %s\n  %s\n", tc.name, f.what());
        ok = false;
      } catch (const std::exception& e) {
        std::printf("FAILED: %s\n  unexpected exception: %s\n", tc.name, e.what());
        ok = false;
      }
      ++s.target;
    } while (s.target < s.seen);
    if (!ok) ++failed;
  }
  const double secs =
      std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  std::printf("shim: %d test cases (%d section runs), %d failed, %.3f s\n", cases, runs, failed,
              secs);
  return failed == 0 ? 0 : 1;
}
