// Runner for the Catch2 shim: runs every registered TEST_CASE (or those whose
// name contains argv[1]), prints one line per case, exits non-zero on failure.
#include <cstdio>
#include <cstring>
#include <exception>

#include "catch2/catch_amalgamated.hpp"

int main(int argc, char** argv) {
  int passed = 0, failed = 0;
  for (const auto& c : catch_shim::registry()) {
    if (argc > 1 && std::strstr(c.name.c_str(), argv[1]) == nullptr) continue;
    try {
      c.fn();
      ++passed;
      std::printf("PASS  %s\n", c.name.c_str());
    } catch (const std::exception& e) {
      ++failed;
      std::printf("FAIL  %s\n  %s\n", c.name.c_str(), e.what());
    }
  }
  std::printf("%d passed, %d failed\n", passed, failed);
  return failed ? 1 : 0;
}
