// ref_keyfile_gen.cpp -- TEST INFRASTRUCTURE ONLY.  Drives the UNMODIFIED
// reference dataio (generate_pair, write_keys_binary/_text, read_keys;
// dataio.cpp, compiled where it lies under /root/reference) from the command
// line, standing in for the reference's `mergebench gen` (whose CLI11
// dependency is absent here).  tests/golden/make_keyfile_golden.py records
// its files as fixtures.
//   ref_keyfile_gen gen DIST NA NB SEED OUT_A OUT_B bin|text
//   ref_keyfile_gen read PATH          (prints count and the keys, one per line)
#include <cstdint>
#include <cstdlib>
#include <iostream>
#include <string>

#include "mergepath/dataio.hpp"

int main(int argc, char **argv) {
  try {
    const std::string cmd = argc > 1 ? argv[1] : "";
    if (cmd == "gen" && argc == 9) {
      auto [a, b] = mergepath::generate_pair(
          mergepath::parse_distribution(argv[2]), std::strtoull(argv[3], nullptr, 10),
          std::strtoull(argv[4], nullptr, 10), std::strtoull(argv[5], nullptr, 10));
      if (std::string(argv[8]) == "text") {
        mergepath::write_keys_text(argv[6], a);
        mergepath::write_keys_text(argv[7], b);
      } else {
        mergepath::write_keys_binary(argv[6], a);
        mergepath::write_keys_binary(argv[7], b);
      }
      return 0;
    }
    if (cmd == "read" && argc == 3) {
      const auto v = mergepath::read_keys(argv[2]);
      std::cout << v.size() << '\n';
      for (auto k : v)
        std::cout << k << '\n';
      return 0;
    }
    std::cerr << "usage: ref_keyfile_gen gen DIST NA NB SEED OUT_A OUT_B bin|text | read PATH\n";
    return 1;
  } catch (const std::invalid_argument &e) {
    std::cerr << "error: " << e.what() << '\n';
    return 3;
  } catch (const std::exception &e) {
    std::cerr << "error: " << e.what() << '\n';
    return 2;
  }
}
