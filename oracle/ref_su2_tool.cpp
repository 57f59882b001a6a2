// oracle/ref_su2_tool.cpp — TEST INFRASTRUCTURE ONLY.  A standalone process
// around the unmodified reference's mesh I/O (mesh_io.cpp), because the
// reference's ostream-based writer must not run inside a Python process that
// has numpy loaded.
//   ref_su2_tool roundtrip IN OUT   write_su2(read_su2(IN)) -> OUT
//   ref_su2_tool time IN REPS       best-of-REPS read_su2(IN) seconds on stdout
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <exception>
#include <string>

#include "icemorph/mesh_io.hpp"

int main(int argc, char** argv) {
  if (argc < 4) {
    std::fprintf(stderr, "usage: %s roundtrip IN OUT | time IN REPS\n", argv[0]);
    return 2;
  }
  try {
    const std::string cmd = argv[1];
    if (cmd == "roundtrip") {
      icemorph::write_su2(icemorph::read_su2(std::string(argv[2])), std::string(argv[3]));
      return 0;
    }
    if (cmd == "time") {
      double best = 1e300;
      size_t nodes = 0;
      for (int r = 0; r < std::atoi(argv[3]); ++r) {
        const auto t0 = std::chrono::steady_clock::now();
        const icemorph::Mesh m = icemorph::read_su2(std::string(argv[2]));
        const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        nodes = m.nodes.size();
        if (s < best) best = s;
      }
      std::printf("%.6f %zu\n", best, nodes);
      return 0;
    }
  } catch (const std::exception& e) {
    std::fprintf(stderr, "%s\n", e.what());
    return 1;
  }
  return 2;
}
