// su2_io.hpp — SU2 ASCII mesh I/O on the host (see su2_io.cu).
#pragma once

#include <stdexcept>
#include <string>
#include <vector>

#include "host_io.hpp"
#include "runtime.hpp"

namespace imb {

// mesh_io.hpp:14-21 ParseError: "path:line: what"
struct ParseFailure : std::runtime_error {
  ParseFailure(const std::string& path, size_t line, const std::string& what);
  size_t line;
};

// A mesh as the C-ABI hands it out: AoS nodes, element CSR (ElementKind ids),
// markers with their boundary elements and first-appearance node lists.
struct HostMesh {
  int dim = 0;
  std::vector<double> xyz;
  std::vector<int> kinds;
  std::vector<size_t> offsets{0}, conn;
  struct Marker {
    std::string name;
    std::vector<int> kinds;
    std::vector<size_t> offsets{0}, conn, nodes, line;
  };
  std::vector<Marker> markers;
  // parse bookkeeping: source line of every point / element, NDIME per NPOIN block
  std::vector<size_t> point_line, elem_line;
  std::vector<int> block_dims;
};

HostMesh read_su2_file(Context& ctx, HostPool& pool, const std::string& path);
void write_su2_file(HostPool& pool, const std::string& path, const HostMesh& m);
// find_coincident_nodes (mesh.cpp:104-157): true and (first, second) = (earlier
// node, node) of the first coincident pair in node order
bool coincident_nodes(Context& ctx, const double* xyz, size_t n, size_t& first, size_t& second);
HostPool& host_pool(Context& ctx);

}  // namespace imb
