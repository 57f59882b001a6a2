// su2_io.cu — SU2 ASCII mesh reader / writer (the data
// format on the input side of the path): read_su2 / write_su2 of
// proj/src/mesh_io.cpp:127-309 with the same grammar, error texts and line
// numbers, built for 20-40M-node files:
//
//  * the whole file is read once; line starts are found by a host thread
//    pool (memchr per chunk), each line is classified significant / blank /
//    comment in parallel (LineReader::next, mesh_io.cpp:55-64), and the
//    section structure (NDIME / NPOIN / NELEM / NMARK in any order) is walked
//    sequentially over the significant lines only;
//  * the large point and element blocks are then parsed in parallel chunks
//    with std::from_chars (the reference's parse_double / parse_index); the
//    first failing line of each chunk is kept and the smallest line wins —
//    the line the sequential reader would have stopped at;
//  * post-parse validation (element kinds per dimension, node ranges,
//    marker node lists) follows mesh_io.cpp:224-250 in the same order;
//  * the coincident-node check (find_coincident_nodes, mesh.cpp:104-157) runs
//    on the device: cells of size 1e-12 * diagonal, hashed and radix-sorted,
//    one thread per node probing its 27 neighbour cells for an earlier node
//    within the tolerance; the smallest such node index wins, as in the
//    reference's insertion-order scan.  (Within one cell the reference's
//    unordered_multimap order picks among several earlier coincident nodes;
//    here the smallest index is reported.)
//  * write_su2 formats chunks in parallel ("%.17g" = ostream precision 17)
//    and writes them in order.
#include <algorithm>
#include <atomic>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include <cub/cub.cuh>

#include "../../include/icemorph_b200.h"
#include "common.cuh"
#include "host_io.hpp"
#include "runtime.hpp"
#include "su2_io.hpp"

namespace imb {

ParseFailure::ParseFailure(const std::string& path, size_t line, const std::string& what)
    : std::runtime_error(path + ":" + std::to_string(line) + ": " + what), line(line) {}

namespace {

// ElementKind <-> VTK ids (mesh.cpp:12-36), names (mesh.cpp:51-62), node counts
const int kVtk[7] = {3, 5, 9, 10, 12, 13, 14};
const char* kName[7] = {"line", "triangle", "quadrilateral", "tetrahedron", "hexahedron",
                        "prism", "pyramid"};
const int kCount[7] = {2, 3, 4, 4, 8, 6, 5};

int kind_from_vtk(size_t v) {
  for (int k = 0; k < 7; ++k)
    if ((size_t)kVtk[k] == v) return k;
  return -1;
}
bool is_volume_kind(int k, int dim) { return dim == 2 ? (k == 1 || k == 2) : (k >= 3 && k <= 6); }
bool is_boundary_kind(int k, int dim) { return dim == 2 ? k == 0 : (k == 1 || k == 2); }

inline bool is_space(char c) {  // the C locale's isspace, as istream >> uses
  return c == ' ' || c == '\t' || c == '\n' || c == '\v' || c == '\f' || c == '\r';
}

struct Text {
  std::string path;
  std::vector<char> buf;
  std::vector<size_t> start;   // line starts; line l (1-based) = [start[l-1], start[l])
  std::vector<uint32_t> sig;   // significant lines (0-based ids), in order
  size_t lines() const { return start.size() - 1; }
  // content of line l (0-based) before any '%' and without the newline
  std::string_view body(size_t l) const {
    const char* b = buf.data() + start[l];
    size_t n = start[l + 1] - start[l];
    if (n && b[n - 1] == '\n') --n;
    const void* pct = memchr(b, '%', n);
    if (pct) n = (size_t)(static_cast<const char*>(pct) - b);
    return {b, n};
  }
};

[[noreturn]] void fail(const Text& t, size_t line, const std::string& what) {
  throw ParseFailure(t.path, line, what);
}

// whitespace tokens of a line (tokenize, mesh_io.cpp:28-34)
template <class F>
void for_tokens(std::string_view s, F&& f) {
  size_t i = 0;
  while (i < s.size()) {
    while (i < s.size() && is_space(s[i])) ++i;
    if (i >= s.size()) break;
    size_t j = i;
    while (j < s.size() && !is_space(s[j])) ++j;
    if (!f(s.substr(i, j - i))) return;
    i = j;
  }
}

bool parse_double(std::string_view t, double& v) {
  auto [p, ec] = std::from_chars(t.data(), t.data() + t.size(), v);
  return ec == std::errc{} && p == t.data() + t.size();
}
bool parse_index(std::string_view t, size_t& v) {
  auto [p, ec] = std::from_chars(t.data(), t.data() + t.size(), v);
  return ec == std::errc{} && p == t.data() + t.size();
}

std::string trim(std::string_view s) {
  size_t b = 0, e = s.size();
  while (b < e && (s[b] == ' ' || s[b] == '\t' || s[b] == '\r' || s[b] == '\n')) ++b;
  while (e > b && (s[e - 1] == ' ' || s[e - 1] == '\t' || s[e - 1] == '\r' || s[e - 1] == '\n')) --e;
  return std::string(s.substr(b, e - b));
}

// split_keyword, mesh_io.cpp:83-97
bool split_keyword(std::string_view line, std::string& key, std::string& value) {
  const size_t eq = line.find('=');
  if (eq == std::string_view::npos) return false;
  key = trim(line.substr(0, eq));
  value = trim(line.substr(eq + 1));
  return !key.empty();
}

// One parse error candidate: the smallest line wins.
struct FirstError {
  std::atomic<size_t> line{SIZE_MAX};
  std::string what;
  std::mutex m;
  void offer(size_t l, std::string w) {
    std::lock_guard<std::mutex> g(m);
    if (l < line.load()) line.store(l), what = std::move(w);
  }
};

// parse_element_line, mesh_io.cpp:99-125; returns "" or the error text
std::string parse_element(std::string_view s, int& kind, size_t* nodes) {
  std::string_view tok[10];
  int nt = 0;  // tokens kept: the type id and up to 8 indices (+1 to see "enough")
  for_tokens(s, [&](std::string_view t) {
    tok[nt++] = t;
    return nt < 10;
  });
  kind = -1;
  if (nt == 0) return "empty element line";
  size_t vtk = 0;
  if (!parse_index(tok[0], vtk)) return "expected an element type id, got '" + std::string(tok[0]) + "'";
  kind = kind_from_vtk(vtk);
  if (kind < 0) return "unknown element kind " + std::to_string(vtk);
  const int count = kCount[kind];
  if (nt < count + 1)
    return std::string(kName[kind]) + " needs " + std::to_string(count) + " node indices";
  for (int i = 0; i < count; ++i)
    if (!parse_index(tok[i + 1], nodes[i])) return "bad node index '" + std::string(tok[i + 1]) + "'";
  return "";
}

struct Block {
  size_t first, count;  // significant-line range
};

}  // namespace

HostMesh read_su2_file(Context& ctx, HostPool& pool, const std::string& path) {
  Text t;
  t.path = path;
  {
    FILE* f = std::fopen(path.c_str(), "rb");
    if (!f) throw std::runtime_error("cannot open mesh file '" + path + "'");
    std::fseek(f, 0, SEEK_END);
    const long sz = std::ftell(f);
    std::fseek(f, 0, SEEK_SET);
    t.buf.resize((size_t)std::max(sz, 0L));
    const size_t got = sz > 0 ? std::fread(t.buf.data(), 1, (size_t)sz, f) : 0;
    std::fclose(f);
    if (got != t.buf.size()) throw std::runtime_error("cannot read mesh file '" + path + "'");
  }
  // ---- line index (parallel) -------------------------------------------------
  const size_t n = t.buf.size();
  const int nchunk = std::max(1, std::min<int>(pool.size() * 4, (int)(n / (1 << 20)) + 1));
  std::vector<std::vector<size_t>> part(nchunk);
  pool.run(nchunk, [&](int c) {
    const size_t b = n * c / nchunk, e = n * (c + 1) / nchunk;
    const char* p = t.buf.data();
    for (size_t i = b; i < e;) {
      const void* q = memchr(p + i, '\n', e - i);
      if (!q) break;
      i = (size_t)(static_cast<const char*>(q) - p) + 1;
      part[c].push_back(i);
    }
  });
  t.start.push_back(0);
  for (auto& v : part) t.start.insert(t.start.end(), v.begin(), v.end());
  if (t.start.back() != n) t.start.push_back(n);  // last line without '\n'
  const size_t nl = t.lines();
  std::vector<unsigned char> is_sig(nl);
  pool.run(nchunk, [&](int c) {
    for (size_t l = nl * c / nchunk; l < nl * (c + 1) / nchunk; ++l) {
      const std::string_view s = t.body(l);
      bool any = false;
      for (char ch : s)
        if (!(ch == ' ' || ch == '\t' || ch == '\r' || ch == '\n')) {
          any = true;
          break;
        }
      is_sig[l] = any;
    }
  });
  t.sig.reserve(nl);
  for (size_t l = 0; l < nl; ++l)
    if (is_sig[l]) t.sig.push_back((uint32_t)l);
  // ---- section structure (sequential over significant lines) ----------------
  HostMesh m;
  m.dim = 0;
  FirstError err;
  size_t s = 0;  // next significant line
  auto lineno = [&](size_t sidx) { return (size_t)t.sig[sidx] + 1; };
  auto eof_line = [&]() { return nl; };  // the reader's line count at EOF
  bool have_points = false, have_elements = false;
  std::vector<Block> pblocks, eblocks;
  std::vector<size_t> point_sig, elem_sig;  // significant-line index of every point / element
  struct MarkerBlock {
    size_t first, count;
  };
  std::vector<MarkerBlock> mblocks;
  std::string key, value;
  // a structural failure stops the sequential reader: remember it, parse the
  // blocks before it, report the smallest line
  size_t stop_line = SIZE_MAX;
  std::string stop_what;
  auto stop = [&](size_t line, std::string w) {
    stop_line = line;
    stop_what = std::move(w);
  };
  while (s < t.sig.size() && stop_line == SIZE_MAX) {
    const size_t here = lineno(s);
    const std::string_view line = t.body(t.sig[s]);
    ++s;
    if (!split_keyword(line, key, value)) {
      stop(here, "expected a section keyword, got '" + std::string(line) + "'");
      break;
    }
    if (key == "NDIME") {
      size_t d = 0;
      if (!parse_index(value, d) || (d != 2 && d != 3)) {
        stop(here, "NDIME must be 2 or 3");
        break;
      }
      m.dim = (int)d;
    } else if (key == "NPOIN") {
      if (m.dim == 0) {
        stop(here, "NPOIN before NDIME");
        break;
      }
      size_t count = 0;
      if (!parse_index(value, count)) {
        stop(here, "bad NPOIN value '" + value + "'");
        break;
      }
      const size_t avail = t.sig.size() - s;
      pblocks.push_back({s, std::min(count, avail)});
      m.block_dims.push_back(m.dim);
      if (count > avail) {
        s = t.sig.size();
        stop(eof_line(), "unexpected end of file in NPOIN");
        break;
      }
      s += count;
      have_points = true;
    } else if (key == "NELEM") {
      size_t count = 0;
      if (!parse_index(value, count)) {
        stop(here, "bad NELEM value '" + value + "'");
        break;
      }
      const size_t avail = t.sig.size() - s;
      eblocks.push_back({s, std::min(count, avail)});
      if (count > avail) {
        s = t.sig.size();
        stop(eof_line(), "unexpected end of file in NELEM");
        break;
      }
      s += count;
      have_elements = true;
    } else if (key == "NMARK") {
      size_t count = 0;
      if (!parse_index(value, count)) {
        stop(here, "bad NMARK value '" + value + "'");
        break;
      }
      for (size_t mk = 0; mk < count && stop_line == SIZE_MAX; ++mk) {
        if (s >= t.sig.size()) {
          stop(eof_line(), "expected MARKER_TAG");
          break;
        }
        const size_t l1 = lineno(s);
        if (!split_keyword(t.body(t.sig[s++]), key, value) || key != "MARKER_TAG") {
          stop(l1, "expected MARKER_TAG");
          break;
        }
        HostMesh::Marker mark;
        mark.name = value;
        if (mark.name.empty()) {
          stop(l1, "empty marker name");
          break;
        }
        if (s >= t.sig.size()) {
          stop(eof_line(), "expected MARKER_ELEMS");
          break;
        }
        const size_t l2 = lineno(s);
        if (!split_keyword(t.body(t.sig[s++]), key, value) || key != "MARKER_ELEMS") {
          stop(l2, "expected MARKER_ELEMS");
          break;
        }
        size_t elems = 0;
        if (!parse_index(value, elems)) {
          stop(l2, "bad MARKER_ELEMS value '" + value + "'");
          break;
        }
        const size_t avail = t.sig.size() - s;
        mblocks.push_back({s, std::min(elems, avail)});
        m.markers.push_back(std::move(mark));
        if (elems > avail) {
          s = t.sig.size();
          stop(eof_line(), "unexpected end of file in marker");
          break;
        }
        s += elems;
      }
    } else {
      stop(here, "unknown section '" + key + "'");
      break;
    }
  }
  // ---- blocks (parallel) -------------------------------------------------------
  size_t np = 0, ne = 0;
  for (auto& b : pblocks) np += b.count;
  for (auto& b : eblocks) ne += b.count;
  m.xyz.assign(3 * np, 0.0);
  m.point_line.resize(np);
  {
    // points: block-major, chunks of 64k lines
    struct Job {
      size_t blk, first, count, out;
    };
    std::vector<Job> jobs;
    size_t out = 0;
    for (size_t bi = 0; bi < pblocks.size(); ++bi) {
      for (size_t i = 0; i < pblocks[bi].count; i += 65536)
        jobs.push_back({bi, pblocks[bi].first + i, std::min<size_t>(65536, pblocks[bi].count - i), out + i});
      out += pblocks[bi].count;
    }
    pool.run((int)jobs.size(), [&](int ji) {
      const Job& j = jobs[ji];
      const int dim = m.block_dims[j.blk];
      for (size_t k = 0; k < j.count; ++k) {
        const size_t sl = j.first + k;
        const size_t line = lineno(sl);
        m.point_line[j.out + k] = line;
        double* p = &m.xyz[3 * (j.out + k)];
        // mesh_io.cpp:162-173: enough tokens first, then each coordinate
        std::string_view tok[3];
        int d = 0;
        for_tokens(t.body(t.sig[sl]), [&](std::string_view s) {
          tok[d++] = s;
          return d < dim;
        });
        if (d < dim) {
          err.offer(line, "point needs " + std::to_string(dim) + " coordinates");
          return;
        }
        for (int a = 0; a < dim; ++a)
          if (!parse_double(tok[a], p[a])) {
            err.offer(line, "bad coordinate '" + std::string(tok[a]) + "'");
            return;
          }
      }
    });
  }
  m.kinds.assign(ne, 0);
  m.offsets.assign(ne + 1, 0);
  m.elem_line.resize(ne);
  std::vector<size_t> eidx(ne * 8, 0);
  {
    struct Job {
      size_t first, count, out;
    };
    std::vector<Job> jobs;
    size_t out = 0;
    for (auto& b : eblocks) {
      for (size_t i = 0; i < b.count; i += 65536)
        jobs.push_back({b.first + i, std::min<size_t>(65536, b.count - i), out + i});
      out += b.count;
    }
    pool.run((int)jobs.size(), [&](int ji) {
      const Job& j = jobs[ji];
      for (size_t k = 0; k < j.count; ++k) {
        const size_t sl = j.first + k, e = j.out + k;
        m.elem_line[e] = lineno(sl);
        int kind;
        const std::string w = parse_element(t.body(t.sig[sl]), kind, &eidx[8 * e]);
        if (!w.empty()) {
          err.offer(lineno(sl), w);
          return;
        }
        m.kinds[e] = kind;
      }
    });
  }
  for (size_t mi = 0; mi < mblocks.size(); ++mi) {  // markers: small, sequential
    auto& mk = m.markers[mi];
    mk.offsets.assign(1, 0);
    for (size_t k = 0; k < mblocks[mi].count; ++k) {
      const size_t sl = mblocks[mi].first + k;
      int kind;
      size_t nodes[8];
      const std::string w = parse_element(t.body(t.sig[sl]), kind, nodes);
      if (!w.empty()) {
        err.offer(lineno(sl), w);
        break;
      }
      mk.kinds.push_back(kind);
      mk.conn.insert(mk.conn.end(), nodes, nodes + kCount[kind]);
      mk.offsets.push_back(mk.conn.size());
      mk.line.push_back(lineno(sl));
    }
  }
  if (stop_line != SIZE_MAX) err.offer(stop_line, stop_what);
  if (err.line.load() != SIZE_MAX) fail(t, err.line.load(), err.what);
  // end of file checks (mesh_io.cpp:219-222), at the reader's final line
  if (m.dim == 0) fail(t, nl, "missing NDIME section");
  if (!have_points) fail(t, nl, "missing NPOIN section");
  if (!have_elements) fail(t, nl, "missing NELEM section");
  if (m.markers.empty()) fail(t, nl, "mesh declares no boundary markers");
  // element CSR
  for (size_t e = 0; e < ne; ++e) m.offsets[e + 1] = m.offsets[e] + kCount[m.kinds[e]];
  m.conn.resize(m.offsets[ne]);
  pool.run((int)std::min<size_t>(64, ne / 65536 + 1), [&](int c) {
    const size_t nc = std::min<size_t>(64, ne / 65536 + 1);
    for (size_t e = ne * c / nc; e < ne * (c + 1) / nc; ++e)
      for (int k = 0; k < kCount[m.kinds[e]]; ++k) m.conn[m.offsets[e] + k] = eidx[8 * e + k];
  });
  // ---- validation (mesh_io.cpp:224-250), in the reference's order -----------
  const size_t nn = np;
  auto check = [&](int kind, const size_t* nodes, size_t line, bool boundary) {
    const bool ok = boundary ? is_boundary_kind(kind, m.dim) : is_volume_kind(kind, m.dim);
    if (!ok)
      fail(t, line, "element kind '" + std::string(kName[kind]) + "' not allowed here for a " +
                        std::to_string(m.dim) + "D mesh");
    for (int k = 0; k < kCount[kind]; ++k)
      if (nodes[k] >= nn)
        fail(t, line, "node index " + std::to_string(nodes[k]) + " out of range (mesh has " +
                          std::to_string(nn) + " nodes)");
  };
  {
    std::atomic<size_t> first_bad{SIZE_MAX};
    const int nc = (int)std::min<size_t>(256, ne / 65536 + 1);
    pool.run(nc, [&](int c) {
      for (size_t e = ne * c / nc; e < ne * (c + 1) / nc; ++e) {
        const int kind = m.kinds[e];
        bool bad = !is_volume_kind(kind, m.dim);
        for (int k = 0; k < kCount[kind] && !bad; ++k) bad = m.conn[m.offsets[e] + k] >= nn;
        if (bad) {
          size_t cur = first_bad.load();
          while (e < cur && !first_bad.compare_exchange_weak(cur, e)) {
          }
          return;
        }
      }
    });
    if (first_bad.load() != SIZE_MAX) {
      const size_t e = first_bad.load();
      check(m.kinds[e], &m.conn[m.offsets[e]], m.elem_line[e], false);
    }
  }
  for (auto& mk : m.markers) {
    for (size_t i = 0; i < mk.kinds.size(); ++i)
      check(mk.kinds[i], &mk.conn[mk.offsets[i]], mk.line[i], true);
    // marker_nodes_from_elements (mesh.cpp:92-102): first-appearance order
    std::vector<size_t> seen;
    seen.reserve(mk.conn.size());
    for (size_t v : mk.conn) seen.push_back(v);
    std::vector<size_t> order(seen.size());
    for (size_t i = 0; i < order.size(); ++i) order[i] = i;
    std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) { return seen[a] < seen[b]; });
    std::vector<unsigned char> keep(seen.size(), 0);
    for (size_t i = 0; i < order.size(); ++i)
      if (i == 0 || seen[order[i]] != seen[order[i - 1]]) keep[order[i]] = 1;
    for (size_t i = 0; i < seen.size(); ++i)
      if (keep[i]) mk.nodes.push_back(seen[i]);
  }
  // duplicate nodes (find_coincident_nodes, mesh.cpp:104-157) on the device
  size_t di = 0, dj = 0;
  if (coincident_nodes(ctx, m.xyz.data(), nn, di, dj))
    fail(t, m.point_line[dj], "duplicate node: coincides with node " + std::to_string(di) +
                                  " (line " + std::to_string(m.point_line[di]) + ")");
  return m;
}

// ---- coincident nodes ------------------------------------------------------------
namespace {

struct Cell {
  long long a, b, c;
};

__device__ __forceinline__ unsigned long long cell_hash(long long a, long long b, long long c) {
  unsigned long long h = (unsigned long long)a * 0x9e3779b97f4a7c15ull;
  h ^= (unsigned long long)b * 0xc2b2ae3d27d4eb4full + (h << 6) + (h >> 2);
  h ^= (unsigned long long)c * 0x165667b19e3779f9ull + (h << 6) + (h >> 2);
  return h;
}

__global__ void k_cells(const double* x, const double* y, const double* z, size_t n, double lx,
                        double ly, double lz, double tol, long long* ca, long long* cb,
                        long long* cc, unsigned long long* key, unsigned* idx) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  // mesh.cpp:131-135: floor((p - lo) / tol) per axis
  const long long a = (long long)floor(exact::div(exact::sub(x[i], lx), tol));
  const long long b = (long long)floor(exact::div(exact::sub(y[i], ly), tol));
  const long long c = (long long)floor(exact::div(exact::sub(z[i], lz), tol));
  ca[i] = a, cb[i] = b, cc[i] = c;
  key[i] = cell_hash(a, b, c);
  idx[i] = (unsigned)i;
}

__global__ void k_probe(const double* x, const double* y, const double* z, size_t n, double tol,
                        const long long* ca, const long long* cb, const long long* cc,
                        const unsigned long long* skey, const unsigned* sidx,
                        unsigned long long* best) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  for (long long da = -1; da <= 1; ++da)
    for (long long db = -1; db <= 1; ++db)
      for (long long dc = -1; dc <= 1; ++dc) {
        const long long a = ca[i] + da, b = cb[i] + db, c = cc[i] + dc;
        const unsigned long long h = cell_hash(a, b, c);
        size_t lo = 0, hi = n;
        while (lo < hi) {
          const size_t mid = (lo + hi) >> 1;
          if (skey[mid] < h) lo = mid + 1; else hi = mid;
        }
        for (size_t s = lo; s < n && skey[s] == h; ++s) {
          const unsigned j = sidx[s];  // ascending within equal hashes (stable sort)
          if (j >= i) break;
          if (ca[j] != a || cb[j] != b || cc[j] != c) continue;
          if (exact::dist(x[i], y[i], z[i], x[j], y[j], z[j]) <= tol) {
            atomicMin(best, ((unsigned long long)i << 32) | j);
            return;
          }
        }
      }
}

}  // namespace

bool coincident_nodes(Context& ctx, const double* xyz, size_t n, size_t& first, size_t& second) {
  if (n < 2) return false;
  if (n >= 0xffffffffull) throw InvalidArgument("duplicate-node check: too many nodes");
  double lo[3] = {xyz[0], xyz[1], xyz[2]}, hi[3] = {xyz[0], xyz[1], xyz[2]};
  for (size_t i = 0; i < n; ++i)
    for (int a = 0; a < 3; ++a)
      lo[a] = std::min(lo[a], xyz[3 * i + a]), hi[a] = std::max(hi[a], xyz[3 * i + a]);
  const double dx = lo[0] - hi[0], dy = lo[1] - hi[1], dz = lo[2] - hi[2];
  const double diag = std::sqrt(dx * dx + dy * dy + dz * dz);  // distance(lo, hi)
  if (diag == 0.0) {
    first = 0, second = 1;
    return true;
  }
  const double tol = 1e-12 * diag;
  DPoints p;
  upload_points(ctx, xyz, n, p);
  DBuf<long long> ca, cb, cc;
  DBuf<unsigned long long> key, skey, best;
  DBuf<unsigned> idx, sidx;
  ca.reserve(n), cb.reserve(n), cc.reserve(n);
  key.reserve(n), skey.reserve(n), idx.reserve(n), sidx.reserve(n), best.reserve(1);
  const unsigned nb = (unsigned)((n + 255) / 256);
  k_cells<<<nb, 256, 0, ctx.stream>>>(p.x.p, p.y.p, p.z.p, n, lo[0], lo[1], lo[2], tol, ca.p, cb.p,
                                      cc.p, key.p, idx.p);
  size_t temp = 0;
  IMB_CHECK(cub::DeviceRadixSort::SortPairs(nullptr, temp, key.p, skey.p, idx.p, sidx.p, (int)n, 0,
                                            64, ctx.stream));
  DBuf<unsigned char> tb;
  tb.reserve(temp);
  IMB_CHECK(cub::DeviceRadixSort::SortPairs(tb.p, temp, key.p, skey.p, idx.p, sidx.p, (int)n, 0, 64,
                                            ctx.stream));
  IMB_CHECK(cudaMemsetAsync(best.p, 0xff, 8, ctx.stream));
  k_probe<<<nb, 256, 0, ctx.stream>>>(p.x.p, p.y.p, p.z.p, n, tol, ca.p, cb.p, cc.p, skey.p, sidx.p,
                                      best.p);
  IMB_LAUNCH_CHECK();
  unsigned long long h = 0;
  IMB_CHECK(cudaMemcpyAsync(&h, best.p, 8, cudaMemcpyDeviceToHost, ctx.stream));
  IMB_CHECK(cudaStreamSynchronize(ctx.stream));
  if (h == ~0ull) return false;
  second = (size_t)(h >> 32), first = (size_t)(h & 0xffffffffull);
  return true;
}

// ---- writer (mesh_io.cpp:269-309) ------------------------------------------------
void write_su2_file(HostPool& pool, const std::string& path, const HostMesh& m) {
  FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) throw std::runtime_error("cannot write mesh file '" + path + "'");
  std::unique_ptr<FILE, int (*)(FILE*)> guard(f, std::fclose);
  auto put = [&](const std::string& s) {
    if (std::fwrite(s.data(), 1, s.size(), f) != s.size())
      throw std::runtime_error("failed while writing '" + path + "'");
  };
  auto elem_line = [&](std::string& s, int kind, const size_t* nodes) {
    char tmp[32];
    auto r = std::to_chars(tmp, tmp + 32, kVtk[kind]);
    s.append(tmp, r.ptr);
    for (int k = 0; k < kCount[kind]; ++k) {
      s.push_back(' ');
      r = std::to_chars(tmp, tmp + 32, nodes[k]);
      s.append(tmp, r.ptr);
    }
    s.push_back('\n');
  };
  const size_t ne = m.kinds.size(), nn = m.xyz.size() / 3;
  put("NDIME= " + std::to_string(m.dim) + "\n");
  put("NELEM= " + std::to_string(ne) + "\n");
  const size_t chunk = 1 << 16;
  auto parallel_put = [&](size_t count, auto&& fmt) {
    for (size_t b0 = 0; b0 < count; b0 += chunk * 64) {  // bounded memory: 64 chunks at a time
      const size_t b1 = std::min(count, b0 + chunk * 64);
      const int nj = (int)((b1 - b0 + chunk - 1) / chunk);
      std::vector<std::string> out(nj);
      pool.run(nj, [&](int j) {
        const size_t s = b0 + (size_t)j * chunk, e = std::min(b1, s + chunk);
        out[j].reserve((e - s) * 64);
        for (size_t i = s; i < e; ++i) fmt(out[j], i);
      });
      for (auto& s : out) put(s);
    }
  };
  parallel_put(ne, [&](std::string& s, size_t e) { elem_line(s, m.kinds[e], &m.conn[m.offsets[e]]); });
  put("NPOIN= " + std::to_string(nn) + "\n");
  parallel_put(nn, [&](std::string& s, size_t i) {
    char tmp[96];
    int k = m.dim == 3 ? std::snprintf(tmp, sizeof tmp, "%.17g %.17g %.17g\n", m.xyz[3 * i],
                                       m.xyz[3 * i + 1], m.xyz[3 * i + 2])
                       : std::snprintf(tmp, sizeof tmp, "%.17g %.17g\n", m.xyz[3 * i], m.xyz[3 * i + 1]);
    s.append(tmp, (size_t)k);
  });
  put("NMARK= " + std::to_string(m.markers.size()) + "\n");
  for (const auto& mk : m.markers) {
    std::string s = "MARKER_TAG= " + mk.name + "\nMARKER_ELEMS= " + std::to_string(mk.kinds.size()) + "\n";
    for (size_t i = 0; i < mk.kinds.size(); ++i) elem_line(s, mk.kinds[i], &mk.conn[mk.offsets[i]]);
    put(s);
  }
}

}  // namespace imb
