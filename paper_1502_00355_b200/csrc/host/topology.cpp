// Host mesh prep (include/trismooth/topology.hpp, include/trismooth/gpu.hpp).
//
// find_neighbors reproduces the reference's Adjacency exactly (proj/src/topology.cpp:12-65):
// raw rows in triangle-visit order (two entries per incidence: the corners other than v, in
// corner order), incident rows ascending, unique = sorted + deduplicated with multiplicities.
// The per-vertex sort/dedup runs on all host cores for large meshes.  build_topology is the
// 64-bit variant the device path uses: it skips the raw list (which overflows int at
// 6*nt > 2^31-1) and derives the same unique rows straight from the incident triangles.
#include <algorithm>
#include <thread>
#include <unordered_map>

#include "trismooth/gpu.hpp"
#include "trismooth/parallel.hpp"
#include "trismooth/topology.hpp"

namespace trismooth {

namespace {

int host_threads(int64_t work) {
  const unsigned hc = std::max(1u, std::thread::hardware_concurrency());
  return static_cast<int>(std::min<int64_t>(std::min<unsigned>(hc, 64u), work / 50000 + 1));
}

template <class F>
void split_run(int64_t n, F&& fn) {
  const int T = host_threads(n);
  if (T <= 1) {
    fn(int64_t{0}, n);
    return;
  }
  std::vector<std::thread> pool;
  const int64_t step = (n + T - 1) / T;
  for (int t = 0; t < T; ++t) {
    const int64_t b = std::min(n, t * step), e = std::min(n, b + step);
    pool.emplace_back([&fn, b, e] { fn(b, e); });
  }
  for (auto& th : pool) th.join();
}

// Sorted-unique rows with multiplicities, from per-vertex candidate rows given by `fill`
// (fill(v, scratch) appends v's raw entries).  Two passes: count, then write.
template <class Off, class Val, class Fill>
void unique_rows(int64_t nv, Fill&& fill, std::vector<Off>& off, std::vector<Val>& vals,
                 std::vector<int>* mult, std::vector<uint8_t>* pinned) {
  std::vector<int64_t> cnt(nv, 0);
  split_run(nv, [&](int64_t b, int64_t e) {
    std::vector<int32_t> row;
    for (int64_t v = b; v < e; ++v) {
      row.clear();
      fill(v, row);
      std::sort(row.begin(), row.end());
      cnt[v] = std::unique(row.begin(), row.end()) - row.begin();
    }
  });
  off.assign(nv + 1, 0);
  for (int64_t v = 0; v < nv; ++v) off[v + 1] = static_cast<Off>(off[v] + cnt[v]);
  vals.resize(static_cast<size_t>(off[nv]));
  if (mult) mult->resize(static_cast<size_t>(off[nv]));
  if (pinned) pinned->assign(nv, 0);
  split_run(nv, [&](int64_t b, int64_t e) {
    std::vector<int32_t> row;
    for (int64_t v = b; v < e; ++v) {
      row.clear();
      fill(v, row);
      std::sort(row.begin(), row.end());
      int64_t o = off[v];
      bool pin = row.empty();
      for (size_t i = 0; i < row.size();) {
        size_t j = i + 1;
        while (j < row.size() && row[j] == row[i]) ++j;
        vals[o] = row[i];
        if (mult) (*mult)[o] = static_cast<int>(j - i);
        pin = pin || (j - i) != 2;
        ++o;
        i = j;
      }
      if (pinned) (*pinned)[v] = pin ? 1 : 0;
    }
  });
}

template <class Storage>
Adjacency adjacency_of(Storage& m) {
  const int nv = m.vertex_count(), nt = m.triangle_count();
  Adjacency adj;
  adj.raw.offsets.assign(nv + 1, 0);
  adj.incident.offsets.assign(nv + 1, 0);
  for (int t = 0; t < nt; ++t)
    for (const int v : m.tri(t)) {
      adj.raw.offsets[v + 1] += 2;
      adj.incident.offsets[v + 1] += 1;
    }
  for (int v = 0; v < nv; ++v) {
    adj.raw.offsets[v + 1] += adj.raw.offsets[v];
    adj.incident.offsets[v + 1] += adj.incident.offsets[v];
  }
  adj.raw.values.resize(adj.raw.offsets[nv]);
  adj.incident.values.resize(adj.incident.offsets[nv]);
  std::vector<int> rpos(adj.raw.offsets.begin(), adj.raw.offsets.end() - 1);
  std::vector<int> ipos(adj.incident.offsets.begin(), adj.incident.offsets.end() - 1);
  for (int t = 0; t < nt; ++t) {
    const auto c = m.tri(t);
    for (int k = 0; k < 3; ++k) {
      const int v = c[k];
      // the corners other than v, in corner order
      adj.raw.values[rpos[v]++] = c[k == 0 ? 1 : 0];
      adj.raw.values[rpos[v]++] = c[k == 2 ? 1 : 2];
      adj.incident.values[ipos[v]++] = t;
    }
  }
  const Csr& raw = adj.raw;
  unique_rows<int, int>(
      nv,
      [&](int64_t v, std::vector<int32_t>& row) {
        const auto r = raw.row(static_cast<int>(v));
        row.insert(row.end(), r.begin(), r.end());
      },
      adj.unique.offsets, adj.unique.values, &adj.multiplicity, nullptr);
  m.assign_adjacency(adj.unique, adj.incident);
  return adj;
}

uint64_t undirected(int a, int b) {
  const uint32_t lo = static_cast<uint32_t>(std::min(a, b)), hi = static_cast<uint32_t>(std::max(a, b));
  return (static_cast<uint64_t>(lo) << 32) | hi;
}

std::unordered_map<uint64_t, int> edge_uses(const Mesh& mesh) {
  std::unordered_map<uint64_t, int> uses;
  uses.reserve(static_cast<size_t>(mesh.triangle_count()) * 2);
  mesh.visit([&](const auto& m) {
    for (int t = 0; t < m.triangle_count(); ++t) {
      const auto c = m.tri(t);
      ++uses[undirected(c[0], c[1])];
      ++uses[undirected(c[1], c[2])];
      ++uses[undirected(c[2], c[0])];
    }
  });
  return uses;
}

}  // namespace

Adjacency find_neighbors(Mesh& mesh) {
  return mesh.visit([](auto& m) { return adjacency_of(m); });
}

void determine_constraints(Mesh& mesh, const Adjacency& adj, ThreadPool* pool) {
  mesh.visit([&](auto& m) {
    auto classify = [&](int b, int e) {
      for (int v = b; v < e; ++v) {
        const int lo = adj.unique.offsets[v], hi = adj.unique.offsets[v + 1];
        bool pin = lo == hi;
        for (int i = lo; i < hi && !pin; ++i) pin = adj.multiplicity[i] != 2;
        m.set_boundary(v, pin);
      }
    };
    const int nv = m.vertex_count();
    if (!pool) {
      classify(0, nv);
      return;
    }
    const int w = pool->workers();
    pool->run(w, [&](int i) {
      const ChunkRange r = worker_chunk(nv, w, i);
      classify(r.begin, r.end);
    });
  });
}

std::vector<bool> boundary_oracle(const Mesh& mesh) {
  std::vector<bool> out(mesh.vertex_count(), false);
  for (const auto& [key, n] : edge_uses(mesh))
    if (n == 1) {
      out[static_cast<size_t>(key >> 32)] = true;
      out[static_cast<size_t>(key & 0xffffffffu)] = true;
    }
  return out;
}

int non_manifold_edge_count(const Mesh& mesh) {
  int count = 0;
  for (const auto& kv : edge_uses(mesh)) count += kv.second > 2 ? 1 : 0;
  return count;
}

namespace gpu {

Topology64 build_topology(int64_t nv, const int32_t* tri, int64_t nt) {
  Topology64 T;
  T.inc_off.assign(nv + 1, 0);
  for (int64_t i = 0; i < 3 * nt; ++i) {
    const int32_t v = tri[i];
    if (v < 0 || v >= nv) throw StructuralError("triangle references a vertex out of range");
    ++T.inc_off[v + 1];
  }
  for (int64_t v = 0; v < nv; ++v) T.inc_off[v + 1] += T.inc_off[v];
  T.inc.resize(static_cast<size_t>(T.inc_off[nv]));
  {
    std::vector<int64_t> pos(T.inc_off.begin(), T.inc_off.end() - 1);
    for (int64_t t = 0; t < nt; ++t)
      for (int k = 0; k < 3; ++k) T.inc[pos[tri[3 * t + k]]++] = static_cast<int32_t>(t);
  }
  unique_rows<int64_t, int32_t>(
      nv,
      [&](int64_t v, std::vector<int32_t>& row) {
        for (int64_t i = T.inc_off[v]; i < T.inc_off[v + 1]; ++i) {
          const int32_t* c = tri + 3 * static_cast<int64_t>(T.inc[i]);
          for (int k = 0; k < 3; ++k)
            if (c[k] != v) row.push_back(c[k]);
        }
      },
      T.nbr_off, T.nbr, nullptr, &T.boundary);
  return T;
}

}  // namespace gpu

}  // namespace trismooth
