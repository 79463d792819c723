// Host-side preparation of the device mesh.  See tsg_prep.hpp.
#include "tsg_prep.hpp"

#include <algorithm>
#include <atomic>
#include <cmath>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <thread>

namespace tsg {

namespace {

uint32_t fan_pack_h(uint32_t i1, uint32_t i2, uint32_t k) { return i1 | (i2 << 15) | (k << 30); }

int worker_count(int64_t n) {
  const unsigned hc = std::max(1u, std::thread::hardware_concurrency());
  const int64_t by_size = n / 65536 + 1;
  return static_cast<int>(std::min<int64_t>(std::min<unsigned>(hc, 64u), by_size));
}

// Contiguous static split of [0, n) over threads; fn(begin, end).
template <class F>
void parallel_ranges(int64_t n, F&& fn) {
  const int T = worker_count(n);
  if (T <= 1) {
    fn(int64_t{0}, n);
    return;
  }
  std::vector<std::thread> th;
  const int64_t step = (n + T - 1) / T;
  for (int t = 0; t < T; ++t) {
    const int64_t b = std::min<int64_t>(n, t * step), e = std::min<int64_t>(n, b + step);
    th.emplace_back([&fn, b, e] { fn(b, e); });
  }
  for (auto& x : th) x.join();
}

// Sorts 64-bit keys in parallel: per-thread std::sort, then pairwise merges.
void parallel_sort(std::vector<uint64_t>& keys) {
  const int64_t n = static_cast<int64_t>(keys.size());
  int T = worker_count(n);
  int P = 1;
  while (P * 2 <= T) P *= 2;
  if (P <= 1) {
    std::sort(keys.begin(), keys.end());
    return;
  }
  std::vector<int64_t> cut(P + 1);
  for (int i = 0; i <= P; ++i) cut[i] = n * i / P;
  {
    std::vector<std::thread> th;
    for (int i = 0; i < P; ++i)
      th.emplace_back([&, i] { std::sort(keys.begin() + cut[i], keys.begin() + cut[i + 1]); });
    for (auto& x : th) x.join();
  }
  for (int width = 1; width < P; width *= 2) {
    std::vector<std::thread> th;
    for (int i = 0; i + width < P; i += 2 * width) {
      const int64_t b = cut[i], m = cut[i + width], e = cut[std::min(i + 2 * width, P)];
      th.emplace_back([&keys, b, m, e] {
        std::inplace_merge(keys.begin() + b, keys.begin() + m, keys.begin() + e);
      });
    }
    for (auto& x : th) x.join();
  }
}

// Hilbert index of (x, y) on a 2^16 x 2^16 lattice.
uint32_t hilbert_d(uint32_t x, uint32_t y) {
  uint32_t d = 0;
  for (uint32_t s = 1u << 15; s > 0; s >>= 1) {
    const uint32_t rx = (x & s) ? 1u : 0u, ry = (y & s) ? 1u : 0u;
    d += s * s * ((3u * rx) ^ ry);
    if (ry == 0) {
      if (rx == 1) {
        x = 0xffffu - x;
        y = 0xffffu - y;
      }
      std::swap(x, y);
    }
  }
  return d;
}

// TSG_PREP_TIMING=1: per-phase wall times of build_host_mesh on stderr (profiling aid).
struct PhaseTimer {
  bool on = std::getenv("TSG_PREP_TIMING") != nullptr;
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  void mark(const char* what) {
    if (!on) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[tsg prep] %-24s %8.1f ms\n", what, std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};

}  // namespace

// Tile records (see tsg_prep.hpp).  Per tile: the sorted external slots referenced by its
// small rows; the small rows grouped by valence (slot order inside a group), each group's
// words stored entry-major: word j of the k-th row of a group of n rows at group base + j*n + k.
std::string build_tiles(HostMesh& hm, const std::vector<uint32_t>& deg, int32_t max_deg) {
  const int64_t nv = hm.nv;
  const int64_t kTile = hm.tile;
  const int64_t ntiles = (nv + kTile - 1) / kTile;
  hm.tmeta.assign(nv, 0);
  hm.tile_rec.assign(ntiles + 1, 0);
  hm.ext_off.assign(ntiles + 1, 0);
  std::vector<std::vector<uint32_t>> ext(ntiles);
  std::vector<uint32_t> words(ntiles, 0);
  auto is_small = [&](int64_t s) { return deg[s] >= 1 && deg[s] <= static_cast<uint32_t>(max_deg); };
  parallel_ranges(ntiles, [&](int64_t tb, int64_t te) {
    for (int64_t t = tb; t < te; ++t) {
      const int64_t base = t * kTile, end = std::min(nv, base + kTile);
      auto& E = ext[t];
      uint32_t count[kMaxCycleDeg + 1] = {};
      for (int64_t s = base; s < end; ++s) {
        if (!is_small(s)) continue;
        ++count[deg[s]];
        for (uint32_t j = hm.off[s]; j < hm.off[s + 1]; ++j) {
          const int64_t u = hm.nbr[j];
          if (u < base || u >= end) E.push_back(static_cast<uint32_t>(u));
        }
      }
      uint32_t gbase[kMaxCycleDeg + 1], fill[kMaxCycleDeg + 1] = {}, w = 0;
      for (int d = 1; d <= max_deg; ++d) {
        gbase[d] = w;
        w += static_cast<uint32_t>(d) * count[d];
      }
      for (int64_t s = base; s < end; ++s) {
        if (!is_small(s)) continue;
        const uint32_t d = deg[s], k = fill[d]++;
        hm.tmeta[s] = (gbase[d] + k) | (d << kMetaDegShift) | (count[d] << kMetaStrideShift);
      }
      std::sort(E.begin(), E.end());
      E.erase(std::unique(E.begin(), E.end()), E.end());
      words[t] = (w + 3) / 4 * 4;  // tiles start 16-byte aligned
    }
  });
  uint64_t wu = 0, eu = 0;
  int32_t max_ext = 0, max_words = 0;
  for (int64_t t = 0; t < ntiles; ++t) {
    hm.tile_rec[t] = static_cast<uint32_t>(wu);
    hm.ext_off[t] = static_cast<uint32_t>(eu);
    wu += words[t];
    eu += ext[t].size();
    max_ext = std::max<int32_t>(max_ext, static_cast<int32_t>(ext[t].size()));
    max_words = std::max<int32_t>(max_words, static_cast<int32_t>(words[t]));
  }
  hm.tile_rec[ntiles] = static_cast<uint32_t>(wu);
  hm.ext_off[ntiles] = static_cast<uint32_t>(eu);
  if (kTile + max_ext >= static_cast<int64_t>(kNoLocal))
    return "a tile references more than " + std::to_string(kNoLocal - kTile - 1) + " external vertices";
  if (max_words > static_cast<int32_t>(kMetaBaseMask) + 1) return "tile words exceed the meta offset field";
  if (wu >= 0xffffffffULL) return "tile records exceed 2^32 words";
  hm.max_ext = max_ext;
  hm.max_rec_words = max_words;
  hm.ext.resize(eu);
  hm.trec.assign(wu, 0);
  parallel_ranges(ntiles, [&](int64_t tb, int64_t te) {
    for (int64_t t = tb; t < te; ++t) {
      const int64_t base = t * kTile, end = std::min(nv, base + kTile);
      const auto& E = ext[t];
      std::copy(E.begin(), E.end(), hm.ext.begin() + hm.ext_off[t]);
      auto local = [&](int64_t u) -> uint32_t {
        if (u >= base && u < end) return static_cast<uint32_t>(u - base);
        const auto it = std::lower_bound(E.begin(), E.end(), static_cast<uint32_t>(u));
        return static_cast<uint32_t>(kTile + (it - E.begin()));
      };
      for (int64_t s = base; s < end; ++s) {
        if (!is_small(s)) continue;
        const uint32_t meta = hm.tmeta[s];
        uint32_t* r = hm.trec.data() + hm.tile_rec[t] + (meta & kMetaBaseMask);
        const uint32_t stride = meta >> kMetaStrideShift;
        const uint32_t o0 = hm.off[s], n = deg[s];
        const bool cyc = hm.has_cycle[s] != 0;
        for (uint32_t j = 0; j < n; ++j) {
          const uint32_t row = local(hm.nbr[o0 + j]);
          const uint32_t cy = cyc ? local(hm.nbr[o0 + hm.cycpos[o0 + j]]) : kNoLocal;
          const uint32_t k = cyc ? hm.cycrot[o0 + j] : 0u;
          r[j * stride] = row | (cy << kWordCycleShift) | (k << kWordRotShift);
        }
      }
    }
  });
  return "";
}

void hilbert_order(int64_t nv, const double* xy, int64_t* order_out) {
  double xmin = INFINITY, xmax = -INFINITY, ymin = INFINITY, ymax = -INFINITY;
  for (int64_t v = 0; v < nv; ++v) {
    xmin = std::min(xmin, xy[2 * v]);
    xmax = std::max(xmax, xy[2 * v]);
    ymin = std::min(ymin, xy[2 * v + 1]);
    ymax = std::max(ymax, xy[2 * v + 1]);
  }
  const double sx = xmax > xmin ? 65535.0 / (xmax - xmin) : 0.0;
  const double sy = ymax > ymin ? 65535.0 / (ymax - ymin) : 0.0;
  std::vector<uint64_t> keys(static_cast<size_t>(nv));
  parallel_ranges(nv, [&](int64_t b, int64_t e) {
    for (int64_t v = b; v < e; ++v) {
      const double fx = std::isfinite(xy[2 * v]) ? (xy[2 * v] - xmin) * sx : 0.0;
      const double fy = std::isfinite(xy[2 * v + 1]) ? (xy[2 * v + 1] - ymin) * sy : 0.0;
      const uint32_t qx = static_cast<uint32_t>(std::clamp(fx, 0.0, 65535.0));
      const uint32_t qy = static_cast<uint32_t>(std::clamp(fy, 0.0, 65535.0));
      keys[v] = (static_cast<uint64_t>(hilbert_d(qx, qy)) << 32) | static_cast<uint64_t>(v);
    }
  });
  parallel_sort(keys);
  for (int64_t s = 0; s < nv; ++s) order_out[s] = static_cast<int64_t>(keys[s] & 0xffffffffu);
}

// Structural checks of a caller-supplied description before anything indexes through it
// (the reference's build_mesh raises StructuralError on the same conditions,
// proj/src/mesh.cpp:69-81): corner ids in range, CSR offsets starting at 0 and
// non-decreasing, entries in range, neighbour rows strictly ascending.  Runs in parallel
// chunks; returns the first problem found.
namespace {

std::string validate_topology(const tsg_mesh_desc& d) {
  const int64_t nv = d.nv, nt = d.nt;
  std::atomic<int> bad{0};  // bit 0 tri, 1 nbr, 2 inc
  parallel_ranges(nt, [&](int64_t b, int64_t e) {
    for (int64_t i = 3 * b; i < 3 * e; ++i)
      if (d.tri[i] < 0 || d.tri[i] >= nv) {
        bad.fetch_or(1);
        return;
      }
  });
  if (bad.load() & 1) return "triangle corner index out of range";
  if (d.nbr_off[0] != 0 || d.inc_off[0] != 0) return "CSR offsets must start at 0";
  parallel_ranges(nv, [&](int64_t b, int64_t e) {
    for (int64_t v = b; v < e; ++v) {
      const int64_t n0 = d.nbr_off[v], n1 = d.nbr_off[v + 1];
      const int64_t i0 = d.inc_off[v], i1 = d.inc_off[v + 1];
      if (n1 < n0) {
        bad.fetch_or(2);
        return;
      }
      if (i1 < i0) {
        bad.fetch_or(4);
        return;
      }
      for (int64_t j = n0; j < n1; ++j)
        if (d.nbr[j] < 0 || d.nbr[j] >= nv || (j > n0 && d.nbr[j] <= d.nbr[j - 1])) {
          bad.fetch_or(2);
          return;
        }
      for (int64_t j = i0; j < i1; ++j)
        if (d.inc[j] < 0 || d.inc[j] >= nt) {
          bad.fetch_or(4);
          return;
        }
    }
  });
  const int f = bad.load();
  if (f & 2) return "neighbour CSR malformed (offsets decreasing, id out of range or row not strictly ascending)";
  if (f & 4) return "incident CSR malformed (offsets decreasing or triangle id out of range)";
  return {};
}

}  // namespace

std::string validate_desc(const tsg_mesh_desc& d, bool topology) {
  const int64_t nv = d.nv;
  if (topology) {
    if (std::string e = validate_topology(d); !e.empty()) return e;
  }
  if (d.order) {
    std::vector<std::atomic<uint8_t>> seen(nv);
    std::atomic<bool> ok{true};
    parallel_ranges(nv, [&](int64_t b, int64_t e) {
      for (int64_t s = b; s < e; ++s) {
        const int64_t v = d.order[s];
        if (v < 0 || v >= nv || seen[v].exchange(1, std::memory_order_relaxed)) {
          ok = false;
          return;
        }
      }
    });
    if (!ok) return "order is not a permutation of 0..nv-1";
  }
  return {};
}

std::string build_host_mesh(const tsg_mesh_desc& d, const Tiers& tiers, HostMesh& hm, int32_t tile) {
  if (tile < 256 || tile > kTileMax || tile % 256) return "tile size must be a multiple of 256 in [256, 1536]";
  hm.tile = tile;
  const int64_t nv = d.nv, nt = d.nt;
  if (nv <= 0 || nt <= 0) return "mesh must have vertices and triangles";
  if (nv >= (int64_t{1} << 31) - 1) return "vertex count exceeds 2^31-1";
  PhaseTimer pt;
  if (std::string e = validate_desc(d); !e.empty()) return e;
  pt.mark("validate");
  hm.nv = nv;
  hm.nt = nt;
  hm.order.resize(nv);
  hm.rank.resize(nv);
  if (d.order) {
    {
      std::vector<std::atomic<uint8_t>> seen(nv);
      std::atomic<bool> ok{true};
      parallel_ranges(nv, [&](int64_t b, int64_t e) {
        for (int64_t s = b; s < e; ++s) {
          const int64_t v = d.order[s];
          if (v < 0 || v >= nv || seen[v].exchange(1, std::memory_order_relaxed)) {
            ok = false;
            return;
          }
          hm.order[s] = v;
        }
      });
      if (!ok) return "order is not a permutation of 0..nv-1";
    }
    // Degree sort inside windows of kSigma consecutive slots of the locality order (SELL-C-σ
    // style): warps then see near-uniform valences (no divergent loop tails) while every
    // window stays spatially compact.  Descending: a tile's longest rows are in its first
    // rounds, overlapping the other warps' work instead of forming a tail (measured: ascending
    // with dynamic rounds 31.7 G, descending with static rounds 33.3 G node-upd/s on cfg3).
    // Results do not depend on the slot order.
    const int64_t kSigma = hm.tile;  // windows coincide with the tiles of tile_update
    auto degree_key = [&](int64_t v) -> int64_t {
      return d.boundary[v] ? 0 : d.nbr_off[v + 1] - d.nbr_off[v];
    };
    parallel_ranges((nv + kSigma - 1) / kSigma, [&](int64_t b, int64_t e) {
      for (int64_t w = b; w < e; ++w) {
        auto first = hm.order.begin() + w * kSigma;
        auto last = hm.order.begin() + std::min(nv, (w + 1) * kSigma);
        std::stable_sort(first, last, [&](int64_t x, int64_t y) { return degree_key(x) > degree_key(y); });
      }
    });
    parallel_ranges(nv, [&](int64_t b, int64_t e) {
      for (int64_t s = b; s < e; ++s) hm.rank[hm.order[s]] = s;
    });
  } else {
    for (int64_t s = 0; s < nv; ++s) hm.order[s] = hm.rank[s] = s;
  }

  pt.mark("slot order");
  // Row lengths: movable vertices only; interior (all multiplicities 2) implies
  // #incident == #unique neighbours, which the fan encoding relies on.
  std::vector<uint32_t> deg(nv, 0);
  std::atomic<int64_t> bad{-1};
  std::atomic<int32_t> maxdeg{0};
  parallel_ranges(nv, [&](int64_t b, int64_t e) {
    int32_t local_max = 0;
    for (int64_t s = b; s < e; ++s) {
      const int64_t v = hm.order[s];
      if (d.boundary[v]) continue;
      const int64_t dn = d.nbr_off[v + 1] - d.nbr_off[v];
      const int64_t di = d.inc_off[v + 1] - d.inc_off[v];
      if (dn != di || dn <= 0 || dn >= 32768) bad = v;
      deg[s] = static_cast<uint32_t>(dn);
      local_max = std::max<int32_t>(local_max, static_cast<int32_t>(dn));
    }
    int32_t cur = maxdeg.load();
    while (local_max > cur && !maxdeg.compare_exchange_weak(cur, local_max)) {
    }
  });
  if (bad >= 0)
    return "movable vertex " + std::to_string(bad.load()) +
           " has inconsistent neighbour / incident counts (or degree >= 32768)";
  hm.max_deg = maxdeg;
  hm.off.assign(nv + 1, 0);
  uint64_t total = 0;
  for (int64_t s = 0; s < nv; ++s) {
    hm.off[s] = static_cast<uint32_t>(total);
    total += deg[s];
    if (total >= 0xffffffffULL) return "adjacency exceeds 2^32 entries";
  }
  hm.off[nv] = static_cast<uint32_t>(total);
  hm.nbr.assign(total, 0);
  hm.fan.assign(total, 0);
  hm.fan16.assign(total, 0);
  hm.cycpos.assign(total, 0);
  hm.cycrot.assign(total, 0);
  hm.has_cycle.assign(nv, 0);

  pt.mark("row lengths + alloc");
  // Device triangle order: identity, or by the smallest slot among the corners (stable) so
  // that the triangle kernels stream coordinates in the same locality order as the vertices.
  hm.tri_order.resize(nt);
  std::vector<int64_t> tri_rank(nt);
  if (!d.order) {
    for (int64_t t = 0; t < nt; ++t) hm.tri_order[t] = tri_rank[t] = t;
  } else {
    std::vector<uint64_t> keys(nt);
    parallel_ranges(nt, [&](int64_t b, int64_t e) {
      for (int64_t t = b; t < e; ++t) {
        const int64_t m = std::min({hm.rank[d.tri[3 * t]], hm.rank[d.tri[3 * t + 1]],
                                    hm.rank[d.tri[3 * t + 2]]});
        keys[t] = (static_cast<uint64_t>(m) << 32) | static_cast<uint64_t>(t);
      }
    });
    if (nt >= (int64_t{1} << 32)) return "triangle count exceeds 2^32";
    parallel_sort(keys);
    for (int64_t i = 0; i < nt; ++i) {
      hm.tri_order[i] = static_cast<int64_t>(keys[i] & 0xffffffffu);
      tri_rank[hm.tri_order[i]] = i;
    }
  }
  hm.tri.resize(3 * nt);
  parallel_ranges(nt, [&](int64_t b, int64_t e) {
    for (int64_t i = b; i < e; ++i) {
      const int64_t t = hm.tri_order[i];
      for (int k = 0; k < 3; ++k) hm.tri[3 * i + k] = static_cast<int32_t>(hm.rank[d.tri[3 * t + k]]);
    }
  });

  pt.mark("triangle order");
  std::atomic<int64_t> broken{-1};
  parallel_ranges(nv, [&](int64_t b, int64_t e) {
    for (int64_t s = b; s < e; ++s) {
      if (deg[s] == 0) continue;
      const int64_t v = hm.order[s];
      const int32_t* row = d.nbr + d.nbr_off[v];
      const int32_t n = static_cast<int32_t>(deg[s]);
      uint32_t* out_n = hm.nbr.data() + hm.off[s];
      uint32_t* out_f = hm.fan.data() + hm.off[s];
      for (int32_t j = 0; j < n; ++j) out_n[j] = static_cast<uint32_t>(hm.rank[row[j]]);
      const bool want_cycle = n <= kMaxCycleDeg;
      int8_t succ[kMaxCycleDeg], indeg[kMaxCycleDeg], rot[kMaxCycleDeg];
      bool cycle_ok = want_cycle;
      if (want_cycle)
        for (int32_t j = 0; j < n; ++j) succ[j] = -1, indeg[j] = 0;
      for (int64_t i = d.inc_off[v], j = 0; i < d.inc_off[v + 1]; ++i, ++j) {
        const int32_t* tv = d.tri + 3 * static_cast<int64_t>(d.inc[i]);
        const int k = tv[0] == v ? 0 : tv[1] == v ? 1 : 2;
        const int32_t a = tv[(k + 1) % 3], c = tv[(k + 2) % 3];
        const int32_t* pa = std::lower_bound(row, row + n, a);
        const int32_t* pc = std::lower_bound(row, row + n, c);
        if (tv[k] != v || pa == row + n || *pa != a || pc == row + n || *pc != c) {
          broken = v;
          return;
        }
        const uint32_t ia = static_cast<uint32_t>(pa - row), ic = static_cast<uint32_t>(pc - row);
        if (cycle_ok) {  // triangle = rotation of (v, a, c): directed link edge ia -> ic
          if (succ[ia] >= 0 || indeg[ic] > 0) {
            cycle_ok = false;
          } else {
            succ[ia] = static_cast<int8_t>(ic);
            indeg[ic] = 1;
            rot[ia] = static_cast<int8_t>(k);
          }
        }
        const int tier = tiers.tier(static_cast<uint32_t>(n));
        if (tier < 2) {
          // ring positions of (p1, p2, p3); v itself is the entry after the tier's last
          uint32_t p[3];
          p[k] = static_cast<uint32_t>(tier == 0 ? tiers.small_max : tiers.medium_max);
          p[(k + 1) % 3] = ia;
          p[(k + 2) % 3] = ic;
          hm.fan16[hm.off[s] + j] = static_cast<uint16_t>(p[0] | (p[1] << 5) | (p[2] << 10));
        }
        out_f[j] = fan_pack_h(ia, ic, static_cast<uint32_t>(k));
      }
      if (cycle_ok) {
        // Single directed cycle through all n positions, starting at position 0.
        uint8_t* cp = hm.cycpos.data() + hm.off[s];
        uint8_t* cr = hm.cycrot.data() + hm.off[s];
        int32_t p = 0, steps = 0;
        do {
          cp[steps] = static_cast<uint8_t>(p);
          cr[steps] = static_cast<uint8_t>(rot[p]);
          p = succ[p];
          ++steps;
        } while (p > 0 && steps < n);
        if (p == 0 && steps == n) hm.has_cycle[s] = 1;
      }
    }
  });
  if (broken >= 0) return "incident / neighbour lists disagree at vertex " + std::to_string(broken.load());

  pt.mark("rows, fans, cycles");
  // Full incident CSR (all vertices) for TwoPhase thresholds and vertex minima.
  hm.vinc_off.assign(nv + 1, 0);
  uint64_t it = 0;
  for (int64_t s = 0; s < nv; ++s) {
    hm.vinc_off[s] = static_cast<uint32_t>(it);
    const int64_t v = hm.order[s];
    it += static_cast<uint64_t>(d.inc_off[v + 1] - d.inc_off[v]);
    if (it >= 0xffffffffULL) return "incidence exceeds 2^32 entries";
  }
  hm.vinc_off[nv] = static_cast<uint32_t>(it);
  hm.vinc.resize(it);
  parallel_ranges(nv, [&](int64_t b, int64_t e) {
    for (int64_t s = b; s < e; ++s) {
      const int64_t v = hm.order[s];
      uint32_t* out = hm.vinc.data() + hm.vinc_off[s];
      int64_t j = 0;
      for (int64_t i = d.inc_off[v]; i < d.inc_off[v + 1]; ++i)
        out[j++] = static_cast<uint32_t>(tri_rank[d.inc[i]]);
      std::sort(out, out + j);
    }
  });

  pt.mark("incident CSR");
  hm.hubs.clear();
  hm.medium.clear();
  hm.large.clear();
  for (int64_t s = 0; s < nv; ++s) {
    if (deg[s] == 0) continue;
    const int tier = tiers.tier(deg[s]);
    if (tier == 1) hm.medium.push_back(static_cast<int32_t>(s));
    if (tier == 2) hm.hubs.push_back(static_cast<int32_t>(s));
    if (deg[s] > static_cast<uint32_t>(kMaxCycleDeg)) hm.large.push_back(static_cast<int32_t>(s));
  }
  pt.mark("tier lists");
  {
    const std::string terr = build_tiles(hm, deg, kMaxCycleDeg);
    if (!terr.empty()) return terr;
    std::vector<uint8_t>().swap(hm.cycpos);  // only build_tiles reads the cycles
    std::vector<uint8_t>().swap(hm.cycrot);
  }
  pt.mark("tiles");
  // Longest rows first: the warp tier's tail is its largest hubs.
  std::stable_sort(hm.large.begin(), hm.large.end(), [&](int32_t x, int32_t y) { return deg[x] > deg[y]; });
  return "";
}

std::string build_form_b(const HostMesh& hm, int32_t chunks, const Tiers& tiers, FormBSchedule& out) {
  const int64_t nv = hm.nv;
  if (chunks < 1) return "chunks must be >= 1";
  const int64_t k = (nv + chunks - 1) / chunks;  // worker_chunk: ceil(n / workers)
  out.chunks = chunks;
  out.nbr_fresh = hm.nbr;
  std::vector<int32_t> level(nv, -1);  // by ORIGINAL id
  int32_t nlev = 0;
  // Forward sweep in original id order: every dependency has a smaller id.
  for (int64_t v = 0; v < nv; ++v) {
    const int64_t s = hm.rank[v];
    const uint32_t o0 = hm.off[s], o1 = hm.off[s + 1];
    if (o0 == o1) continue;  // pinned
    int32_t L = 0;
    const int64_t cv = v / k;
    for (uint32_t j = o0; j < o1; ++j) {
      const uint32_t us = hm.nbr[j];
      const int64_t u = hm.order[us];
      if (u < v && u / k == cv) {
        out.nbr_fresh[j] |= 0x80000000u;
        if (level[u] >= 0) L = std::max(L, level[u] + 1);
      }
    }
    level[v] = L;
    nlev = std::max(nlev, L + 1);
  }
  // counts[t][L + 1]: vertices of tier t on level L, then prefix sums -> list offsets
  std::vector<int64_t> counts[3];
  for (auto& c : counts) c.assign(nlev + 1, 0);
  for (int64_t s = 0; s < nv; ++s) {
    const int32_t L = level[hm.order[s]];
    if (L >= 0) ++counts[tiers.tier(hm.off[s + 1] - hm.off[s])][L + 1];
  }
  for (auto& c : counts)
    for (int32_t L = 0; L < nlev; ++L) c[L + 1] += c[L];
  std::vector<int32_t>* lists[3] = {&out.nodes, &out.medium, &out.hubs};
  std::vector<int64_t> fill[3];
  for (int t = 0; t < 3; ++t) {
    lists[t]->assign(counts[t][nlev], 0);
    fill[t].assign(counts[t].begin(), counts[t].end() - 1);
  }
  for (int64_t s = 0; s < nv; ++s) {  // slot-ascending inside each level
    const int32_t L = level[hm.order[s]];
    if (L < 0) continue;
    const int t = tiers.tier(hm.off[s + 1] - hm.off[s]);
    (*lists[t])[fill[t][L]++] = static_cast<int32_t>(s);
  }
  {
    // Chunk schedule: counting sort of the movable vertices by (chunk, level); slot order
    // inside a level.
    const int64_t nchunks = (nv + k - 1) / k;
    std::vector<int32_t> chunk_levels(nchunks, 0);
    for (int64_t v = 0; v < nv; ++v)
      if (level[v] >= 0) chunk_levels[v / k] = std::max(chunk_levels[v / k], level[v] + 1);
    out.chunk_lvl.assign(nchunks + 1, 0);
    for (int64_t c = 0; c < nchunks; ++c) out.chunk_lvl[c + 1] = out.chunk_lvl[c] + chunk_levels[c];
    const int64_t total_lv = out.chunk_lvl[nchunks];
    std::vector<int64_t> cnt(total_lv + 1, 0);
    for (int64_t s = 0; s < nv; ++s) {
      const int64_t v = hm.order[s];
      if (level[v] >= 0) ++cnt[out.chunk_lvl[v / k] + level[v] + 1];
    }
    for (int64_t i = 0; i < total_lv; ++i) cnt[i + 1] += cnt[i];
    out.lvl_off.assign(cnt.begin(), cnt.end());
    out.cb_order.assign(cnt[total_lv], 0);
    std::vector<int64_t> fillp(cnt.begin(), cnt.end() - 1);
    for (int64_t s = 0; s < nv; ++s) {
      const int64_t v = hm.order[s];
      if (level[v] >= 0) out.cb_order[fillp[out.chunk_lvl[v / k] + level[v]]++] = static_cast<int32_t>(s);
    }
    out.cb_rec.assign(out.cb_order.size() * kChunkRecWords, 0);
    for (size_t p = 0; p < out.cb_order.size(); ++p) {
      const int64_t s = out.cb_order[p];
      const uint32_t o0 = hm.off[s], n = hm.off[s + 1] - o0;
      uint32_t* r = out.cb_rec.data() + p * kChunkRecWords;
      r[0] = static_cast<uint32_t>(s);
      r[1] = n;
      if (n <= static_cast<uint32_t>(kChunkRecMaxDeg))
        for (uint32_t j = 0; j < n; ++j) {
          r[2 + j] = out.nbr_fresh[o0 + j];
          r[2 + kChunkRecMaxDeg + j] = hm.fan[o0 + j];
        }
    }
    out.max_chunk_work = 0;
    for (int64_t c = 0; c < nchunks; ++c)
      out.max_chunk_work = std::max<int64_t>(out.max_chunk_work, cnt[out.chunk_lvl[c + 1]] - cnt[out.chunk_lvl[c]]);
  }
  {
    // Dataflow order: by level, slot-ascending inside a level (counting sort).
    std::vector<int64_t> cnt(nlev + 1, 0);
    for (int64_t s = 0; s < nv; ++s) {
      const int32_t L = level[hm.order[s]];
      if (L >= 0) ++cnt[L + 1];
    }
    for (int32_t L = 0; L < nlev; ++L) cnt[L + 1] += cnt[L];
    out.flow_rec.assign(static_cast<size_t>(cnt[nlev]) * kChunkRecWords, 0);
    for (int64_t s = 0; s < nv; ++s) {
      const int32_t L = level[hm.order[s]];
      if (L < 0) continue;
      uint32_t* r = out.flow_rec.data() + static_cast<size_t>(cnt[L]++) * kChunkRecWords;
      const uint32_t o0 = hm.off[s], n = hm.off[s + 1] - o0;
      r[0] = static_cast<uint32_t>(s);
      r[1] = n;
      if (n <= static_cast<uint32_t>(kChunkRecMaxDeg))
        for (uint32_t j = 0; j < n; ++j) {
          r[2 + j] = out.nbr_fresh[o0 + j];
          r[2 + kChunkRecMaxDeg + j] = hm.fan[o0 + j];
        }
    }
  }
  out.levels.resize(nlev);
  for (int32_t L = 0; L < nlev; ++L) {
    Phase& ph = out.levels[L];
    ph.small_begin = counts[0][L];
    ph.small_count = counts[0][L + 1] - counts[0][L];
    ph.medium_begin = counts[1][L];
    ph.medium_count = counts[1][L + 1] - counts[1][L];
    ph.hub_begin = counts[2][L];
    ph.hub_count = counts[2][L + 1] - counts[2][L];
  }
  return "";
}

}  // namespace tsg
