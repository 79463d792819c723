// trismooth adjacency and constraints — drop-in public API of
// proj/include/trismooth/topology.hpp.  Host mesh prep for the B200 engine: the unique
// neighbour rows (ascending) and incident rows built here are what libtsg converts into its
// slot-ordered device arrays.
#pragma once

#include <vector>

#include "trismooth/mesh.hpp"

namespace trismooth {

class ThreadPool;

/// raw: two entries per incidence in triangle-visit order (duplicates kept);
/// unique: sorted, deduplicated, with per-entry occurrence counts in `multiplicity`;
/// incident: triangle ids, ascending.
struct Adjacency {
  Csr raw;
  Csr unique;
  std::vector<int> multiplicity;
  Csr incident;
};

/// Builds the adjacency and installs unique neighbours + incident triangles in the mesh.
/// Output is identical to the reference's single-threaded build (the raw recording order is
/// part of the contract); large meshes are processed in parallel per vertex range.
Adjacency find_neighbors(Mesh& mesh);

/// Pins a vertex when it has no neighbours or any neighbour occurs other than twice.
void determine_constraints(Mesh& mesh, const Adjacency& adj, ThreadPool* pool = nullptr);

/// Independent check: boundary iff on an edge used by exactly one triangle.
std::vector<bool> boundary_oracle(const Mesh& mesh);

/// Undirected edges used by three or more triangles.
int non_manifold_edge_count(const Mesh& mesh);

}  // namespace trismooth
