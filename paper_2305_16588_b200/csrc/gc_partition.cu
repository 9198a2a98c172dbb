// Inter-clique LDG partition (host preprocessing, native C++ in the library).
//
// Restates the reference's streaming linear-deterministic-greedy placement and its
// boundary refinement (src/partition.py:37-160) with identical results:
//   * adjacency = out-edges then in-edges per vertex, in-edges by (source, edge)
//     order (the stable argsort of _undirected_csr, partition.py:37-48);
//   * stream order = level-order BFS from the caller's root order (the device
//     permutation KeyedRng(seed).derive(0x5EED).permutation(n), partition.py:51-72),
//     each level the sorted set of unvisited neighbours;
//   * placement: score_p = count_p * (1 - size_p / capacity) in double, full parts
//     -inf; best score, then least loaded, then lowest index (partition.py:112-122);
//   * refinement passes over the sorted boundary of the pass start, sequential
//     cut-reducing moves, stop when a pass leaves the cut unchanged
//     (partition.py:124-152); a pass that raises the cut is GC_ERR_ASSERT.
// The greedy is one placement after another (each depends on the previous), so it
// stays on the host; the O(m) passes are linear scans over the CSR.

#include <algorithm>
#include <cmath>
#include <limits>
#include <vector>

#include "gc_common.cuh"

namespace {

struct Undirected {
    std::vector<uint64_t> off;
    std::vector<uint32_t> nbr;
};

Undirected undirected_csr(const uint64_t* ro, const uint32_t* ci, uint64_t n, uint64_t m) {
    Undirected u;
    u.off.assign(n + 1, 0);
    for (uint64_t v = 0; v < n; ++v) u.off[v + 1] += ro[v + 1] - ro[v];
    for (uint64_t e = 0; e < m; ++e) u.off[(uint64_t)ci[e] + 1] += 1;
    for (uint64_t v = 0; v < n; ++v) u.off[v + 1] += u.off[v];
    u.nbr.resize(2 * m);
    std::vector<uint64_t> cur(n);
    for (uint64_t v = 0; v < n; ++v) {
        const uint64_t d = ro[v + 1] - ro[v];
        std::copy(ci + ro[v], ci + ro[v + 1], u.nbr.begin() + u.off[v]);
        cur[v] = u.off[v] + d;
    }
    for (uint64_t s = 0; s < n; ++s)
        for (uint64_t e = ro[s]; e < ro[s + 1]; ++e) u.nbr[cur[ci[e]]++] = (uint32_t)s;
    return u;
}

std::vector<uint32_t> bfs_order(const Undirected& g, uint64_t n, const int64_t* roots) {
    std::vector<uint8_t> seen(n, 0);
    std::vector<uint32_t> out;
    out.reserve(n);
    std::vector<uint32_t> frontier, next;
    for (uint64_t r = 0; r < n; ++r) {
        const uint32_t root = (uint32_t)roots[r];
        if (seen[root]) continue;
        seen[root] = 1;
        frontier.assign(1, root);
        while (!frontier.empty()) {
            out.insert(out.end(), frontier.begin(), frontier.end());
            next.clear();
            for (uint32_t v : frontier)
                for (uint64_t k = g.off[v]; k < g.off[v + 1]; ++k) {
                    const uint32_t w = g.nbr[k];
                    if (!seen[w]) {
                        seen[w] = 1;
                        next.push_back(w);
                    }
                }
            std::sort(next.begin(), next.end());
            frontier.swap(next);
        }
    }
    return out;
}

uint64_t cut_count(const uint64_t* ro, const uint32_t* ci, uint64_t n, const int32_t* a) {
    uint64_t cut = 0;
    for (uint64_t v = 0; v < n; ++v)
        for (uint64_t e = ro[v]; e < ro[v + 1]; ++e) cut += a[v] != a[ci[e]];
    return cut;
}

void refine_pass(const Undirected& g, const uint64_t* ro, const uint32_t* ci, uint64_t n, int32_t* a,
                 std::vector<int64_t>& sizes, int64_t capacity, uint32_t k) {
    std::vector<uint8_t> boundary(n, 0);
    for (uint64_t v = 0; v < n; ++v)
        for (uint64_t e = ro[v]; e < ro[v + 1]; ++e)
            if (a[v] != a[ci[e]]) boundary[v] = boundary[ci[e]] = 1;
    std::vector<int64_t> cnt(k), gain(k);
    for (uint64_t v = 0; v < n; ++v) {
        if (!boundary[v]) continue;
        std::fill(cnt.begin(), cnt.end(), 0);
        bool any = false;
        for (uint64_t e = g.off[v]; e < g.off[v + 1]; ++e) {
            const uint32_t w = g.nbr[e];
            if (w == v) continue;
            ++cnt[a[w]];
            any = true;
        }
        if (!any) continue;
        const int32_t current = a[v];
        uint32_t target = 0;
        for (uint32_t p = 0; p < k; ++p) {
            gain[p] = sizes[p] >= capacity ? -1 : cnt[p] - cnt[current];
            if (p == (uint32_t)current) gain[p] = 0;
            if (gain[p] > gain[target]) target = p;
        }
        if (gain[target] > 0) {
            a[v] = (int32_t)target;
            sizes[current] -= 1;
            sizes[target] += 1;
        }
    }
}

}  // namespace

extern "C" {

int gc_partition_ldg(const uint64_t* h_row_offsets, const uint32_t* h_cols, uint64_t num_vertices,
                     uint64_t num_edges, const int64_t* h_root_order, uint32_t num_parts, int64_t capacity,
                     int refine_passes, int32_t* h_assignment, uint64_t* h_cuts) {
    GC_REQUIRE(num_parts >= 1, GC_ERR_VALUE, "gc_partition_ldg: num_parts must be >= 1");
    GC_REQUIRE(num_parts <= num_vertices, GC_ERR_VALUE, "gc_partition_ldg: num_parts exceeds num_vertices");
    GC_REQUIRE(num_vertices < (1ull << 32), GC_ERR_VALUE, "gc_partition_ldg: at most 2^32 - 1 vertices");
    GC_REQUIRE(capacity >= 1 && (uint64_t)capacity * num_parts >= num_vertices, GC_ERR_VALUE,
               "gc_partition_ldg: capacity * num_parts must cover every vertex");
    GC_REQUIRE(h_row_offsets && h_assignment && (num_vertices == 0 || h_root_order), GC_ERR_VALUE,
               "gc_partition_ldg: null array");
    const uint64_t n = num_vertices;
    const uint32_t k = num_parts;
    {
        std::vector<uint8_t> hit(n, 0);
        for (uint64_t v = 0; v < n; ++v) {
            const int64_t r = h_root_order[v];
            GC_REQUIRE(r >= 0 && (uint64_t)r < n && !hit[r], GC_ERR_VALUE,
                       "gc_partition_ldg: root order is not a permutation of the vertices");
            hit[r] = 1;
        }
    }
    const Undirected g = undirected_csr(h_row_offsets, h_cols, n, num_edges);
    const std::vector<uint32_t> order = bfs_order(g, n, h_root_order);

    std::fill(h_assignment, h_assignment + n, -1);
    std::vector<int64_t> sizes(k, 0), cnt(k, 0);
    const double cap = (double)capacity;
    for (uint32_t v : order) {
        std::fill(cnt.begin(), cnt.end(), 0);
        for (uint64_t e = g.off[v]; e < g.off[v + 1]; ++e) {
            const uint32_t w = g.nbr[e];
            if (w != v && h_assignment[w] >= 0) ++cnt[h_assignment[w]];
        }
        uint32_t best = 0;
        double best_score = 0.0;
        for (uint32_t p = 0; p < k; ++p) {
            const double score = sizes[p] >= capacity ? -std::numeric_limits<double>::infinity()
                                                      : (double)cnt[p] * (1.0 - (double)sizes[p] / cap);
            if (p == 0 || score > best_score || (score == best_score && sizes[p] < sizes[best])) {
                best = p;
                best_score = score;
            }
        }
        h_assignment[v] = (int32_t)best;
        sizes[best] += 1;
    }

    for (int pass = 0; pass < refine_passes; ++pass) {
        const uint64_t before = cut_count(h_row_offsets, h_cols, n, h_assignment);
        refine_pass(g, h_row_offsets, h_cols, n, h_assignment, sizes, capacity, k);
        const uint64_t after = cut_count(h_row_offsets, h_cols, n, h_assignment);
        if (h_cuts) {
            h_cuts[2 * pass] = before;
            h_cuts[2 * pass + 1] = after;
        }
        GC_REQUIRE(after <= before, GC_ERR_ASSERT, "refinement pass increased the edge cut");
        if (after == before) break;
    }
    return GC_OK;
}

}  // extern "C"
