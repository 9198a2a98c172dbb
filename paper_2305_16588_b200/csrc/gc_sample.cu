// K2 hop_expand: one hop of the reference's L-hop sampler (_expand_frontier,
// sampling.py:84-117) for a window of W independent mini-batches in one launch.
//
// Per CTA tile of up to 256 frontier positions (tile ids claimed from a counter):
//   phase 1  thread-per-position: v, row offsets, deg, take = min(deg, fanout);
//            presampling counters (warp-aggregated), seed marking; CTA scan of take;
//            the tile aggregate is published for the decoupled look-back.
//   phase 2a selection into a shared-memory list of source edge indices (copy path:
//            CSR order; choice path: the `fanout` smallest (hash_pairs(i, j), j) in
//            ascending order — bit-exact with the lexsort at sampling.py:108-114 and
//            the scalar oracle tests/helpers.py:95-110) — thread-per-position sorted
//            networks for short lists, warp-per-position extraction otherwise.
//   look-back exclusive prefix of the batch's output (after phase 2a, so the
//            predecessor tiles have normally finished).
//   phase 2b flat, coalesced emission: out[prefix + k] = col[src_edge[k]], marking the
//            batch's visited bitmap for dedup (K3).
// Keys depend only on (position, edge index), never on neighbour ids (rng.py:68-72),
// so only the `take` selected column entries are read from the topology.
#include <type_traits>

#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>

#include "gc_common.cuh"

namespace gc {

#ifndef GC_HOP_THREADS
#define GC_HOP_THREADS 256  // 128 measured 2% slower at C2 hop 3
#endif
constexpr int kHopThreads = GC_HOP_THREADS;  // CTA threads; a tile is kTilePos x PPT frontier positions
constexpr int kTilePos = kHopThreads;
// staged output items per round: 24 KB of u32 edge indices (plain CSR) or 40 KB of
// u64 (tiered), so a 512-position tile of fanout 10 stages in one round
__host__ __device__ constexpr int item_cap(bool tiered) { return tiered ? 20 * kHopThreads : 24 * kHopThreads; }
// emission items in flight per thread: a full tile of 256 positions with take =
// fanout stages exactly `fanout` items per thread, so for the small networks S - 1
// (the largest fanout of the network) covers it in one pass (C2 hop 3: 1.68 -> 1.60
// ms); S = 11 (fanouts 8-10) takes two passes of 5 (C2 hop 2: 0.246 -> 0.235 ms);
// wider fanouts keep 4 (measured faster than 8-12 for S = 16)
template <int S>
__host__ __device__ constexpr int emit_items() {
    return S > 1 && S <= 8 ? S - 1 : (S == 11 ? 5 : 4);
}
// resident CTAs per SM the register budget targets: 6 (40 registers, no spills) for
// S <= 8, 5 up to S = 16 (C3 hop 2, S = 11: 15.0 ms at 5 vs 16.1 at 6), 4 (64 registers) above and for the
// generic kernel (measured: C2 hop 3 1.73 -> 1.68 ms; C3 hop 1, fanout 25, was at one
// CTA per SM with 181 registers)
#ifndef GC_HOP_MIN_BLOCKS
#define GC_HOP_MIN_BLOCKS 6
#endif
constexpr int kHopMinBlocks = GC_HOP_MIN_BLOCKS;
#ifndef GC_HOP_PPT
#define GC_HOP_PPT 2  // frontier positions per thread of the small-network kernels
#endif
template <int S>
constexpr int hop_min_blocks() {
    return (S > 0 && S <= 8 ? kHopMinBlocks : (S > 0 && S <= 16 ? 5 : 4)) * 256 / kHopThreads;
}

constexpr int kTierShift = 56;  // staged edge index = (tier code << 56) | edge within that tier's CSR
constexpr uint64_t kEdgeMask = (1ull << kTierShift) - 1;

struct HopParams {
    const uint64_t* ro;
    const uint32_t* ci;
    uint64_t n;
    const uint32_t* loc;
    const uint64_t* soff[GC_MAX_PEERS];
    const uint32_t* scols[GC_MAX_PEERS];
    uint32_t self_rank;
    uint32_t full_on_host;
    uint64_t* tier_reads;
    const uint32_t* frontier;
    uint64_t fstride;
    const uint32_t* fcount;
    uint32_t fanout;
    uint32_t tiles_per_batch;
    uint32_t tile_pos;
    const uint64_t* hop_keys;
    uint32_t* out_off;
    uint64_t ostride;
    uint32_t* out_nbrs;
    uint64_t nstride;
    uint32_t* out_count;
    uint32_t* bitmap;
    uint64_t bwords;
    uint32_t* summary;
    uint64_t swords;
    int mark_frontier;
    uint64_t* topo_reads;
    uint64_t* edge_trav;
    uint64_t* txn_total;
    uint32_t cls;
    uint32_t u32b;
    uint64_t* tile_state;
    uint32_t* tile_counter;  // [num_batches]: batch b's tile ids are claimed from [b] in dispatch order (zeroed per launch)
    int exact_only;  // test hook: always take the 64-bit extraction path
    uint32_t k32;    // == 32, opaque to the compiler (see PairHashHigh::hi_counter)
};

static int g_exact_only = 0;

// Staged output items: u64 edge indices (tier code in bits 56..63 when TIERED), or u32
// edge indices for the plain CSR (m < 2^32), which halves the staging traffic.
template <typename Item>
__device__ __forceinline__ void stage(Item* s_items, uint32_t item, uint32_t r0, uint32_t r1, uint64_t edge) {
    if (item >= r0 && item < r1) s_items[item - r0] = (Item)edge;
}

// Exact winner among lanes in `cand` by (lo32 of key, edge index) once the high
// words tie; all lanes return the same winning edge index.
__device__ __forceinline__ uint32_t tie_break(unsigned cand, uint64_t key, uint32_t j) {
    const int lane = threadIdx.x & 31;
    bool in = (cand >> lane) & 1u;
    uint32_t lo = in ? (uint32_t)key : 0xFFFFFFFFu;
    uint32_t jj = in ? j : 0xFFFFFFFFu;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        uint32_t olo = __shfl_xor_sync(kFull, lo, o);
        uint32_t oj = __shfl_xor_sync(kFull, jj, o);
        if (olo < lo || (olo == lo && oj < jj)) {
            lo = olo;
            jj = oj;
        }
    }
    return jj;
}

// Choice path with every candidate key resident in registers: lane l holds edges
// j = l + 32 r for r < R. Extracts the first min(fanout, needed) minima in order.
template <int R, typename Item>
__device__ __forceinline__ void select_registers(uint64_t hc, uint32_t deg, uint32_t fanout, uint64_t o0,
                                                 uint32_t excl, uint32_t r0, uint32_t r1, Item* s_items) {
    const int lane = threadIdx.x & 31;
    uint64_t key[R];
    uint32_t rank[R];
    unsigned live = 0;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const uint32_t j = lane + 32 * r;
        key[r] = hash_pair(hc, j);
        rank[r] = 0xFFFFFFFFu;
        if (j < deg) live |= 1u << r;
    }
    // lane-local minimum among live candidates (j ascending with r: strict < keeps the
    // smaller edge index on equal keys)
    auto local_min = [&](uint64_t& lm, int& lr) {
        lm = ~0ull;
        lr = -1;
#pragma unroll
        for (int r = 0; r < R; ++r)
            if (((live >> r) & 1u) && (lr < 0 || key[r] < lm)) {
                lm = key[r];
                lr = r;
            }
    };
    uint64_t lm;
    int lr;
    local_min(lm, lr);
    // extraction beyond the staged window is not needed
    const uint32_t stop = min(fanout, r1 - excl);
    for (uint32_t it = 0; it < stop; ++it) {
        const uint32_t hi = lr >= 0 ? (uint32_t)(lm >> 32) : 0xFFFFFFFFu;
        const uint32_t m = __reduce_min_sync(kFull, hi);
        bool win = lr >= 0 && hi == m;
        const unsigned cand = __ballot_sync(kFull, win);
        if (cand & (cand - 1u)) {
            // several lanes share the high word: exact (lo32, j) order decides (rare)
            const uint32_t wj = tie_break(cand, lm, lane + 32u * (uint32_t)(lr < 0 ? 0 : lr));
            win = (wj & 31u) == (uint32_t)lane;
        }
        if (win) {
#pragma unroll
            for (int r = 0; r < R; ++r)
                if (r == lr) rank[r] = it;
            live &= ~(1u << lr);
            if (R == 1)
                lr = -1;
            else
                local_min(lm, lr);
        }
    }
    // each lane stages its own winners: item excl + rank <- edge o0 + j
#pragma unroll
    for (int r = 0; r < R; ++r)
        if (rank[r] != 0xFFFFFFFFu) stage(s_items, excl + rank[r], r0, r1, o0 + (uint64_t)(lane + 32 * r));
}

// Fast choice path: candidate j of lane l is j = l + 32 r (r < R). Each key is
// packed into 32 bits as (top 32-IB bits of the 64-bit key) << IB | j, which makes
// every packed value unique, so one REDUX.MIN per extraction names the winner with
// no ballot. The packed order equals the exact (key, j) order unless two
// candidates share the packed prefix; such a prefix tie shows up as two equal
// prefixes among consecutively extracted values (one extra extraction covers the
// selection boundary), in which case this returns false and the caller reruns the
// exact 64-bit path. Ties need two of <=128 uniform keys to agree in 25-27 bits.
template <int R, typename Item>
__device__ __forceinline__ bool select_packed(uint64_t hc, uint32_t deg, uint32_t fanout, uint64_t o0, uint32_t excl,
                                              uint32_t r0, uint32_t r1, Item* s_items) {
    constexpr int IB = R == 1 ? 5 : (R == 2 ? 6 : 7);
    constexpr uint32_t kIdx = (1u << IB) - 1u;
    const uint32_t lane = threadIdx.x & 31;
    uint32_t pk[R];
    uint32_t rank[R];
    const PairHashHigh hh(hc);  // j < 128: only key bits >= 37 are used
#pragma unroll
    for (int r = 0; r < R; ++r) {
        const uint32_t j = lane + 32u * r;
        pk[r] = j < deg ? (hh.hi(j) & ~kIdx) | j : 0xFFFFFFFFu;
        rank[r] = 0xFFFFFFFFu;
    }
    uint32_t lmin = pk[0];
#pragma unroll
    for (int r = 1; r < R; ++r) lmin = min(lmin, pk[r]);
    const uint32_t stop = min(fanout, r1 - excl);  // stop < deg here
    uint32_t prev = 0xFFFFFFFFu;
    bool tie = false;
    for (uint32_t it = 0; it <= stop; ++it) {
        const uint32_t m = __reduce_min_sync(kFull, lmin);
        const uint32_t hi = m >> IB;
        tie |= (it != 0) & (hi == prev);
        prev = hi;
        if (it < stop && lane == (m & 31u)) {
            const uint32_t wr = (m & kIdx) >> 5;
#pragma unroll
            for (int r = 0; r < R; ++r)
                if (r == (int)wr) {
                    rank[r] = it;
                    pk[r] = 0xFFFFFFFFu;
                }
            lmin = pk[0];
#pragma unroll
            for (int r = 1; r < R; ++r) lmin = min(lmin, pk[r]);
        }
    }
    if (tie) return false;
#pragma unroll
    for (int r = 0; r < R; ++r)
        if (rank[r] != 0xFFFFFFFFu) stage(s_items, excl + rank[r], r0, r1, o0 + (uint64_t)(lane + 32u * r));
    return true;
}

// Choice path for long adjacency lists: keys are recomputed each extraction step
// above the last emitted (key, j), so any degree is handled exactly.
template <typename Item>
__device__ void select_streaming(uint64_t hc, uint32_t deg, uint32_t fanout, uint64_t o0, uint32_t excl, uint32_t r0,
                                 uint32_t r1, Item* s_items) {
    const int lane = threadIdx.x & 31;
    uint64_t lk = 0;
    uint32_t lj = 0;
    bool have_last = false;
    uint32_t stop = min(fanout, r1 - excl);
    for (uint32_t it = 0; it < stop; ++it) {
        uint64_t bk = ~0ull;
        uint32_t bj = 0xFFFFFFFFu;
        for (uint32_t j = lane; j < deg; j += 32) {
            uint64_t k = hash_pair(hc, j);
            if (have_last && (k < lk || (k == lk && j <= lj))) continue;
            if (bj == 0xFFFFFFFFu || k < bk) {
                bk = k;
                bj = j;
            }
        }
        // warp argmin over (key, j)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            uint64_t ok = __shfl_xor_sync(kFull, bk, o);
            uint32_t oj = __shfl_xor_sync(kFull, bj, o);
            if (oj != 0xFFFFFFFFu && (bj == 0xFFFFFFFFu || ok < bk || (ok == bk && oj < bj))) {
                bk = ok;
                bj = oj;
            }
        }
        if (lane == 0) stage(s_items, excl + it, r0, r1, o0 + bj);
        lk = bk;
        lj = bj;
        have_last = true;
    }
}

// Thread-per-position choice path for deg <= 64 and fanout < S: the thread streams
// its deg keys through a branchless S-slot min/max insertion network on packed
// 32-bit values (25-bit key prefix << 7 | c, c = (G & 0xFF) + j the hash counter),
// which keeps the S smallest in order. Two equal prefixes among ranks 0..fanout mean
// the packed order may differ from the exact (key, j) order: return false and let a
// warp redo the position exactly. deg > fanout >= TRI - 1, so the first TRI
// candidates are inserted with the network peeled: slots still holding +inf fold away.
template <int S>
__device__ __forceinline__ void insert_slot(uint32_t (&t)[S], uint32_t x) {
#pragma unroll
    for (int s = S - 1; s >= 1; --s) t[s] = max(t[s - 1], min(t[s], x));
    t[0] = min(t[0], x);
}

// Two candidates at once: with a < b, the k-th smallest of t U {a, b} is
// min(t[k], max(t[k-1], a), max(t[k-2], b)) — a three-input VIMNMX3 plus two maxes
// per slot for two candidates, against two ops per slot per candidate one at a time.
template <int S>
__device__ __forceinline__ void insert_pair(uint32_t (&t)[S], uint32_t x, uint32_t y) {
    const uint32_t a = min(x, y), b = max(x, y);
#pragma unroll
    for (int s = S - 1; s >= 2; --s) t[s] = min(min(t[s], max(t[s - 1], a)), max(t[s - 2], b));
    if (S > 1) t[1] = min(min(t[1], max(t[0], a)), b);
    t[0] = min(t[0], a);
}

template <int S>
__host__ __device__ constexpr int peeled_candidates() {
    return S == 4 ? 2 : S == 6 ? 5 : S == 8 ? 7 : S == 11 ? 9 : S == 16 ? 12 : S == 21 ? 17 : S == 26 ? 22 : 27;
}

// Packed key of hash counter c: (key[63:39] << 7) | c
__device__ __forceinline__ uint32_t packed_key(const PairHashHigh& hh, uint32_t c, uint32_t k32) {
    return (hh.hi_counter(c, k32) & ~127u) | c;
}

// The remaining candidates [c, cend) of one position, in pairs
template <int S>
__device__ __forceinline__ void fill_tail(uint32_t (&t)[S], const PairHashHigh& hh, uint32_t c, uint32_t cend,
                                          uint32_t k32) {
#pragma unroll 2
    for (; c + 1 < cend; c += 2) insert_pair<S>(t, packed_key(hh, c, k32), packed_key(hh, c + 1, k32));
    if (c < cend) insert_slot<S>(t, packed_key(hh, c, k32));
}

// Ties and staging of a filled network. CHECKED = false: the tile stages in one round
// (r0 = 0, every item in range), so the per-item window test is dropped.
template <int S, bool CHECKED, typename Item>
__device__ __forceinline__ bool stage_network(const uint32_t (&t)[S], uint32_t fanout, uint64_t o0, uint32_t excl,
                                              uint32_t r0, uint32_t r1, Item* s_items) {
    constexpr int IB = 7;
    const uint64_t base = o0 - kGoldenLow;
    if (!CHECKED && fanout == S - 1) {
        // the widest fanout of the network (C2 hop 3: 5 of S = 6): every slot is
        // checked and staged without per-slot predicates, from one base address
        bool tie = false;
#pragma unroll
        for (int s = 0; s + 1 < S; ++s) tie |= (t[s] >> IB) == (t[s + 1] >> IB);
        if (tie) return false;
        Item* const out = s_items + excl;
#pragma unroll
        for (int s = 0; s + 1 < S; ++s) out[s] = (Item)(base + (t[s] & ((1u << IB) - 1u)));
        return true;
    }
    bool tie = false;
#pragma unroll
    for (int s = 0; s + 1 < S; ++s) tie |= (s < (int)fanout) & ((t[s] >> IB) == (t[s + 1] >> IB));
    if (tie) return false;
#pragma unroll
    for (int s = 0; s < S; ++s)
        if (s < (int)fanout) {
            const uint64_t e = base + (t[s] & ((1u << IB) - 1u));
            if (CHECKED)
                stage(s_items, excl + s, r0, r1, e);
            else
                s_items[excl + s] = (Item)e;
        }
    return true;
}

// Thread-per-position choice path for deg <= 64 and fanout < S: the thread streams
// its deg keys through a branchless S-slot min/max insertion network on packed
// 32-bit values (25-bit key prefix << 7 | c, c = (G & 0xFF) + j the hash counter),
// which keeps the S smallest in order. Two equal prefixes among ranks 0..fanout mean
// the packed order may differ from the exact (key, j) order: return false and let a
// warp redo the position exactly. deg > fanout >= TRI - 1, so the first TRI
// candidates are inserted with the network peeled: slots still holding +inf fold away.
template <int S, bool CHECKED, typename Item>
__device__ __forceinline__ bool select_thread(uint64_t hc, uint32_t deg, uint32_t fanout, uint64_t o0, uint32_t excl,
                                              uint32_t r0, uint32_t r1, Item* s_items, uint32_t k32) {
    constexpr int TRI = peeled_candidates<S>() & ~1;  // peeled in pairs
    uint32_t t[S];
#pragma unroll
    for (int s = 0; s < S; ++s) t[s] = 0xFFFFFFFFu;
    const PairHashHigh hh(hc);  // deg <= 64: key bits 63..38 from the specialised hash
#pragma unroll
    for (int j = 0; j < TRI; j += 2) {
        const uint32_t c = kGoldenLow + j;
        insert_pair<S>(t, packed_key(hh, c, k32), packed_key(hh, c + 1, k32));
    }
    fill_tail<S>(t, hh, kGoldenLow + TRI, kGoldenLow + deg, k32);
    return stage_network<S, CHECKED>(t, fanout, o0, excl, r0, r1, s_items);
}

// Two positions of one thread through their networks together (PPT = 2, both on the
// thread path, one staging round): the candidates both have go through one loop whose
// body holds two independent insertion chains, so the scheduler has twice the
// independent work per warp; the longer list finishes alone.
template <int S, typename Item>
__device__ __forceinline__ void select_thread_two(const uint64_t (&hc)[2], const uint32_t (&deg)[2],
                                                  const uint64_t (&o0)[2], const uint32_t (&excl)[2], uint32_t fanout,
                                                  Item* s_items, uint32_t k32, bool (&need_warp)[2]) {
    constexpr int TRI = peeled_candidates<S>() & ~1;
    uint32_t ta[S], tb[S];
#pragma unroll
    for (int s = 0; s < S; ++s) ta[s] = tb[s] = 0xFFFFFFFFu;
    const PairHashHigh ha(hc[0]), hb(hc[1]);
#pragma unroll
    for (int j = 0; j < TRI; j += 2) {
        const uint32_t c = kGoldenLow + j;
        insert_pair<S>(ta, packed_key(ha, c, k32), packed_key(ha, c + 1, k32));
        insert_pair<S>(tb, packed_key(hb, c, k32), packed_key(hb, c + 1, k32));
    }
    const uint32_t cboth = kGoldenLow + min(deg[0], deg[1]);
    uint32_t c = kGoldenLow + TRI;
    for (; c + 1 < cboth; c += 2) {
        insert_pair<S>(ta, packed_key(ha, c, k32), packed_key(ha, c + 1, k32));
        insert_pair<S>(tb, packed_key(hb, c, k32), packed_key(hb, c + 1, k32));
    }
    fill_tail<S>(ta, ha, c, kGoldenLow + deg[0], k32);
    fill_tail<S>(tb, hb, c, kGoldenLow + deg[1], k32);
    need_warp[0] = !stage_network<S, false>(ta, fanout, o0[0], excl[0], 0u, 0u, s_items);
    need_warp[1] = !stage_network<S, false>(tb, fanout, o0[1], excl[1], 0u, 0u, s_items);
}

// Warp-cooperative selection of one position (long lists, wide fanouts, tie redo).
template <typename Item>
__device__ __forceinline__ void select_warp(uint64_t hc, uint32_t d, uint32_t fanout, uint64_t base, uint32_t e0,
                                            uint32_t r0, uint32_t r1, Item* s_items, bool exact) {
    if (exact && d <= 128) {
        if (d <= 32)
            select_registers<1>(hc, d, fanout, base, e0, r0, r1, s_items);
        else if (d <= 64)
            select_registers<2>(hc, d, fanout, base, e0, r0, r1, s_items);
        else
            select_registers<4>(hc, d, fanout, base, e0, r0, r1, s_items);
    } else if (d <= 32) {
        if (!select_packed<1>(hc, d, fanout, base, e0, r0, r1, s_items))
            select_registers<1>(hc, d, fanout, base, e0, r0, r1, s_items);
    } else if (d <= 64) {
        if (!select_packed<2>(hc, d, fanout, base, e0, r0, r1, s_items))
            select_registers<2>(hc, d, fanout, base, e0, r0, r1, s_items);
    } else if (d <= 128) {
        if (!select_packed<4>(hc, d, fanout, base, e0, r0, r1, s_items))
            select_registers<4>(hc, d, fanout, base, e0, r0, r1, s_items);
    } else {
        select_streaming(hc, d, fanout, base, e0, r0, r1, s_items);
    }
}

// Emission of one group of K staged items per thread (item q at items[q * kHopThreads]):
// column loads, then visited-word loads, then streaming stores and the (rare) atomics,
// so the dependent-load chains of the K items overlap. FULL: all K are in range, so
// there are no per-item predicates and every address is one base plus an immediate.
template <int K, bool FULL, bool TIERED, typename Item>
__device__ __forceinline__ void emit_group(const Item* items, uint32_t left, uint32_t* dst, const HopParams& p,
                                           uint32_t* bm, uint32_t* sm) {
    const uint32_t* __restrict__ ci = p.ci;
    uint32_t u[K];
#pragma unroll
    for (int q = 0; q < K; ++q) {
        u[q] = 0;
        if (FULL || q * kHopThreads < left) {
            const uint64_t it = items[q * kHopThreads];  // u32 items widen for the plain CSR
            if (TIERED) {
                const uint32_t code = (uint32_t)(it >> kTierShift);
                const uint32_t* cols = code ? p.scols[code - 1] : ci;
                u[q] = __ldg(cols + (it & kEdgeMask));
            } else {
                u[q] = __ldg(ci + it);
            }
        }
    }
    if (bm == nullptr) {
#pragma unroll
        for (int q = 0; q < K; ++q)
            if (FULL || q * kHopThreads < left) __stcs(dst + q * kHopThreads, u[q]);
        return;
    }
    uint32_t w[K];
#pragma unroll
    for (int q = 0; q < K; ++q) w[q] = (FULL || q * kHopThreads < left) ? bm[u[q] >> 5] : ~0u;
#pragma unroll
    for (int q = 0; q < K; ++q)
        if (FULL || q * kHopThreads < left) __stcs(dst + q * kHopThreads, u[q]);
    if (sm == nullptr) {
#pragma unroll
        for (int q = 0; q < K; ++q)
            if (!((w[q] >> (u[q] & 31)) & 1u)) atomicOr(bm + (u[q] >> 5), 1u << (u[q] & 31));
    } else {
#pragma unroll
        for (int q = 0; q < K; ++q)
            if (!((w[q] >> (u[q] & 31)) & 1u)) mark_visited_unchecked(bm, sm, u[q]);
    }
}

// TIERED: the topology has a location table or lives in host memory, so rows resolve
// through the tier rule and staged edges carry a slab code; otherwise the plain CSR.
// PPT frontier positions per thread (blocked: thread i owns positions PPT*i ..
// PPT*i + PPT-1 of the tile). PPT = 2 for the small networks: phase 1's chain of
// dependent loads (tile claim -> frontier -> row offsets) and the per-tile work (scan,
// look-back, uniform setup) are then paid once per 512 positions instead of 256.
template <int S, bool TIERED, int PPT>
__global__ void __launch_bounds__(kHopThreads, hop_min_blocks<S>()) k_hop_expand(HopParams p) {
    using Scan = cub::BlockScan<uint32_t, kHopThreads>;
    using Reduce = cub::BlockReduce<uint64_t, kHopThreads>;
    __shared__ union {
        typename Scan::TempStorage scan;
        typename Reduce::TempStorage reduce;
    } tmp;
    using Item = typename std::conditional<TIERED, uint64_t, uint32_t>::type;
    constexpr uint32_t kCap = item_cap(TIERED);
    __shared__ Item s_items[kCap];
    __shared__ uint64_t s_prefix;
    __shared__ uint32_t s_vid;
    __shared__ uint32_t s_arrive;  // warps done with phase 2a (the first runs the look-back)

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    // grid = (tiles per batch, batches). The tile id within batch b is claimed from the
    // batch's counter, not blockIdx.x: a tile only starts after every lower tile of its
    // batch has been handed to a running CTA, so each predecessor its look-back waits on
    // is resident or done whatever order the hardware dispatches CTAs in
    const uint32_t b = blockIdx.y;
    if (tid == 0) {
        s_vid = atomicAdd(p.tile_counter + b, 1u);
        s_arrive = 0;
    }
    // batch-uniform loads overlap the claim's round trip
    const uint32_t F = p.fcount[b];
    const uint64_t hkey = p.hop_keys[b];
    __syncthreads();
    const uint32_t t = s_vid;
    const uint64_t p0 = (uint64_t)t * p.tile_pos;
    if (p0 >= F && t != 0) return;  // past the end of this batch's frontier: no successor needs it
    const uint32_t npos = p0 < F ? (uint32_t)((F - p0) < (uint64_t)p.tile_pos ? (F - p0) : (uint64_t)p.tile_pos) : 0u;

    // ---- phase 1: per position degree, take and position hash
    bool valid[PPT];
    uint32_t v[PPT], deg[PPT], take[PPT];
    uint64_t o0[PPT], hc[PPT];
    int tier[PPT];  // 0 local, 1 peer slab, 2 host; the full CSR is local unless it lives in host memory
    const uint32_t* fr = p.frontier + b * p.fstride + p0 + (uint32_t)tid * PPT;
#pragma unroll
    for (int q = 0; q < PPT; ++q) {
        valid[q] = (uint32_t)tid * PPT + q < npos;
        v[q] = valid[q] ? fr[q] : 0u;
        deg[q] = 0;
        take[q] = 0;
        o0[q] = 0;
        hc[q] = 0;
        tier[q] = TIERED ? 2 : 0;
    }
#pragma unroll
    for (int q = 0; q < PPT; ++q) {
        if (valid[q]) {
            if (!TIERED && v[q] < p.n) {
                o0[q] = p.ro[v[q]];
                deg[q] = (uint32_t)(p.ro[v[q] + 1] - o0[q]);
            } else if (v[q] < p.n) {
                const uint32_t L = p.loc ? __ldg(p.loc + v[q]) : GC_TIER_HOST;
                if (L == GC_TIER_HOST) {
                    o0[q] = p.ro[v[q]];
                    deg[q] = (uint32_t)(p.ro[v[q] + 1] - o0[q]);
                } else {
                    const uint32_t g = L >> 28, slot = L & 0x0FFFFFFFu;
                    const uint64_t* so = p.soff[g];
                    o0[q] = so[slot];
                    deg[q] = (uint32_t)(so[slot + 1] - o0[q]);
                    o0[q] |= (uint64_t)(g + 1) << kTierShift;  // tag: read the columns from slab g
                    tier[q] = g == p.self_rank ? 0 : 1;
                }
            }
        }
    }
#pragma unroll
    for (int q = 0; q < PPT; ++q) {
        if (valid[q]) {
            take[q] = min(deg[q], p.fanout);
            if (p.mark_frontier && p.bitmap && v[q] < p.n)
                mark_visited(p.bitmap + b * p.bwords, p.summary ? p.summary + b * p.swords : nullptr, v[q]);
            // hash_counters(position), position = index in this batch's frontier (rng.py:64-66)
            if (deg[q] > p.fanout) hc[q] = hash_counter(hkey, p0 + (uint32_t)tid * PPT + q);
        }
    }
    if (p.topo_reads || p.edge_trav) {
#pragma unroll
        for (int q = 0; q < PPT; ++q) {
            // ids outside [0, n) are rejected on the host; never let one index a counter
            const bool counted = valid[q] && v[q] < p.n;
            unsigned act = __ballot_sync(kFull, counted);
            if (counted) {
                // vertex 0 of a Zipf graph fills ~1/5 of a frontier: one atomic per
                // distinct vertex per warp (take depends on v only)
                unsigned peers = __match_any_sync(act, v[q]);
                if (lane == __ffs(peers) - 1) {
                    unsigned long long c = __popc(peers);
                    if (p.topo_reads) atomicAdd((unsigned long long*)(p.topo_reads + v[q]), c);
                    if (p.edge_trav && take[q]) atomicAdd((unsigned long long*)(p.edge_trav + v[q]), c * take[q]);
                }
            }
        }
    }
    if (TIERED && p.tier_reads) {
        // topology reads by tier: positions and sampled edges (PCIe bytes for the host tier)
#pragma unroll
        for (int c = 0; c < 3; ++c) {
            uint32_t n = 0, e = 0;
#pragma unroll
            for (int q = 0; q < PPT; ++q) {
                n += __popc(__ballot_sync(kFull, valid[q] && tier[q] == c));
                e += (valid[q] && tier[q] == c) ? take[q] : 0u;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) e += __shfl_xor_sync(kFull, e, o);
            if (lane == 0 && n) {
                atomicAdd((unsigned long long*)(p.tier_reads + c), (unsigned long long)n);
                atomicAdd((unsigned long long*)(p.tier_reads + 3 + c), (unsigned long long)e);
            }
        }
        // PCIe transactions of host-tier reads, t(v) = 1 + ceil(deg * 4 / CLS)
        uint32_t tx = 0;
#pragma unroll
        for (int q = 0; q < PPT; ++q)
            tx += (valid[q] && tier[q] == 2) ? 1u + (uint32_t)(((uint64_t)deg[q] * p.u32b + p.cls - 1) / p.cls) : 0u;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) tx += __shfl_xor_sync(kFull, tx, o);
        if (lane == 0 && tx) atomicAdd((unsigned long long*)(p.tier_reads + 6), (unsigned long long)tx);
    }
    if (p.txn_total) {
        // t(v) = 1 + ceil(nc(v) * uint32_bytes / CLS), sampling.py:177-187
        uint64_t tv = 0;
#pragma unroll
        for (int q = 0; q < PPT; ++q) tv += valid[q] ? 1ull + ((uint64_t)deg[q] * p.u32b + p.cls - 1) / p.cls : 0ull;
        uint64_t sum = Reduce(tmp.reduce).Sum(tv);
        if (tid == 0 && sum) atomicAdd((unsigned long long*)p.txn_total, (unsigned long long)sum);
        __syncthreads();
    }
    uint32_t excl[PPT], total;
    Scan(tmp.scan).ExclusiveSum(take, excl, total);
    const uint64_t sidx = (uint64_t)b * p.tiles_per_batch + t;
    const uint64_t sfirst = (uint64_t)b * p.tiles_per_batch;
    if (tid == 0 && t != 0) publish(p.tile_state + sidx, kFlagAgg | total);

    uint32_t* out = p.out_nbrs + b * p.nstride;
    uint32_t* bm = p.bitmap ? p.bitmap + b * p.bwords : nullptr;
    uint32_t* sm = p.summary ? p.summary + b * p.swords : nullptr;
    const uint32_t rounds = (total + kCap - 1) / kCap;

    for (uint32_t r = 0; r < max(rounds, 1u); ++r) {
        const uint32_t r0 = r * kCap;
        const uint32_t r1 = min(total, r0 + kCap);
        // ---- phase 2a: stage the source edge index of every output item in [r0, r1)
        bool need_warp[PPT];
        bool done_two = false;
#ifndef GC_NO_DUAL
        if constexpr (PPT == 2 && S > 0) {
            const auto choice = [&](int q) {
                return valid[q] && !p.exact_only && deg[q] > p.fanout && deg[q] <= 64 && p.fanout < (uint32_t)S;
            };
            if (rounds <= 1 && choice(0) && choice(1)) {
                bool nw[2];
                select_thread_two<S>(reinterpret_cast<const uint64_t(&)[2]>(hc), reinterpret_cast<const uint32_t(&)[2]>(deg),
                                     reinterpret_cast<const uint64_t(&)[2]>(o0), reinterpret_cast<const uint32_t(&)[2]>(excl),
                                     p.fanout, s_items, p.k32, nw);
                need_warp[0] = nw[0];
                need_warp[1] = nw[1];
                done_two = true;
            }
        }
#endif
#pragma unroll
        for (int q = 0; q < PPT; ++q) {
            if (done_two) break;
            need_warp[q] = false;
            const bool thread_copy = deg[q] <= p.fanout && deg[q] <= 64;
            const bool thread_choice =
                S > 0 && !p.exact_only && deg[q] > p.fanout && deg[q] <= 64 && p.fanout < (uint32_t)S;
            if (valid[q] && take[q] && excl[q] + take[q] > r0 && excl[q] < r1) {
                if (thread_copy) {
                    if (rounds <= 1)
                        for (uint32_t k = 0; k < deg[q]; ++k) s_items[excl[q] + k] = (Item)(o0[q] + k);
                    else
                        for (uint32_t k = 0; k < deg[q]; ++k) stage(s_items, excl[q] + k, r0, r1, o0[q] + k);
                } else if (thread_choice) {
                    need_warp[q] = rounds <= 1 ? !select_thread<(S > 0 ? S : 4), false>(
                                                     hc[q], deg[q], p.fanout, o0[q], excl[q], r0, r1, s_items, p.k32)
                                               : !select_thread<(S > 0 ? S : 4), true>(
                                                     hc[q], deg[q], p.fanout, o0[q], excl[q], r0, r1, s_items, p.k32);
                } else {
                    need_warp[q] = true;
                }
            }
        }
#pragma unroll
        for (int q = 0; q < PPT; ++q) {
            unsigned todo = __ballot_sync(kFull, need_warp[q]);
            while (todo) {
                const int src = __ffs(todo) - 1;
                todo &= todo - 1u;
                const uint32_t d = __shfl_sync(kFull, deg[q], src);
                const uint64_t base = __shfl_sync(kFull, o0[q], src);
                const uint32_t e0 = __shfl_sync(kFull, excl[q], src);
                const uint64_t h = __shfl_sync(kFull, hc[q], src);
                if (d <= p.fanout) {
                    for (uint32_t k = lane; k < d; k += 32) stage(s_items, e0 + k, r0, r1, base + k);
                } else {
                    select_warp(h, d, p.fanout, base, e0, r0, r1, s_items, p.exact_only);
                }
            }
        }
        if (r == 0) {
            // ---- look-back for the batch-level output prefix of this tile, run by the
            // first warp to finish its selection: its L2 round trips overlap the other
            // warps' selection (warp 0, the lowest-priority warp of the CTA under the
            // highest-warp-id-first issue policy, is usually the last to finish)
            uint32_t first = 0;
            if (lane == 0) first = atomicAdd(&s_arrive, 1u) == 0u;
            if (__shfl_sync(kFull, first, 0)) {
                uint64_t pre = lookback_warp(p.tile_state, sfirst, sidx, total);
                if (lane == 0) s_prefix = pre;
            }
            __syncthreads();
            const uint32_t prefix = (uint32_t)s_prefix;
            uint32_t* offs = p.out_off + b * p.ostride;
#pragma unroll
            for (int q = 0; q < PPT; ++q) {
                const uint64_t pos = p0 + (uint32_t)tid * PPT + q;
                if (valid[q]) __stcs(offs + pos, prefix + excl[q]);
                if (valid[q] && pos + 1 == F) {
                    offs[F] = prefix + excl[q] + take[q];
                    p.out_count[b] = prefix + excl[q] + take[q];
                }
            }
            if (F == 0 && tid == 0) {
                offs[0] = 0;
                p.out_count[b] = 0;
            }
        } else {
            __syncthreads();
        }
        // ---- phase 2b: coalesced emission of the staged items
        const uint32_t cnt = r1 > r0 ? r1 - r0 : 0;
        uint32_t* dst = out + (uint32_t)s_prefix + r0;
        constexpr int kEmit = emit_items<S>();
        for (uint32_t k0 = tid; k0 < cnt; k0 += kEmit * kHopThreads) {
            if (k0 + (kEmit - 1) * kHopThreads < cnt)
                emit_group<kEmit, true, TIERED>(s_items + k0, cnt - k0, dst + k0, p, bm, sm);
            else
                emit_group<kEmit, false, TIERED>(s_items + k0, cnt - k0, dst + k0, p, bm, sm);
        }
        // s_items is reused by the next round only; the last round exits without a barrier
        if (r + 1 < rounds) __syncthreads();
    }
}

// positions per thread: 2 for the networks up to S = 11 (fanout <= 10: a 512-position
// tile stages at most 5120 items in one round), else 1 — as launch_hop instantiates
static int positions_per_thread(uint32_t fanout, bool tiered) {
    (void)tiered;
    return fanout < 11 ? GC_HOP_PPT : 1;
}

// positions per tile: one staging round whenever fanout <= 128
static uint32_t tile_positions(uint32_t fanout, bool tiered) {
    const uint32_t cap = (uint32_t)kTilePos * positions_per_thread(fanout, tiered);
    uint32_t tp = (uint32_t)item_cap(tiered) / (fanout ? fanout : 1);
    tp = tp >= cap ? cap : (tp / 32) * 32;
    return tp < 32 ? 32 : tp;
}

static unsigned tiles_for(uint32_t max_frontier, uint32_t tile_pos) {
    unsigned t = (max_frontier + tile_pos - 1) / tile_pos;
    return t ? t : 1u;
}

// smallest insertion network holding ranks 0..fanout (0: no thread path)
static int network_slots(uint32_t fanout) {
    const int sizes[] = {4, 6, 8, 11, 16, 21, 26, 32};
    for (int s : sizes)
        if (fanout < (uint32_t)s) return s;
    return 0;
}

template <int S>
static void launch_hop(const HopParams& p, dim3 grid, bool tiered, cudaStream_t s) {
    constexpr int PPT_CSR = S > 0 && S <= 11 ? GC_HOP_PPT : 1;
    constexpr int PPT_TIERED = PPT_CSR;
    if (tiered)
        k_hop_expand<S, true, PPT_TIERED><<<grid, kHopThreads, 0, s>>>(p);
    else
        k_hop_expand<S, false, PPT_CSR><<<grid, kHopThreads, 0, s>>>(p);
}

}  // namespace gc

using namespace gc;

extern "C" {

int gc_set_option(int option, int value) {
    if (option == GC_OPT_DEFER_ROWS) {
        GC_REQUIRE(value >= 0 && value <= 4096, GC_ERR_VALUE, "gc_set_option: GC_OPT_DEFER_ROWS out of range");
        gc::set_defer_rows(value);
        return GC_OK;
    }
    if (option == GC_OPT_DEFER_ORDER) {
        GC_REQUIRE(value == 0 || value == 1, GC_ERR_VALUE, "gc_set_option: GC_OPT_DEFER_ORDER must be 0 or 1");
        gc::set_defer_order(value);
        return GC_OK;
    }
    if (option == GC_OPT_GATHER_CTAS_PER_SM) {
        GC_REQUIRE(value >= 1 && value <= 64, GC_ERR_VALUE, "gc_set_option: GC_OPT_GATHER_CTAS_PER_SM out of range");
        gc::set_gather_ctas_per_sm(value);
        return GC_OK;
    }
    if (option == GC_OPT_DEFER_CTAS) {
        GC_REQUIRE(value >= 1 && value <= 65535, GC_ERR_VALUE, "gc_set_option: GC_OPT_DEFER_CTAS out of range");
        gc::set_defer_ctas(value);
        return GC_OK;
    }
    if (option == GC_OPT_UNIQUE_BATCH_CTAS) {
        GC_REQUIRE(value >= 0, GC_ERR_VALUE, "gc_set_option: GC_OPT_UNIQUE_BATCH_CTAS out of range");
        gc::set_unique_batch_min(value);
        return GC_OK;
    }
    GC_REQUIRE(option == GC_OPT_EXACT_SELECTION, GC_ERR_VALUE, "gc_set_option: unknown option");
    g_exact_only = value ? 1 : 0;
    return GC_OK;
}

size_t gc_hop_expand_temp_bytes(uint32_t num_batches, uint32_t max_frontier) {
    return align_up((size_t)num_batches * tiles_for(max_frontier, 32) * sizeof(uint64_t), 256) +
           align_up((size_t)num_batches * sizeof(uint32_t), 256);
}

int gc_hop_expand(const gc_topology_t* topo, const uint32_t* d_frontier, uint64_t frontier_stride,
                  const uint32_t* d_frontier_count, uint32_t max_frontier, uint32_t fanout,
                  const uint64_t* d_hop_keys, uint32_t num_batches, uint32_t* d_out_offsets,
                  uint64_t offsets_stride, uint32_t* d_out_nbrs, uint64_t nbrs_stride, uint32_t* d_out_count,
                  const gc_visited_t* visited, int mark_frontier, const gc_hotness_t* hot,
                  void* d_temp, size_t temp_bytes, void* stream) {
    GC_REQUIRE(topo && topo->full.row_offsets, GC_ERR_VALUE, "gc_hop_expand: topology is null");
    const gc_csr_t* graph = &topo->full;
    GC_REQUIRE(fanout >= 1, GC_ERR_VALUE, "fanouts must all be >= 1");
    GC_REQUIRE((uint64_t)max_frontier * fanout < (1ull << 32), GC_ERR_VALUE,
               "gc_hop_expand: max_frontier * fanout must be < 2^32 per batch");
    GC_REQUIRE(offsets_stride >= (uint64_t)max_frontier + 1, GC_ERR_VALUE, "gc_hop_expand: offsets stride too small");
    GC_REQUIRE(graph->num_edges == 0 || graph->col_indices, GC_ERR_VALUE, "gc_hop_expand: graph has no columns");
    if (num_batches == 0) return GC_OK;
    const size_t need = gc_hop_expand_temp_bytes(num_batches, max_frontier);
    GC_REQUIRE(d_temp && temp_bytes >= need, GC_ERR_VALUE, "gc_hop_expand: temp buffer too small");
    cudaStream_t s = as_stream(stream);
    // the plain-CSR kernel stages 32-bit edge indices; a CSR with 2^32 or more edges
    // takes the tiered kernel (64-bit items), which also reads a location-free CSR
    const bool tiered = topo->location != nullptr || topo->full_on_host || graph->num_edges >= (1ull << 32);
    const uint32_t tile_pos = tile_positions(fanout, tiered);
    const unsigned tiles = tiles_for(max_frontier, tile_pos);
    HopParams p{};
    p.tile_pos = tile_pos;
    p.ro = graph->row_offsets;
    p.ci = graph->col_indices;
    p.loc = topo->location;
    for (int g = 0; g < GC_MAX_PEERS; ++g) {
        p.soff[g] = topo->slab_offsets[g];
        p.scols[g] = topo->slab_cols[g];
    }
    p.self_rank = topo->self_rank;
    p.full_on_host = topo->full_on_host;
    p.tier_reads = topo->tier_reads;
    p.n = (uint64_t)graph->num_vertices;
    p.frontier = d_frontier;
    p.fstride = frontier_stride;
    p.fcount = d_frontier_count;
    p.fanout = fanout;
    p.tiles_per_batch = tiles;
    p.hop_keys = d_hop_keys;
    p.out_off = d_out_offsets;
    p.ostride = offsets_stride;
    p.out_nbrs = d_out_nbrs;
    p.nstride = nbrs_stride;
    p.out_count = d_out_count;
    if (visited) {
        p.bitmap = visited->bitmap;
        p.bwords = visited->words;
        p.summary = visited->summary;
        p.swords = visited->summary_words;
    }
    p.mark_frontier = mark_frontier;
    p.exact_only = g_exact_only;
    p.k32 = 32;
    p.cls = 64;
    p.u32b = 4;
    if (hot) {
        p.topo_reads = hot->topo_reads;
        p.edge_trav = hot->edge_traversals;
        p.txn_total = hot->txn_total;
        p.cls = hot->cache_line_bytes ? hot->cache_line_bytes : 64;
        p.u32b = hot->uint32_bytes ? hot->uint32_bytes : 4;
    }
    const size_t state_bytes = align_up((size_t)num_batches * tiles * sizeof(uint64_t), 256);
    p.tile_state = static_cast<uint64_t*>(d_temp);
    p.tile_counter = reinterpret_cast<uint32_t*>(static_cast<char*>(d_temp) + state_bytes);
    GC_TRY(cudaMemsetAsync(d_temp, 0, state_bytes + align_up((size_t)num_batches * sizeof(uint32_t), 256), s),
           "gc_hop_expand memset");
    GC_REQUIRE(num_batches <= 65535 && tiles < (1u << 31), GC_ERR_VALUE, "gc_hop_expand: window too large");
    const dim3 grid(tiles, num_batches);
    switch (network_slots(fanout)) {
        case 4: launch_hop<4>(p, grid, tiered, s); break;
        case 6: launch_hop<6>(p, grid, tiered, s); break;
        case 8: launch_hop<8>(p, grid, tiered, s); break;
        case 11: launch_hop<11>(p, grid, tiered, s); break;
        case 16: launch_hop<16>(p, grid, tiered, s); break;
        case 21: launch_hop<21>(p, grid, tiered, s); break;
        case 26: launch_hop<26>(p, grid, tiered, s); break;
        case 32: launch_hop<32>(p, grid, tiered, s); break;
        default: launch_hop<0>(p, grid, tiered, s); break;
    }
    GC_CHECK_LAUNCH("gc_hop_expand");
    return GC_OK;
}

}  // extern "C"
