// Row-partitioned hierarchy for multi-GPU solves.
//
// Every rank builds the same host hierarchy (bit-exact setup), then takes its
// slice of each level:
//  * distributed level: contiguous owned rows [lo, hi). Level 0 is split
//    evenly; a coarse level inherits the partition induced by its aggregates
//    (coarse row c is owned by the owner of its first member; ids follow
//    node-HEM discovery order, so owned coarse rows are contiguous). Halo
//    layout: when the ghost ids each peer supplies fill (nearly) contiguous
//    ranges -- always for slab partitions of structured grids -- the "window"
//    layout keeps global column offsets (local column = c - lo, ghosts at
//    negative / >= n_own positions of the x vectors), so the row-pattern
//    format still applies; otherwise columns are renumbered [own | ghost],
//    ghosts sorted by global id. Entry order within a row is untouched, so
//    every row sum keeps the reference's bits.
//  * replicated level (n < gather_rows, and everything below it): held whole
//    on every rank and solved redundantly after one gather of its rhs.
// Exchange plans say which owned entries each peer needs (send lists) and
// where each peer's values land in the ghost region (recv offsets).
#pragma once

#include <cstdint>
#include <vector>

#include "sb_internal.h"

namespace sb {

struct Exchange {
    std::vector<int> send_peers, recv_peers;   // ascending peer ranks
    std::vector<int64_t> send_off, recv_off;   // prefix offsets (size peers + 1)
    std::vector<int32_t> send_idx;             // owned local indices to pack, grouped by send peer
    std::vector<int64_t> recv_dst;             // where each recv peer's chunk lands, relative to the
                                               // receiving buffer (halo: the own-rows pointer of x)
    int64_t total_send() const { return send_off.empty() ? 0 : send_off.back(); }
    int64_t total_recv() const { return recv_off.empty() ? 0 : recv_off.back(); }
};

struct PartLevel {
    bool replicated = false;
    int64_t n_glob = 0, lo = 0, hi = 0;  // owned rows (replicated: [0, n_glob))
    HostCsr A;                            // owned rows; columns: window mode c - lo (negative below),
                                          // compact mode [own | ghost]
    std::vector<int64_t> ghost_glob;      // global ids exchanged into the halo (window mode: whole ranges)
    int64_t wb = 0, wa = 0;               // x-like vectors hold wb rows below own and wa above
    Exchange halo;                        // x halo for SpMV / sweeps / residual
    // restriction into the next level
    int64_t c_lo = 0, c_hi = 0;           // owned coarse rows (global ids)
    std::vector<int32_t> mem0, mem1;      // members of owned coarse rows: index into [own r | r ghosts], -1 none
    std::vector<int64_t> rghost_glob;     // residual entries needed from peers (straddling aggregates)
    Exchange rx;
    // prolongation from the next level
    std::vector<int32_t> parent;          // own fine row -> index into [own coarse | xc ghosts] (or global if next replicated)
    std::vector<int64_t> xcghost_glob;
    Exchange px;
    // gather of the next level's rhs when it is the first replicated level
    std::vector<int64_t> gather_lo;       // per rank: owned coarse range of the next level
};

struct Partition {
    int rank = 0, nranks = 1;
    int first_replicated = 0;             // index of the first replicated level (== nlevels if none)
    std::vector<PartLevel> L;
    // per level, per rank: owned range (distributed levels)
    std::vector<std::vector<int64_t>> bounds;  // bounds[k][r] .. bounds[k][r+1]
};

// Builds rank `rank`'s partition of h. gather_rows: levels with fewer global
// rows (and all coarser ones) are replicated; level 0 is always distributed
// when nranks > 1.
Partition build_partition(const Hier &h, int rank, int nranks, int64_t gather_rows);

} // namespace sb
