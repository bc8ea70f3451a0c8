// Row partition + exchange plans (see sb_dist.h). Host code only: every rank
// computes the same plans from the same (bit-exact) hierarchy, so no
// communication is needed to agree on them.

#include "sb_dist.h"

#include <algorithm>
#include <cstring>

namespace sb {

namespace {

int owner_of(const std::vector<int64_t> &b, int64_t j) {
    return static_cast<int>(std::upper_bound(b.begin(), b.end(), j) - b.begin()) - 1;
}

// first (smallest) member of every coarse row
std::vector<int64_t> first_members(const std::vector<int32_t> &agg, int64_t nc) {
    std::vector<int64_t> m0(static_cast<size_t>(nc), -1);
    for (int64_t i = 0; i < static_cast<int64_t>(agg.size()); ++i)
        if (m0[agg[i]] < 0) m0[agg[i]] = i;
    return m0;
}

// Induced coarse bounds: coarse row c belongs to the owner of its first member.
std::vector<int64_t> induced_bounds(const std::vector<int64_t> &fb, const std::vector<int32_t> &agg, int64_t nc,
                                    int nranks) {
    const std::vector<int64_t> m0 = first_members(agg, nc);
    std::vector<int64_t> cb(static_cast<size_t>(nranks) + 1, nc);
    cb[0] = 0;
    int prev = 0;
    for (int64_t c = 0; c < nc; ++c) {
        const int o = owner_of(fb, m0[c]);
        if (o < prev)
            throw invalid_argument("partition: coarse numbering is not monotone in the fine partition");
        for (int r = prev + 1; r <= o; ++r) cb[r] = c;
        prev = o;
    }
    for (int r = prev + 1; r <= nranks; ++r) cb[r] = nc;
    return cb;
}

// Exchange plan for "rank needs the entries `need` (global ids, sorted,
// grouped by owner) of a vector distributed by bounds b". `need_of(q)` gives
// the same list for every other rank q (to build this rank's send lists).
template <typename NeedOf>
Exchange make_exchange(const std::vector<int64_t> &b, int rank, int nranks, const std::vector<int64_t> &need,
                       NeedOf need_of) {
    Exchange e;
    e.recv_off.push_back(0);
    for (size_t i = 0; i < need.size();) {
        const int o = owner_of(b, need[i]);
        size_t j = i;
        while (j < need.size() && owner_of(b, need[j]) == o) ++j;
        e.recv_peers.push_back(o);
        e.recv_dst.push_back(e.recv_off.back());  // packed (callers may remap)
        e.recv_off.push_back(static_cast<int64_t>(j));
        i = j;
    }
    e.send_off.push_back(0);
    for (int q = 0; q < nranks; ++q) {
        if (q == rank) continue;
        const std::vector<int64_t> nq = need_of(q);
        int64_t cnt = 0;
        for (int64_t g : nq)
            if (g >= b[rank] && g < b[rank + 1]) {
                e.send_idx.push_back(static_cast<int32_t>(g - b[rank]));
                ++cnt;
            }
        if (cnt) {
            e.send_peers.push_back(q);
            e.send_off.push_back(e.send_off.back() + cnt);
        }
    }
    return e;
}

// ghost columns (global ids, sorted) of the rows [lo, hi) of A
std::vector<int64_t> ghosts_of(const HostCsr &A, int64_t lo, int64_t hi) {
    std::vector<int64_t> g;
    for (int64_t i = lo; i < hi; ++i)
        for (int64_t k = A.rp[i]; k < A.rp[i + 1]; ++k)
            if (A.ci[k] < lo || A.ci[k] >= hi) g.push_back(A.ci[k]);
    std::sort(g.begin(), g.end());
    g.erase(std::unique(g.begin(), g.end()), g.end());
    return g;
}

// Halo ids rank q receives for rows [b[q], b[q+1]) of A, and whether they
// use the window layout: the ghost ids of each peer widened to the peer's
// [min, max] range when the widened total stays within 2x the ghosts (+64).
std::vector<int64_t> halo_need(const HostCsr &A, const std::vector<int64_t> &b, int q, bool *window) {
    const std::vector<int64_t> g = ghosts_of(A, b[q], b[q + 1]);
    std::vector<int64_t> w;
    for (size_t i = 0; i < g.size();) {
        const int o = owner_of(b, g[i]);
        size_t j = i;
        while (j < g.size() && owner_of(b, g[j]) == o) ++j;
        for (int64_t id = g[i]; id <= g[j - 1]; ++id) w.push_back(id);
        i = j;
    }
    *window = static_cast<int64_t>(w.size()) <= 2 * static_cast<int64_t>(g.size()) + 64;
    return *window ? w : g;
}

// second members (owned elsewhere) of the coarse rows [c_lo, c_hi)
std::vector<int64_t> partner_ghosts(const std::vector<int32_t> &agg, const std::vector<int64_t> &fb, int owner,
                                    int64_t c_lo, int64_t c_hi) {
    std::vector<int64_t> g;
    for (int64_t i = 0; i < static_cast<int64_t>(agg.size()); ++i) {
        const int64_t c = agg[i];
        if (c >= c_lo && c < c_hi && (i < fb[owner] || i >= fb[owner + 1])) g.push_back(i);
    }
    std::sort(g.begin(), g.end());
    return g;
}

// coarse parents (owned elsewhere) of the fine rows [lo, hi)
std::vector<int64_t> parent_ghosts(const std::vector<int32_t> &agg, int64_t lo, int64_t hi, int64_t c_lo,
                                   int64_t c_hi) {
    std::vector<int64_t> g;
    for (int64_t i = lo; i < hi; ++i)
        if (agg[i] < c_lo || agg[i] >= c_hi) g.push_back(agg[i]);
    std::sort(g.begin(), g.end());
    g.erase(std::unique(g.begin(), g.end()), g.end());
    return g;
}

} // namespace

Partition build_partition(const Hier &h, int rank, int nranks, int64_t gather_rows) {
    if (nranks < 1 || rank < 0 || rank >= nranks) throw invalid_argument("partition: bad rank / world size");
    const int L = static_cast<int>(h.levels.size());
    Partition P;
    P.rank = rank;
    P.nranks = nranks;
    P.L.resize(static_cast<size_t>(L));
    P.bounds.resize(static_cast<size_t>(L));
    // which levels are distributed
    int fr = L;
    for (int k = 0; k < L; ++k) {
        const bool dist = nranks > 1 && k + 1 < L && (k == 0 || h.levels[k].A.n >= gather_rows);
        if (!dist) {
            fr = k;
            break;
        }
    }
    if (nranks == 1) fr = 0;
    P.first_replicated = fr;
    // bounds
    const int64_t n0 = h.levels[0].A.n;
    P.bounds[0].resize(static_cast<size_t>(nranks) + 1);
    for (int r = 0; r <= nranks; ++r) P.bounds[0][r] = n0 * r / nranks;
    for (int k = 0; k + 1 < L && k + 1 <= fr; ++k)
        P.bounds[k + 1] = induced_bounds(P.bounds[k], h.levels[k].agg, h.levels[k].n_coarse, nranks);
    for (int k = 0; k < L; ++k) {
        const HostLevel &H = h.levels[static_cast<size_t>(k)];
        PartLevel &pl = P.L[static_cast<size_t>(k)];
        pl.n_glob = H.A.n;
        if (k >= fr) {  // replicated: the whole level
            pl.replicated = true;
            pl.lo = 0;
            pl.hi = H.A.n;
            pl.A = H.A;
            if (k + 1 < L) {
                pl.c_lo = 0;
                pl.c_hi = H.n_coarse;
                pl.parent.assign(H.agg.begin(), H.agg.end());
            }
            continue;
        }
        const std::vector<int64_t> &b = P.bounds[k];
        pl.lo = b[rank];
        pl.hi = b[rank + 1];
        const int64_t nl = pl.hi - pl.lo;
        // local matrix: window layout (global offsets kept) or [own | ghost] columns
        bool window = false;
        pl.ghost_glob = halo_need(H.A, b, rank, &window);
        const int64_t n_below = std::lower_bound(pl.ghost_glob.begin(), pl.ghost_glob.end(), pl.lo) - pl.ghost_glob.begin();
        if (window) {
            pl.wb = n_below ? pl.lo - pl.ghost_glob.front() : 0;
            pl.wa = static_cast<int64_t>(pl.ghost_glob.size()) > n_below ? pl.ghost_glob.back() + 1 - pl.hi : 0;
        } else {
            pl.wb = 0;
            pl.wa = static_cast<int64_t>(pl.ghost_glob.size());
        }
        pl.A.n = nl;
        pl.A.ncols = nl + pl.wa;
        pl.A.rp.assign(static_cast<size_t>(nl) + 1, 0);
        for (int64_t i = pl.lo; i < pl.hi; ++i) {
            for (int64_t kk = H.A.rp[i]; kk < H.A.rp[i + 1]; ++kk) {
                const int64_t c = H.A.ci[kk];
                int64_t lc;
                if (window || (c >= pl.lo && c < pl.hi)) lc = c - pl.lo;
                else lc = nl + (std::lower_bound(pl.ghost_glob.begin(), pl.ghost_glob.end(), c) - pl.ghost_glob.begin());
                pl.A.ci.push_back(static_cast<int32_t>(lc));
                pl.A.v.push_back(H.A.v[kk]);
            }
            pl.A.rp[i - pl.lo + 1] = static_cast<int64_t>(pl.A.ci.size());
        }
        pl.A.sync_rp32();
        pl.halo = make_exchange(b, rank, nranks, pl.ghost_glob, [&](int q) {
            bool wq = false;
            return halo_need(H.A, b, q, &wq);
        });
        for (size_t j = 0; j < pl.halo.recv_peers.size(); ++j)  // chunk destinations (relative to own row 0)
            pl.halo.recv_dst[j] = window ? pl.ghost_glob[static_cast<size_t>(pl.halo.recv_off[j])] - pl.lo
                                         : nl + pl.halo.recv_off[j];
        // restriction / prolongation with the next level
        const bool next_rep = k + 1 >= fr;
        const std::vector<int64_t> cb =
            next_rep ? induced_bounds(b, H.agg, H.n_coarse, nranks) : P.bounds[k + 1];
        pl.gather_lo = cb;
        pl.c_lo = cb[rank];
        pl.c_hi = cb[rank + 1];
        const std::vector<int64_t> m0 = first_members(H.agg, H.n_coarse);
        pl.rghost_glob = partner_ghosts(H.agg, b, rank, pl.c_lo, pl.c_hi);
        pl.rx = make_exchange(b, rank, nranks, pl.rghost_glob,
                              [&](int q) { return partner_ghosts(H.agg, b, q, cb[q], cb[q + 1]); });
        pl.mem0.assign(static_cast<size_t>(pl.c_hi - pl.c_lo), -1);
        pl.mem1.assign(static_cast<size_t>(pl.c_hi - pl.c_lo), -1);
        auto rloc = [&](int64_t i) -> int32_t {
            if (i >= pl.lo && i < pl.hi) return static_cast<int32_t>(i - pl.lo);
            return static_cast<int32_t>(
                nl + (std::lower_bound(pl.rghost_glob.begin(), pl.rghost_glob.end(), i) - pl.rghost_glob.begin()));
        };
        for (int64_t i = 0; i < H.A.n; ++i) {  // members ascending
            const int64_t c = H.agg[i];
            if (c < pl.c_lo || c >= pl.c_hi) continue;
            int32_t &m = pl.mem0[c - pl.c_lo] < 0 ? pl.mem0[c - pl.c_lo] : pl.mem1[c - pl.c_lo];
            m = rloc(i);
        }
        (void)m0;
        if (next_rep) {
            pl.parent.resize(static_cast<size_t>(nl));
            for (int64_t i = pl.lo; i < pl.hi; ++i) pl.parent[i - pl.lo] = H.agg[i];  // global coarse id
        } else {
            pl.xcghost_glob = parent_ghosts(H.agg, pl.lo, pl.hi, pl.c_lo, pl.c_hi);
            pl.px = make_exchange(cb, rank, nranks, pl.xcghost_glob, [&](int q) {
                return parent_ghosts(H.agg, b[q], b[q + 1], cb[q], cb[q + 1]);
            });
            const int64_t ncl = pl.c_hi - pl.c_lo;
            pl.parent.resize(static_cast<size_t>(nl));
            for (int64_t i = pl.lo; i < pl.hi; ++i) {
                const int64_t c = H.agg[i];
                pl.parent[i - pl.lo] =
                    (c >= pl.c_lo && c < pl.c_hi)
                        ? static_cast<int32_t>(c - pl.c_lo)
                        : static_cast<int32_t>(ncl + (std::lower_bound(pl.xcghost_glob.begin(), pl.xcghost_glob.end(), c) -
                                                      pl.xcghost_glob.begin()));
            }
        }
    }
    return P;
}

} // namespace sb

// ---------------------------------------------------------------------------
// C ABI: plan inspection (host only; used by the multi-process gloo tests)
// ---------------------------------------------------------------------------
using namespace sb;

struct sb_part_s {
    Partition p;
};

extern "C" {

int sb_partition(sb_hier h, int rank, int nranks, int64_t gather_rows, sb_part *out) {
    return guard([&] {
        Hier *H = hier_of(h);
        if (!H || !out) throw invalid_argument("sb_partition: null argument");
        *out = new sb_part_s{build_partition(*H, rank, nranks, gather_rows)};
    });
}

void sb_partition_free(sb_part p) { delete p; }

int sb_partition_info(sb_part p, int *nlevels, int *first_replicated) {
    if (!p) return SB_EINVAL;
    *nlevels = static_cast<int>(p->p.L.size());
    *first_replicated = p->p.first_replicated;
    return SB_OK;
}

// Level k of this rank. i64[0..10] = {n_glob, lo, hi, n_ghost, c_lo, c_hi,
// n_rghost, n_xcghost, replicated, wb, wa}. Borrowed arrays (valid while p lives):
// A (local CSR), ghost / rghost / xcghost global ids, mem0 / mem1 / parent,
// and the three exchange plans (peers, offsets, send indices).
int sb_partition_level(sb_part p, int k, int64_t *i64, sb_csr *A, const int64_t **ghost, const int64_t **rghost,
                       const int64_t **xcghost, const int32_t **mem0, const int32_t **mem1, const int32_t **parent) {
    return guard([&] {
        if (!p || k < 0 || k >= static_cast<int>(p->p.L.size())) throw invalid_argument("sb_partition_level: level");
        const PartLevel &l = p->p.L[static_cast<size_t>(k)];
        const int64_t v[11] = {l.n_glob, l.lo, l.hi, static_cast<int64_t>(l.ghost_glob.size()), l.c_lo, l.c_hi,
                               static_cast<int64_t>(l.rghost_glob.size()), static_cast<int64_t>(l.xcghost_glob.size()),
                               l.replicated ? 1 : 0, l.wb, l.wa};
        std::memcpy(i64, v, sizeof(v));
        if (A) {
            A->nrows = l.A.n;
            A->ncols = l.A.ncols;
            A->row_ptr32 = l.A.rp32.empty() ? nullptr : l.A.rp32.data();
            A->row_ptr64 = l.A.rp32.empty() ? l.A.rp.data() : nullptr;
            A->col_idx = l.A.ci.data();
            A->values = l.A.v.data();
        }
        if (ghost) *ghost = l.ghost_glob.data();
        if (rghost) *rghost = l.rghost_glob.data();
        if (xcghost) *xcghost = l.xcghost_glob.data();
        if (mem0) *mem0 = l.mem0.data();
        if (mem1) *mem1 = l.mem1.data();
        if (parent) *parent = l.parent.data();
    });
}

// Exchange plan `which` (0 halo, 1 residual partners, 2 coarse parents) of
// level k: counts[0..3] = {n_send_peers, n_recv_peers, total_send, total_recv}.
int sb_partition_exchange(sb_part p, int k, int which, int64_t *counts, const int **send_peers,
                          const int64_t **send_off, const int32_t **send_idx, const int **recv_peers,
                          const int64_t **recv_off, const int64_t **recv_dst) {
    return guard([&] {
        if (!p || k < 0 || k >= static_cast<int>(p->p.L.size())) throw invalid_argument("sb_partition_exchange: level");
        const PartLevel &l = p->p.L[static_cast<size_t>(k)];
        const Exchange &e = which == 0 ? l.halo : which == 1 ? l.rx : l.px;
        counts[0] = static_cast<int64_t>(e.send_peers.size());
        counts[1] = static_cast<int64_t>(e.recv_peers.size());
        counts[2] = e.total_send();
        counts[3] = e.total_recv();
        *send_peers = e.send_peers.data();
        *send_off = e.send_off.data();
        *send_idx = e.send_idx.data();
        *recv_peers = e.recv_peers.data();
        *recv_off = e.recv_off.data();
        if (recv_dst) *recv_dst = e.recv_dst.data();
    });
}

} // extern "C"
