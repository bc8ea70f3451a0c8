// Multi-rank solve phase, included at the end of sb_runtime.cu.
//
// One device context per rank holds the rank's slice of every distributed
// level (columns [own | ghost]) and the whole of every replicated level. The
// V-cycle runs the same bitwise kernels level by level; before every kernel
// that gathers x the ghost region is refreshed (halo exchange), straddling
// aggregates exchange residuals / coarse corrections, and at the first
// replicated level the restricted rhs is gathered so every rank solves the
// bottom of the hierarchy redundantly (no scatter back). Krylov dot products
// are rank-local deterministic reductions + an allreduce, after which a
// one-thread kernel runs the reference's scalar logic on every rank.
//
// Three transports:
//  * NCCL (one rank per process / GPU; libnccl.so.2 loaded with dlopen):
//    grouped send/recv for exchanges, ncclAllReduce for dots;
//  * peer memory (P2P, one rank per process / GPU, or in-process ranks): every
//    rank exports the buffers its peers read (CUDA IPC handles; on one node
//    they map over NVLink / NVSwitch) and a monotonic epoch counter. An
//    exchange is: publish (epoch += 1 after the producing kernels), wait until
//    the peers' epochs reach ours (one spinning thread), then the receiver
//    gathers its ghost values straight out of the peers' own rows. Dot products
//    sum every rank's partials in rank order (deterministic, no NCCL);
//  * in-process "virtual ranks" (all ranks in this process, one device):
//    receivers pull peer values with a gather kernel; ordering through CUDA
//    events. Used to test the partitioned GPU path on a single GPU.

#include <dlfcn.h>

#include <nccl.h>

#include "sb_dist.h"

namespace sb {

// ---- NCCL (dlopen) -------------------------------------------------------------
struct NcclApi {
    void *h = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
};

static NcclApi &nccl() {
    static NcclApi api;
    if (api.h) return api;
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) throw cuda_error(std::string("libnccl.so.2 not loadable: ") + dlerror());
    auto sym = [&](const char *n) {
        void *p = dlsym(h, n);
        if (!p) throw cuda_error(std::string("NCCL symbol missing: ") + n);
        return p;
    };
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
    api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
    api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
    api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
    api.h = h;
    return api;
}

#define NC(x)                                                                                        \
    do {                                                                                             \
        ncclResult_t r_ = (x);                                                                       \
        if (r_ != ncclSuccess) throw sb::cuda_error(std::string(#x) + ": " + nccl().GetErrorString(r_)); \
    } while (0)

// ---- device kernels of the partitioned path ---------------------------------------

// dst[i] = src[idx[i]] (pack for NCCL / pull from a peer's buffer in-process)
__global__ void k_gather_idx(int64_t n, const double *__restrict__ src, const int32_t *__restrict__ idx,
                             double *__restrict__ dst) {
    pdl_wait();
    GRID_LOOP(i, n) dst[i] = src[idx[i]];
}

// restriction of owned coarse rows: members index [own r | r ghosts]
__global__ void k_restrict_dist(int64_t nc, const int2 *__restrict__ mem, const double *__restrict__ r,
                                const double *__restrict__ rg, int64_t n_own, double *__restrict__ fc) {
    pdl_wait();
    GRID_LOOP(c, nc) {
        const int2 m = mem[c];
        double s = __dadd_rn(0.0, m.x < n_own ? r[m.x] : rg[m.x - n_own]);
        if (m.y >= 0) s = __dadd_rn(s, m.y < n_own ? r[m.y] : rg[m.y - n_own]);
        fc[c] = s;
    }
}

// x_out = x_in + (0.0 + x_c[parent]) with parents in [own coarse | ghosts]
__global__ void k_prolong_dist(int64_t n, const int32_t *__restrict__ parent, const double *xin,
                               const double *__restrict__ xc, const double *__restrict__ xcg, int64_t nc_own,
                               double *xout) {
    pdl_wait();
    GRID_LOOP(i, n) {
        const int64_t p = parent[i];
        xout[i] = __dadd_rn(xin[i], __dadd_rn(0.0, p < nc_own ? xc[p] : xcg[p - nc_own]));
    }
}

// ---- peer-memory (P2P) transport kernels ----
// publish: every kernel this rank issued before is complete; make its writes
// visible system-wide, then advance the epoch (single writer)
__global__ void k_p2p_publish(unsigned long long *epoch) {
    pdl_wait();
    __threadfence_system();
    const unsigned long long e = *reinterpret_cast<volatile unsigned long long *>(epoch) + 1ull;
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(epoch), "l"(e) : "memory");
}
// wait until each listed peer's epoch reached ours (acquire)
__global__ void k_p2p_wait(const unsigned long long *epoch, const unsigned long long *const *peer_epoch, int npeers) {
    pdl_wait();
    const unsigned long long want = *reinterpret_cast<const volatile unsigned long long *>(epoch);
    for (int i = threadIdx.x; i < npeers; i += blockDim.x) {
        unsigned long long v;
        do {
            asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(peer_epoch[i]) : "memory");
        } while (v < want);
    }
    __syncthreads();
}
// ghost(dst[i]) = peer_own[src[i]]: the receiver pulls its ghost values out of
// a peer's own rows (peer memory: L2-bypassing loads)
__global__ void k_p2p_gather(int64_t n, const double *peer_own, const int32_t *__restrict__ src,
                             double *__restrict__ dst) {
    pdl_wait();
    GRID_LOOP(i, n) dst[i] = __ldcv(peer_own + src[i]);
}
__global__ void k_p2p_copy(int64_t n, const double *src, double *__restrict__ dst) {
    pdl_wait();
    GRID_LOOP(i, n) dst[i] = __ldcv(src + i);
}
// every rank's partials (slot `slot`) summed in rank order -> st->red
__global__ void k_p2p_put(const double *part, double *slotbase, const int *slot) {
    pdl_wait();
    double *dst = slotbase + 2 * (*slot & 1);
    dst[0] = part[0];
    dst[1] = part[1];
}
__global__ void k_p2p_sum(const double *const *slots, int nranks, int *slot, double *out) {
    pdl_wait();
    const int sl = *slot & 1;
    double a = 0.0, b = 0.0;
    for (int r = 0; r < nranks; ++r) {
        a += __ldcv(slots[r] + 2 * sl);
        b += __ldcv(slots[r] + 2 * sl + 1);
    }
    out[0] = a;
    out[1] = b;
    *slot = sl + 1;
}

// in-process allreduce: every rank sums the ranks' partials in rank order
__global__ void k_sum_partials(const double *const *parts, int nranks, double *out) {
    pdl_wait();
    double a = 0.0, b = 0.0;
    for (int r = 0; r < nranks; ++r) {
        a += parts[r][0];
        b += parts[r][1];
    }
    out[0] = a;
    out[1] = b;
}

// ---- partitioned device hierarchy --------------------------------------------------

struct DevExch {
    std::vector<int> send_peers, recv_peers;
    std::vector<int64_t> send_off, recv_off, recv_dst;
    int32_t *send_idx = nullptr;  // device
    double *sendbuf = nullptr;    // device (NCCL packing)
    int64_t nsend = 0, nrecv = 0;
};

struct DistLevel {
    bool dist = false, next_rep = false;
    int64_t n_own = 0, n_ext = 0, nc_own = 0, c_lo = 0;
    int64_t wb = 0, wa = 0;  // x-like vectors: wb rows below own row 0, wa above (n_ext = n_own + wa)
    int64_t q_ilo = 0, q_ihi = 0;  // interior row pairs: no column outside the own rows (swept while the halo flies)
    double *rg = nullptr, *xcg = nullptr;  // residual-partner / coarse-parent ghosts
    DevExch halo, rx, px;
    std::vector<int64_t> gather_lo;  // first replicated level: owned pieces per rank
};

struct RankDev {
    int rank = 0;
    sb_ctx c = nullptr;
    Partition P;
    std::vector<DistLevel> D;
    cudaEvent_t ready = nullptr, done = nullptr;
    cudaStream_t s = nullptr;      // stream the solve is emitted on (the context stream, or a graph body's)
    cudaStream_t s2 = nullptr;     // side stream: the halo exchange overlapping the interior sweep
    cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
    double **part_ptrs = nullptr;  // in-process: device array of every rank's st->part
    // P2P transport
    unsigned long long *epoch = nullptr;  // exported
    double *pslots = nullptr;             // exported: 2 slots x 2 partials
    int *pslot = nullptr;                 // which slot the next allreduce uses
    const unsigned long long **peer_epochs = nullptr;  // device: every rank's epoch pointer (rank order)
    const double **peer_slots = nullptr;               // device: every rank's pslots (rank order)
    std::vector<const unsigned long long *> h_peer_epochs;
    std::vector<std::vector<const double *>> peer_own;  // [buffer id][rank]: that rank's own-row-0 pointer
    std::map<const double *, int> buf_id;               // own-row-0 pointer -> exported buffer id
    std::vector<std::pair<void *, int64_t>> exported;   // (allocation base, own-row-0 offset in bytes) per id
    std::vector<const double *> exported_own;           // own-row-0 pointer per id
    std::vector<void *> opened;                          // IPC mappings to close
    // per distributed level and plan (halo, rx, px): the peers' send indices
    // for this rank, aligned with recv_off
    std::vector<std::array<int32_t *, 3>> src_idx;
    int64_t lo = 0, hi = 0;        // owned rows of level 0
};

} // namespace sb

struct sb_dist_s {
    std::vector<sb::RankDev> R;  // ranks hosted by this process
    int nranks = 1, fr = 0;
    bool local = false;
    ncclComm_t comm = nullptr;
    double last_ms = 0.0;
    int last_launches = 0;
    std::map<std::string, sb::GraphEntry> cache;  // captured whole-solve graphs (NCCL / P2P mode)
    bool p2p = false;       // peer-memory transport
    bool connected = false; // P2P: peers' buffers mapped
    bool graph_failed = false;  // capture failed once: eager from then on (graph_error says why)
    std::string graph_error;
};

namespace sb {

static DevExch upload_exch(sb_ctx c, const Exchange &e) {
    DevExch d;
    d.send_peers = e.send_peers;
    d.recv_peers = e.recv_peers;
    d.send_off = e.send_off.empty() ? std::vector<int64_t>{0} : e.send_off;
    d.recv_off = e.recv_off.empty() ? std::vector<int64_t>{0} : e.recv_off;
    d.recv_dst = e.recv_dst;
    d.nsend = e.total_send();
    d.nrecv = e.total_recv();
    d.send_idx = dalloc<int32_t>(c, std::max<int64_t>(d.nsend, 1), false);
    if (d.nsend)
        CK(cudaMemcpy(d.send_idx, e.send_idx.data(), sizeof(int32_t) * e.send_idx.size(), cudaMemcpyHostToDevice));
    d.sendbuf = dalloc<double>(c, std::max<int64_t>(d.nsend, 1), false);
    return d;
}

// Partitioned level: local matrix + [own | ghost] workspaces + plans.
static void upload_dist_level(sb_ctx c, const PartLevel &pl, DevLevel &D, DistLevel &DL) {
    upload_matrix(c, pl.A, D);
    DL.dist = true;
    DL.n_own = pl.hi - pl.lo;
    DL.n_ext = pl.A.ncols;
    DL.wb = pl.wb;
    DL.wa = pl.wa;
    DL.nc_own = pl.c_hi - pl.c_lo;
    DL.c_lo = pl.c_lo;
    D.nc = DL.nc_own;
    D.agg = dalloc<int32_t>(c, DL.n_own);  // parents
    CK(cudaMemcpy(D.agg, pl.parent.data(), sizeof(int32_t) * pl.parent.size(), cudaMemcpyHostToDevice));
    std::vector<int2> mem(static_cast<size_t>(DL.nc_own));
    for (size_t q = 0; q < mem.size(); ++q) mem[q] = make_int2(pl.mem0[q], pl.mem1[q]);
    D.mem = dalloc<int2>(c, std::max<int64_t>(DL.nc_own, 1));
    CK(cudaMemcpy(D.mem, mem.data(), sizeof(int2) * mem.size(), cudaMemcpyHostToDevice));
    D.t = dalloc<double>(c, DL.wb + DL.n_ext) + DL.wb;  // own row 0 at the returned pointer
    D.x = dalloc<double>(c, DL.wb + DL.n_ext) + DL.wb;
    D.f = dalloc<double>(c, DL.n_own);
    DL.rg = dalloc<double>(c, std::max<int64_t>(static_cast<int64_t>(pl.rghost_glob.size()), 1));
    DL.xcg = dalloc<double>(c, std::max<int64_t>(static_cast<int64_t>(pl.xcghost_glob.size()), 1));
    {  // interior rows: a contiguous block whose columns are all own rows and
       // that no peer reads (P2P gathers read the sender's vector while the
       // interior of the next sweep is written; row pairs)
        const HostCsr &A = pl.A;
        const int64_t n = A.n;
        std::vector<char> sent(static_cast<size_t>(n), 0);
        for (int32_t i : pl.halo.send_idx)
            if (i >= 0 && i < n) sent[static_cast<size_t>(i)] = 1;
        auto ghosty = [&](int64_t i) {
            if (sent[static_cast<size_t>(i)]) return true;
            for (int64_t e = A.rp[i]; e < A.rp[i + 1]; ++e)
                if (A.ci[e] < 0 || A.ci[e] >= n) return true;
            return false;
        };
        int64_t lo = 0, hi = n;
        while (lo < n && ghosty(lo)) ++lo;
        while (hi > lo && ghosty(hi - 1)) --hi;
        bool ok = hi - lo >= 1024;
        for (int64_t i = lo; ok && i < hi; ++i) ok = !ghosty(i);
        lo = (lo + 1) / 2;  // pairs fully inside [lo, hi)
        hi = hi / 2;
        DL.q_ilo = ok ? lo : 0;
        DL.q_ihi = ok ? hi : 0;
    }
    DL.halo = upload_exch(c, pl.halo);
    DL.rx = upload_exch(c, pl.rx);
    DL.px = upload_exch(c, pl.px);
    DL.gather_lo = pl.gather_lo;
}

// ---- collectives ---------------------------------------------------------------------

static void barrier_local(sb_dist d) {
    for (auto &r : d->R) CK(cudaEventRecord(r.done, r.s));
    for (auto &r : d->R)
        for (auto &q : d->R)
            if (&q != &r) CK(cudaStreamWaitEvent(r.s, q.done, 0));
}

// P2P: publish this rank's epoch, then wait until every rank reached it (the
// producers' writes are visible; no rank can overwrite a buffer a peer still
// reads, because every rank publishes only after its previous gathers)
static void p2p_publish(sb_dist d) {
    for (auto &r : d->R) launch_k(r.c, k_p2p_publish, dim3(1), dim3(1), 0, r.s, r.epoch);
}
static void p2p_wait(sb_dist d) {
    for (auto &r : d->R)
        launch_k(r.c, k_p2p_wait, dim3(1), dim3(32), 0, r.s, static_cast<const unsigned long long *>(r.epoch),
                 static_cast<const unsigned long long *const *>(r.peer_epochs), d->nranks);
}
static void p2p_sync(sb_dist d) {
    p2p_publish(d);
    p2p_wait(d);
}

// Fill the ghost entries of every rank r from own(q) of its peers q, per the
// level-k plan `which`: chunk j of r lands at dst(r) + recv_dst[j] (halo: dst
// is the own-rows pointer of the x vector; rx / px: the packed ghost buffers).
static void exchange(sb_dist d, int k, int which, const std::function<const double *(RankDev &)> &own,
                     const std::function<double *(RankDev &)> &ghost, bool skip_sync = false) {
    auto plan = [&](RankDev &r) -> DevExch & {
        DistLevel &L = r.D[static_cast<size_t>(k)];
        return which == 0 ? L.halo : which == 1 ? L.rx : L.px;
    };
    if (d->p2p) {
        if (!skip_sync) p2p_sync(d);
        for (auto &r : d->R) {
            DevExch &e = plan(r);
            if (e.recv_peers.empty()) continue;
            const int id = r.buf_id.at(own(r));
            const int32_t *src = r.src_idx[static_cast<size_t>(k)][static_cast<size_t>(which)];
            for (size_t j = 0; j < e.recv_peers.size(); ++j) {
                const int64_t cnt = e.recv_off[j + 1] - e.recv_off[j];
                if (!cnt) continue;
                launch_k(r.c, k_p2p_gather, dim3(vec_grid(cnt)), dim3(kVecThreads), 0, r.s, cnt,
                         r.peer_own[static_cast<size_t>(id)][static_cast<size_t>(e.recv_peers[j])],
                         src + e.recv_off[j], ghost(r) + e.recv_dst[j]);
            }
        }
        return;
    }
    if (d->local) {
        for (auto &r : d->R) CK(cudaEventRecord(r.ready, r.s));
        for (auto &r : d->R) {
            DevExch &e = plan(r);
            for (size_t j = 0; j < e.recv_peers.size(); ++j) {
                RankDev &q = d->R[static_cast<size_t>(e.recv_peers[j])];
                DevExch &eq = plan(q);
                size_t jj = 0;
                while (jj < eq.send_peers.size() && eq.send_peers[jj] != r.rank) ++jj;
                if (jj == eq.send_peers.size()) throw runtime_error("exchange: inconsistent plans");
                const int64_t cnt = e.recv_off[j + 1] - e.recv_off[j];
                CK(cudaStreamWaitEvent(r.s, q.ready, 0));
                launch_k(r.c, k_gather_idx, dim3(vec_grid(cnt)), dim3(kVecThreads), 0, r.s, cnt, own(q),
                         static_cast<const int32_t *>(eq.send_idx + eq.send_off[jj]), ghost(r) + e.recv_dst[j]);
            }
        }
        barrier_local(d);
        return;
    }
    RankDev &r = d->R[0];
    DevExch &e = plan(r);
    if (e.nsend == 0 && e.nrecv == 0) return;
    cudaStream_t s = r.s;
    if (e.nsend)
        launch_k(r.c, k_gather_idx, dim3(vec_grid(e.nsend)), dim3(kVecThreads), 0, s, e.nsend, own(r),
                 static_cast<const int32_t *>(e.send_idx), e.sendbuf);
    NC(nccl().GroupStart());
    for (size_t j = 0; j < e.send_peers.size(); ++j)
        NC(nccl().Send(e.sendbuf + e.send_off[j], static_cast<size_t>(e.send_off[j + 1] - e.send_off[j]), ncclFloat64,
                       e.send_peers[j], d->comm, s));
    for (size_t j = 0; j < e.recv_peers.size(); ++j)
        NC(nccl().Recv(ghost(r) + e.recv_dst[j], static_cast<size_t>(e.recv_off[j + 1] - e.recv_off[j]), ncclFloat64,
                       e.recv_peers[j], d->comm, s));
    NC(nccl().GroupEnd());
}

// every rank ends with the whole vector v(r) whose piece [b[q], b[q+1]) rank q owns
static void allgatherv(sb_dist d, const std::vector<int64_t> &b, const std::function<double *(RankDev &)> &v) {
    if (d->p2p) {
        p2p_sync(d);
        for (auto &r : d->R) {
            const int id = r.buf_id.at(v(r));
            for (int q = 0; q < d->nranks; ++q) {
                const int64_t cnt = b[q + 1] - b[q];
                if (q == r.rank || cnt == 0) continue;
                launch_k(r.c, k_p2p_copy, dim3(vec_grid(cnt)), dim3(kVecThreads), 0, r.s, cnt,
                         r.peer_own[static_cast<size_t>(id)][static_cast<size_t>(q)] + b[q], v(r) + b[q]);
            }
        }
        return;
    }
    if (d->local) {
        for (auto &r : d->R) CK(cudaEventRecord(r.ready, r.s));
        for (auto &r : d->R)
            for (auto &q : d->R) {
                if (&q == &r || b[q.rank + 1] == b[q.rank]) continue;
                CK(cudaStreamWaitEvent(r.s, q.ready, 0));
                CK(cudaMemcpyAsync(v(r) + b[q.rank], v(q) + b[q.rank],
                                   sizeof(double) * static_cast<size_t>(b[q.rank + 1] - b[q.rank]),
                                   cudaMemcpyDeviceToDevice, r.s));
            }
        barrier_local(d);
        return;
    }
    RankDev &r = d->R[0];
    NC(nccl().GroupStart());
    for (int q = 0; q < d->nranks; ++q) {
        if (q == r.rank) continue;
        if (b[r.rank + 1] > b[r.rank])
            NC(nccl().Send(v(r) + b[r.rank], static_cast<size_t>(b[r.rank + 1] - b[r.rank]), ncclFloat64, q, d->comm,
                           r.s));
        if (b[q + 1] > b[q])
            NC(nccl().Recv(v(r) + b[q], static_cast<size_t>(b[q + 1] - b[q]), ncclFloat64, q, d->comm, r.s));
    }
    NC(nccl().GroupEnd());
}

// st->red = sum over ranks of st->part; then the scalar logic `op` on every rank
static void allreduce_logic(sb_dist d, int op, CondSet cs = CondSet{{0, 0}, 0}) {
    if (d->p2p) {
        for (auto &r : d->R)
            launch_k(r.c, k_p2p_put, dim3(1), dim3(1), 0, r.s, static_cast<const double *>(r.c->st->part), r.pslots,
                     static_cast<const int *>(r.pslot));
        p2p_sync(d);
        for (auto &r : d->R)
            launch_k(r.c, k_p2p_sum, dim3(1), dim3(1), 0, r.s, static_cast<const double *const *>(r.peer_slots),
                     d->nranks, r.pslot, r.c->st->red);
    } else if (d->local) {
        for (auto &r : d->R) CK(cudaEventRecord(r.ready, r.s));
        for (auto &r : d->R) {
            for (auto &q : d->R)
                if (&q != &r) CK(cudaStreamWaitEvent(r.s, q.ready, 0));
            launch_k(r.c, k_sum_partials, dim3(1), dim3(1), 0, r.s,
                     static_cast<const double *const *>(r.part_ptrs), d->nranks, r.c->st->red);
        }
        barrier_local(d);
    } else {
        RankDev &r = d->R[0];
        NC(nccl().AllReduce(r.c->st->part, r.c->st->red, 2, ncclFloat64, ncclSum, d->comm, r.s));
    }
    for (auto &r : d->R) launch_k(r.c, k_logic, dim3(1), dim3(1), 0, r.s, r.c->st, op, cs);
}

static Red red_partial(sb_ctx c, int nval, const double *w0 = nullptr, const double *w1 = nullptr) {
    return make_red(c, EP_PARTIAL, nval, w0, w1);
}

// ---- distributed V-cycle ------------------------------------------------------------------

// One V-cycle from level k with per-rank rhs f(r) and output X(r) (own rows;
// X has room for ghosts). Bitwise equal to the single-GPU cycle.
static void dist_vcycle(sb_dist d, const Cyc &cp, int k, const std::vector<const double *> &f,
                        const std::vector<double *> &X, bool zero) {
    const size_t N = d->R.size();
    if (k >= d->fr) {
        for (size_t i = 0; i < N; ++i) emit_vcycle(d->R[i].c, d->R[i].s, cp, k, f[i], X[i], zero);
        return;
    }
    std::vector<double *> cur(N), oth(N);
    auto lev = [&](size_t i) -> DevLevel & { return d->R[i].c->L[static_cast<size_t>(k)]; };
    auto dl = [&](size_t i) -> DistLevel & { return d->R[i].D[static_cast<size_t>(k)]; };
    auto halo = [&](std::vector<double *> &v) {
        std::vector<double *> vv = v;
        exchange(d, k, 0, [&](RankDev &r) -> const double * { return vv[static_cast<size_t>(&r - d->R.data())]; },
                 [&](RankDev &r) { return vv[static_cast<size_t>(&r - d->R.data())]; });
    };
    auto sweep = [&]() {
        for (size_t i = 0; i < N; ++i) launch_jacobi(d->R[i].c, lev(i), d->R[i].s, cur[i], f[i], oth[i], cp.omega);
        std::swap(cur, oth);
    };
    // halo exchange + sweep. A rank whose level has an interior block of row
    // pairs (no ghost column) sweeps it on its stream while the exchange runs
    // on the side stream, then sweeps the edge rows once the ghosts are in.
    static const bool overlap_env = [] {
        const char *e = std::getenv("SB_DIST_OVERLAP");
        return !(e && std::atoi(e) == 0);
    }();
    auto can_overlap = [&](size_t i) {
        return overlap_env && dl(i).q_ihi > dl(i).q_ilo && cross_range_ok(lev(i), cur[i], f[i], oth[i]);
    };
    auto halo_sweep = [&]() {
        bool any = false;
        for (size_t i = 0; i < N; ++i) any = any || can_overlap(i);
        if (!any) {
            halo(cur);
            sweep();
            return;
        }
        if (d->p2p) {
            // peer memory: publish, sweep the interior (the peers catch up
            // meanwhile), then wait, gather the ghosts, sweep the edge rows
            p2p_publish(d);
            for (size_t i = 0; i < N; ++i)
                if (can_overlap(i))
                    launch_jacobi_range(d->R[i].c, lev(i), d->R[i].s, cur[i], f[i], oth[i], cp.omega, dl(i).q_ilo,
                                        dl(i).q_ihi);
            p2p_wait(d);
            std::vector<double *> vv = cur;
            exchange(d, k, 0, [&](RankDev &r) -> const double * { return vv[static_cast<size_t>(&r - d->R.data())]; },
                     [&](RankDev &r) { return vv[static_cast<size_t>(&r - d->R.data())]; }, true);
        } else if (tl_eager) {
            // (eager launches only) the exchange on the side stream while the
            // interior is swept on the rank's stream
            std::vector<cudaStream_t> main(N);
            for (size_t i = 0; i < N; ++i) {
                RankDev &r = d->R[i];
                main[i] = r.s;
                CK(cudaEventRecord(r.ev_fork, r.s));
                CK(cudaStreamWaitEvent(r.s2, r.ev_fork, 0));
                if (can_overlap(i))
                    launch_jacobi_range(r.c, lev(i), r.s, cur[i], f[i], oth[i], cp.omega, dl(i).q_ilo, dl(i).q_ihi);
                r.s = r.s2;
            }
            halo(cur);  // on the side streams
            for (size_t i = 0; i < N; ++i) {
                RankDev &r = d->R[i];
                CK(cudaEventRecord(r.ev_join, r.s2));
                r.s = main[i];
                CK(cudaStreamWaitEvent(r.s, r.ev_join, 0));
            }
        } else {
            halo(cur);
            sweep();
            return;
        }
        for (size_t i = 0; i < N; ++i) {
            RankDev &r = d->R[i];
            if (can_overlap(i)) {
                const int64_t np = lev(i).n / 2;
                launch_jacobi_range(r.c, lev(i), r.s, cur[i], f[i], oth[i], cp.omega, 0, dl(i).q_ilo);
                launch_jacobi_range(r.c, lev(i), r.s, cur[i], f[i], oth[i], cp.omega, dl(i).q_ihi, np);
            } else {
                launch_jacobi(r.c, lev(i), r.s, cur[i], f[i], oth[i], cp.omega);
            }
        }
        std::swap(cur, oth);
    };
    for (size_t i = 0; i < N; ++i) {
        cur[i] = X[i];
        oth[i] = lev(i).t;
    }
    if (zero) {
        if (cp.pre >= 1) {
            for (size_t i = 0; i < N; ++i)
                launch_k(d->R[i].c, k_jacobi_zero, dim3(vec_grid(dl(i).n_own)), dim3(kVecThreads), 0,
                         d->R[i].s, dl(i).n_own, f[i], static_cast<const double *>(lev(i).diag), cur[i],
                         cp.omega);
            for (int s = 1; s < cp.pre; ++s) halo_sweep();
        } else {
            for (size_t i = 0; i < N; ++i)
                CK(cudaMemsetAsync(cur[i], 0, sizeof(double) * static_cast<size_t>(dl(i).n_own), d->R[i].s));
        }
    } else {
        for (int s = 0; s < cp.pre; ++s) halo_sweep();
    }
    // residual, partner residuals, restriction. A rank whose aggregates are all
    // local (no straddling pair: no rx plan; every BASELINE grid at plane-aligned
    // splits) runs the single-GPU fused residual + restriction kernel
    // (k_pat_resid_restrict: no r vector) when the coarse level is partitioned too.
    halo(cur);
    const bool next_rep = k + 1 >= d->fr;
    auto fused_rr = [&](size_t i) {
        const DistLevel &L = dl(i);
        return !next_rep && lev(i).pat && L.rx.nsend == 0 && L.rx.nrecv == 0;
    };
    for (size_t i = 0; i < N; ++i) {
        if (fused_rr(i)) continue;
        launch_csr<M_RESID, 0>(d->R[i].c, lev(i), d->R[i].s, cur[i], f[i], d->R[i].c->rs, 0.0, nullptr,
                               Red{});
    }
    exchange(d, k, 1, [&](RankDev &r) -> const double * { return r.c->rs; },
             [&](RankDev &r) { return r.D[static_cast<size_t>(k)].rg; });
    for (size_t i = 0; i < N; ++i) {
        DevLevel &lc = d->R[i].c->L[static_cast<size_t>(k) + 1];
        if (fused_rr(i)) {
            launch_pat_rr(d->R[i].c, lev(i), lc, d->R[i].s, cur[i], f[i], nullptr, cp.omega);
            continue;
        }
        double *out = next_rep ? lc.f + dl(i).c_lo : lc.f;
        launch_k(d->R[i].c, k_restrict_dist, dim3(vec_grid(dl(i).nc_own)), dim3(kVecThreads), 0, d->R[i].s,
                 dl(i).nc_own, static_cast<const int2 *>(lev(i).mem), static_cast<const double *>(d->R[i].c->rs),
                 static_cast<const double *>(dl(i).rg), dl(i).n_own, out);
    }
    if (next_rep)
        allgatherv(d, dl(0).gather_lo, [&](RankDev &r) { return r.c->L[static_cast<size_t>(k) + 1].f; });
    std::vector<const double *> fc(N);
    std::vector<double *> xc(N);
    for (size_t i = 0; i < N; ++i) {
        fc[i] = d->R[i].c->L[static_cast<size_t>(k) + 1].f;
        xc[i] = d->R[i].c->L[static_cast<size_t>(k) + 1].x;
    }
    dist_vcycle(d, cp, k + 1, fc, xc, true);
    if (!next_rep)
        exchange(d, k, 2, [&](RankDev &r) -> const double * { return r.c->L[static_cast<size_t>(k) + 1].x; },
                 [&](RankDev &r) { return r.D[static_cast<size_t>(k)].xcg; });
    std::vector<double *> pout(N);
    for (size_t i = 0; i < N; ++i) {
        pout[i] = (cp.post % 2 == 0) ? X[i] : lev(i).t;
        const int64_t ncown = next_rep ? (int64_t(1) << 62) : dl(i).nc_own;
        launch_k(d->R[i].c, k_prolong_dist, dim3(vec_grid(dl(i).n_own)), dim3(kVecThreads), 0, d->R[i].s,
                 dl(i).n_own, static_cast<const int32_t *>(lev(i).agg), static_cast<const double *>(cur[i]),
                 static_cast<const double *>(xc[i]), static_cast<const double *>(dl(i).xcg), ncown, pout[i]);
        cur[i] = pout[i];
        oth[i] = (pout[i] == X[i]) ? lev(i).t : X[i];
    }
    for (int s = 0; s < cp.post; ++s) halo_sweep();
}

// ---- distributed Krylov drivers -------------------------------------------------------------
// The control flow of build_pcg / build_bicg (conditional nodes driven by the
// scalar logic, every condition = !st->done), expressed once: with one rank
// per process (NCCL) the whole solve is captured as ONE CUDA graph (the NCCL
// calls are captured with it) and launched once; with in-process virtual
// ranks it runs eagerly with host-side evaluation of each condition (tl_eager).

static void dist_halo_vec(sb_dist d, int kv) {
    exchange(d, 0, 0, [&](RankDev &r) -> const double * { return r.c->kv[kv]; },
             [&](RankDev &r) { return r.c->kv[kv]; });
}

// conditional region: the body is emitted on rank 0's body stream when capturing
static void dist_cond(sb_dist d, int depth, cudaGraphConditionalHandle h, cudaGraphConditionalNodeType type,
                      const std::function<void(int)> &body) {
    RankDev &r0 = d->R[0];
    add_cond(r0.c, r0.s, depth, h, type, [&](cudaStream_t sb, int d2) {
        const cudaStream_t saved = r0.s;
        if (!tl_eager) r0.s = sb;
        body(d2);
        r0.s = saved;
    });
}

// vectors: KX x, KR r, KZ z, KP p, KAP Ap, KB b (own rows; x / p / pt / st with ghost room)
static void dist_pcg(sb_dist d, const Cyc *cp) {
    const size_t N = d->R.size();
    sb_ctx c0 = d->R[0].c;
    int mark = c0->launch_count;
    auto plan = [&](int &field) {  // graph mode: rank 0's kernels emitted since the last mark
        if (!tl_eager) field = c0->launch_count - mark;
        mark = c0->launch_count;
    };
    auto each = [&](const std::function<void(RankDev &, int64_t)> &fn) {
        for (auto &r : d->R) fn(r, r.D[0].n_own);
    };
    auto precond = [&](int in, int out) {
        if (cp) {
            std::vector<const double *> f(N);
            std::vector<double *> X(N);
            for (size_t i = 0; i < N; ++i) {
                f[i] = d->R[i].c->kv[in];
                X[i] = d->R[i].c->kv[out];
            }
            dist_vcycle(d, *cp, 0, f, X, true);
        } else {
            each([&](RankDev &r, int64_t n) {
                CK(cudaMemcpyAsync(r.c->kv[out], r.c->kv[in], sizeof(double) * n, cudaMemcpyDeviceToDevice, r.s));
            });
        }
    };
    each([&](RankDev &r, int64_t n) {
        launch_k(r.c, k_init, dim3(vec_grid(n)), dim3(kVecThreads), 0, r.s, n,
                 static_cast<const double *>(r.c->kv[KB]), r.c->kv[KX], r.c->kv[KR], red_partial(r.c, 1));
    });
    cudaGraphConditionalHandle h_pro = new_handle(d->R[0].s);
    allreduce_logic(d, EP_INIT_NORM, conds({h_pro}));
    plan(c0->plan.pre);
    dist_cond(d, 0, h_pro, cudaGraphCondTypeIf, [&](int d1) {
        precond(KR, KZ);
        each([&](RankDev &r, int64_t n) {
            launch_k(r.c, k_copy_dot, dim3(vec_grid(n)), dim3(kVecThreads), 0, r.s, n,
                     static_cast<const double *>(r.c->kv[KZ]), r.c->kv[KP], static_cast<double *>(nullptr),
                     static_cast<const double *>(r.c->kv[KR]), red_partial(r.c, 1), X0{});
        });
        cudaGraphConditionalHandle h_loop = new_handle(d->R[0].s);
        allreduce_logic(d, EP_PCG_RZ0, conds({h_loop}));
        plan(c0->plan.once);
        dist_cond(d, d1, h_loop, cudaGraphCondTypeWhile, [&](int d2) {
            dist_halo_vec(d, KP);
            each([&](RankDev &r, int64_t) {
                launch_csr<M_SPMV, 1>(r.c, r.c->L[0], r.s, r.c->kv[KP], nullptr, r.c->kv[KAP], 0.0, nullptr,
                                      red_partial(r.c, 1, r.c->kv[KP]));
            });
            allreduce_logic(d, EP_PCG_PAP);
            each([&](RankDev &r, int64_t n) {
                launch_k(r.c, k_pcg_update, dim3(vec_grid(n)), dim3(kVecThreads), 0, r.s, n, r.c->kv[KX],
                         r.c->kv[KR], static_cast<const double *>(r.c->kv[KP]),
                         static_cast<const double *>(r.c->kv[KAP]), red_partial(r.c, 1), X0{});
            });
            cudaGraphConditionalHandle h_vc = new_handle(d->R[0].s);
            allreduce_logic(d, EP_PCG_RN, conds({h_vc, h_loop}));
            plan(c0->plan.per_it);
            dist_cond(d, d2, h_vc, cudaGraphCondTypeIf, [&](int) {
                precond(KR, KZ);
                each([&](RankDev &r, int64_t n) {
                    launch_k(r.c, k_dot, dim3(vec_grid(n)), dim3(kVecThreads), 0, r.s, n,
                             static_cast<const double *>(r.c->kv[KR]), static_cast<const double *>(r.c->kv[KZ]),
                             static_cast<const int *>(nullptr), red_partial(r.c, 1));
                });
                allreduce_logic(d, EP_PCG_RZ);
                each([&](RankDev &r, int64_t n) {
                    launch_k(r.c, k_xpay, dim3(vec_grid(n)), dim3(kVecThreads), 0, r.s, n,
                             static_cast<const double *>(r.c->kv[KZ]), r.c->kv[KP],
                             static_cast<const DevState *>(r.c->st));
                });
                plan(c0->plan.per_it_cond);
            });
        });
    });
    // true residual
    dist_halo_vec(d, KX);
    each([&](RankDev &r, int64_t) {
        launch_csr<M_RESID, 1>(r.c, r.c->L[0], r.s, r.c->kv[KX], r.c->kv[KB], r.c->rs, 0.0, nullptr,
                               red_partial(r.c, 1));
    });
    allreduce_logic(d, EP_STORE);
    plan(c0->plan.post);
}

static void dist_bicg(sb_dist d, const Cyc *cp) {
    const size_t N = d->R.size();
    sb_ctx c0 = d->R[0].c;
    int mark = c0->launch_count;
    auto plan = [&](int &field) {  // graph mode: rank 0's kernels emitted since the last mark
        if (!tl_eager) field = c0->launch_count - mark;
        mark = c0->launch_count;
    };
    auto each = [&](const std::function<void(RankDev &, int64_t)> &fn) {
        for (auto &r : d->R) fn(r, r.D[0].n_own);
    };
    auto precond = [&](int in, int out) {
        if (cp) {
            std::vector<const double *> f(N);
            std::vector<double *> X(N);
            for (size_t i = 0; i < N; ++i) {
                f[i] = d->R[i].c->kv[in];
                X[i] = d->R[i].c->kv[out];
            }
            dist_vcycle(d, *cp, 0, f, X, true);
        } else {
            each([&](RankDev &r, int64_t n) {
                CK(cudaMemcpyAsync(r.c->kv[out], r.c->kv[in], sizeof(double) * n, cudaMemcpyDeviceToDevice, r.s));
            });
        }
    };
    each([&](RankDev &r, int64_t n) {
        launch_k(r.c, k_init, dim3(vec_grid(n)), dim3(kVecThreads), 0, r.s, n,
                 static_cast<const double *>(r.c->kv[KB]), r.c->kv[KX], r.c->kv[KR], red_partial(r.c, 1));
    });
    cudaGraphConditionalHandle h_pro = new_handle(d->R[0].s);
    allreduce_logic(d, EP_INIT_NORM, conds({h_pro}));
    plan(c0->plan.pre);
    dist_cond(d, 0, h_pro, cudaGraphCondTypeIf, [&](int d1) {
        each([&](RankDev &r, int64_t n) {
            launch_k(r.c, k_copy_dot, dim3(vec_grid(n)), dim3(kVecThreads), 0, r.s, n,
                     static_cast<const double *>(r.c->kv[KR]), r.c->kv[KRBAR], r.c->kv[KP],
                     static_cast<const double *>(r.c->kv[KR]), red_partial(r.c, 1), X0{});
        });
        cudaGraphConditionalHandle h_loop = new_handle(d->R[0].s);
        allreduce_logic(d, EP_BI_RHO0, conds({h_loop}));
        plan(c0->plan.once);
        dist_cond(d, d1, h_loop, cudaGraphCondTypeWhile, [&](int d2) {
            precond(KP, KPT);
            dist_halo_vec(d, KPT);
            each([&](RankDev &r, int64_t) {
                launch_csr<M_SPMV, 1>(r.c, r.c->L[0], r.s, r.c->kv[KPT], nullptr, r.c->kv[KAPT], 0.0, nullptr,
                                      red_partial(r.c, 1, r.c->kv[KRBAR]));
            });
            allreduce_logic(d, EP_BI_DENOM);
            each([&](RankDev &r, int64_t n) {
                launch_k(r.c, k_bi_s, dim3(vec_grid(n)), dim3(kVecThreads), 0, r.s, n,
                         static_cast<const double *>(r.c->kv[KR]), static_cast<const double *>(r.c->kv[KAPT]),
                         r.c->kv[KS], red_partial(r.c, 1), X0{});
            });
            cudaGraphConditionalHandle h_v2 = new_handle(d->R[0].s);
            allreduce_logic(d, EP_BI_SN, conds({h_v2}));
            each([&](RankDev &r, int64_t n) {
                launch_k(r.c, k_bi_half, dim3(vec_grid(n)), dim3(kVecThreads), 0, r.s, n, r.c->kv[KX],
                         static_cast<const double *>(r.c->kv[KPT]), static_cast<const DevState *>(r.c->st));
            });
            plan(c0->plan.per_it);
            dist_cond(d, d2, h_v2, cudaGraphCondTypeIf, [&](int) {
                precond(KS, KST);
                dist_halo_vec(d, KST);
                each([&](RankDev &r, int64_t) {
                    launch_csr<M_SPMV, 2>(r.c, r.c->L[0], r.s, r.c->kv[KST], nullptr, r.c->kv[KAST], 0.0, nullptr,
                                          red_partial(r.c, 2, nullptr, r.c->kv[KS]));
                });
                allreduce_logic(d, EP_BI_AS);
                each([&](RankDev &r, int64_t n) {
                    launch_k(r.c, k_bi_update, dim3(vec_grid(n)), dim3(kVecThreads), 0, r.s, n, r.c->kv[KX],
                             r.c->kv[KR], static_cast<const double *>(r.c->kv[KPT]),
                             static_cast<const double *>(r.c->kv[KST]), static_cast<const double *>(r.c->kv[KS]),
                             static_cast<const double *>(r.c->kv[KAST]), static_cast<const double *>(r.c->kv[KRBAR]),
                             red_partial(r.c, 2));
                });
                allreduce_logic(d, EP_BI_RN_RHO);
                each([&](RankDev &r, int64_t n) {
                    launch_k(r.c, k_bi_p, dim3(vec_grid(n)), dim3(kVecThreads), 0, r.s, n,
                             static_cast<const double *>(r.c->kv[KR]), r.c->kv[KP],
                             static_cast<const double *>(r.c->kv[KAPT]), static_cast<const DevState *>(r.c->st), X0{});
                });
                plan(c0->plan.per_it_cond);
            });
            // the loop condition after the iteration (!done), as build_bicg's k_set_cond
            RankDev &r0 = d->R[0];
            k_set_cond<<<1, 1, 0, r0.s>>>(r0.c->st, conds({h_loop}));
            CK(cudaGetLastError());
            ++r0.c->launch_count;
            if (!tl_eager) ++c0->plan.per_it;
            mark = c0->launch_count;
        });
    });
    dist_halo_vec(d, KX);
    each([&](RankDev &r, int64_t) {
        launch_csr<M_RESID, 1>(r.c, r.c->L[0], r.s, r.c->kv[KX], r.c->kv[KB], r.c->rs, 0.0, nullptr,
                               red_partial(r.c, 1));
    });
    allreduce_logic(d, EP_STORE);
    plan(c0->plan.post);
}

// ---- construction ------------------------------------------------------------------------------

static void build_rank(sb_dist d, RankDev &R, const Hier &h, int rank, int64_t gather_rows,
                       const sb_device_opts &o) {
    R.rank = rank;
    R.P = build_partition(h, rank, d->nranks, gather_rows);
    d->fr = R.P.first_replicated;
    sb_ctx c = ctx_begin(o);
    R.c = c;
    const int L = static_cast<int>(h.levels.size());
    c->L.resize(static_cast<size_t>(L));
    R.D.resize(static_cast<size_t>(L));
    for (int k = 0; k < L; ++k) {
        if (k < d->fr) upload_dist_level(c, R.P.L[static_cast<size_t>(k)], c->L[static_cast<size_t>(k)], R.D[k]);
        else upload_level(c, h.levels[static_cast<size_t>(k)], c->L[static_cast<size_t>(k)], k + 1 == L, -1);
    }
    const int64_t nvec = d->fr > 0 ? R.D[0].n_ext : h.levels[0].A.n;
    if (d->fr == 0) R.D[0].n_own = R.D[0].n_ext = h.levels[0].A.n;
    R.lo = R.P.L[0].lo;
    R.hi = R.P.L[0].hi;
    ctx_finish(c, h, o, nvec, d->fr, d->fr > 0 ? R.D[0].wb : 0);
    R.s = c->stream;
    CK(cudaStreamCreateWithFlags(&R.s2, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&R.ev_fork, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&R.ev_join, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&R.ready, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&R.done, cudaEventDisableTiming));
}

// ---- peer-memory transport: buffers, plans, connection -----------------------------

static void *alloc_base(const void *p) {
    static PFN_cuMemGetAddressRange_v3020 range = [] {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q{};
        CK(cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q));
        if (q != cudaDriverEntryPointSuccess || !fn) throw cuda_error("cuMemGetAddressRange unavailable");
        return reinterpret_cast<PFN_cuMemGetAddressRange_v3020>(fn);
    }();
    CUdeviceptr base = 0;
    size_t size = 0;
    if (range(&base, &size, reinterpret_cast<CUdeviceptr>(p)) != CUDA_SUCCESS)
        throw cuda_error("cuMemGetAddressRange failed");
    return reinterpret_cast<void *>(base);
}

// The buffers peers read, in the same order on every rank (ids): the x / t
// vectors of every distributed level, the residual, the first replicated
// level's rhs, the Krylov vectors; then the partial-sum slots. Plus the epoch.
static void p2p_register(sb_dist d, RankDev &R) {
    sb_ctx c = R.c;
    R.epoch = dalloc<unsigned long long>(c, 1, false);
    R.pslots = dalloc<double>(c, 4, false);
    R.pslot = dalloc<int>(c, 1, false);
    auto reg = [&](const double *own) {
        if (!own) throw runtime_error("p2p_register: null buffer");
        if (R.buf_id.count(own)) throw runtime_error("p2p_register: buffer registered twice");
        R.buf_id[own] = static_cast<int>(R.exported.size());
        void *base = alloc_base(own);
        R.exported.push_back({base, reinterpret_cast<const char *>(own) - static_cast<const char *>(base)});
        R.exported_own.push_back(own);
    };
    const int L = static_cast<int>(c->L.size());
    for (int k = 0; k < d->fr; ++k) {
        reg(c->L[static_cast<size_t>(k)].x);
        reg(c->L[static_cast<size_t>(k)].t);
    }
    reg(c->rs);
    if (d->fr > 0 && d->fr < L) reg(c->L[static_cast<size_t>(d->fr)].f);
    for (double *v : c->kv) reg(v);
    reg(R.pslots);
}

// src_idx[k][which]: for each recv chunk of this rank's plan, the SENDING
// peer's own-row indices (its send list towards this rank), concatenated in
// recv order. parts(q) = rank q's host partition.
static void p2p_plans(RankDev &R, const std::function<const Partition &(int)> &parts) {
    R.src_idx.assign(R.D.size(), {nullptr, nullptr, nullptr});
    for (size_t k = 0; k < R.D.size(); ++k) {
        if (!R.D[k].dist) continue;
        for (int which = 0; which < 3; ++which) {
            const DistLevel &L = R.D[k];
            const DevExch &e = which == 0 ? L.halo : which == 1 ? L.rx : L.px;
            std::vector<int32_t> idx;
            for (size_t j = 0; j < e.recv_peers.size(); ++j) {
                const PartLevel &pl = parts(e.recv_peers[j]).L[k];
                const Exchange &x = which == 0 ? pl.halo : which == 1 ? pl.rx : pl.px;
                size_t jj = 0;
                while (jj < x.send_peers.size() && x.send_peers[jj] != R.rank) ++jj;
                if (jj == x.send_peers.size()) throw runtime_error("p2p: inconsistent exchange plans");
                const int64_t cnt = x.send_off[jj + 1] - x.send_off[jj];
                if (cnt != e.recv_off[j + 1] - e.recv_off[j]) throw runtime_error("p2p: plan size mismatch");
                idx.insert(idx.end(), x.send_idx.begin() + x.send_off[jj], x.send_idx.begin() + x.send_off[jj + 1]);
            }
            auto *dv = dalloc<int32_t>(R.c, std::max<int64_t>(static_cast<int64_t>(idx.size()), 1), false);
            if (!idx.empty())
                CK(cudaMemcpy(dv, idx.data(), sizeof(int32_t) * idx.size(), cudaMemcpyHostToDevice));
            R.src_idx[k][static_cast<size_t>(which)] = dv;
        }
    }
}

// device tables of every rank's epoch and partial slots, in rank order
static void p2p_tables(RankDev &R, const std::vector<const unsigned long long *> &epochs,
                       const std::vector<const double *> &slots) {
    R.h_peer_epochs = epochs;
    R.peer_epochs = dalloc<const unsigned long long *>(R.c, static_cast<int64_t>(epochs.size()), false);
    CK(cudaMemcpy(R.peer_epochs, epochs.data(), sizeof(void *) * epochs.size(), cudaMemcpyHostToDevice));
    R.peer_slots = dalloc<const double *>(R.c, static_cast<int64_t>(slots.size()), false);
    CK(cudaMemcpy(R.peer_slots, slots.data(), sizeof(void *) * slots.size(), cudaMemcpyHostToDevice));
}

static int run_dist(sb_dist d, SolveKind kind, const sb_cycle *cpa, const double *b, double *x, double tol,
                    int max_iters, sb_report *rep, bool device_ptrs) {
    // (graph mode: b and x are staged through the rank's own vectors, so the
    // captured graph does not depend on them)
    const auto t0 = std::chrono::steady_clock::now();
    const char *who = kind == K_PCG ? "pcg" : "pbicgstab";
    if (!(tol > 0.0)) throw invalid_argument(std::string(who) + ": tol must be > 0");
    if (d->p2p && !d->connected) throw invalid_argument(std::string(who) + ": P2P ranks not connected");
    Cyc cyc;
    const Cyc *cp = nullptr;
    if (cpa) {
        for (auto &r : d->R) cyc = check_cycle(r.c, cpa, who);
        cp = &cyc;
    }
    for (auto &r : d->R) {
        CK(cudaSetDevice(r.c->device));
        ensure_hist(r.c, std::max(max_iters, 0) + 2);
        DevState hs;
        std::memset(&hs, 0, sizeof(hs));
        hs.tol = tol;
        hs.max_iters = max_iters;
        hs.hist_cap = r.c->hist_cap;
        hs.hist_r = r.c->hist_r;
        hs.hist_t = r.c->hist_t;
        CK(cudaMemcpyAsync(r.c->st, &hs, sizeof(hs), cudaMemcpyHostToDevice, r.c->stream));
        // b: in-process mode takes the global vector, NCCL mode the rank's slice
        const double *src = d->local ? b + r.lo : b;
        CK(cudaMemcpyAsync(r.c->kv[KB], src, sizeof(double) * static_cast<size_t>(r.hi - r.lo),
                           device_ptrs ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, r.c->stream));
    }
    RankDev &r0 = d->R[0];
    for (auto &r : d->R) {
        r.c->launch_count = 0;
        r.s = r.c->stream;
    }
    for (auto &r : d->R) CK(cudaEventRecord(r.c->ev0, r.c->stream));
    // one rank per process: the whole solve as one graph (NCCL calls captured);
    // in-process ranks or use_graphs = 0: eager, host-evaluated conditions
    bool graph = d->R.size() == 1 && !d->local && r0.c->graphs && !d->graph_failed;
    if (graph) {
        const std::string key = key_of(kind == K_PCG ? "dist-pcg" : "dist-bicg", cp, nullptr, nullptr, r0.c->hist_r);
        auto it = d->cache.find(key);
        if (it == d->cache.end()) {
            GraphEntry e;
            r0.c->plan = LaunchPlan{};
            e.g = begin_capture(r0.c);
            try {
                if (kind == K_PCG) dist_pcg(d, cp);
                else dist_bicg(d, cp);
                end_capture(r0.c, e.g);
                CK(cudaGraphInstantiate(&e.exec, e.g, 0));
                e.plan = r0.c->plan;
                it = d->cache.emplace(key, e).first;
            } catch (const std::exception &ex) {
                // a transport that cannot be captured (e.g. a library inserting
                // host nodes into conditional bodies): run eagerly from now on
                cudaGraph_t dummy = nullptr;
                cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
                cudaStreamIsCapturing(r0.c->stream, &st);
                if (st != cudaStreamCaptureStatusNone) cudaStreamEndCapture(r0.c->stream, &dummy);
                if (dummy) cudaGraphDestroy(dummy);
                if (e.g) cudaGraphDestroy(e.g);
                cudaGetLastError();
                d->graph_failed = true;
                d->graph_error = ex.what();
                graph = false;
            }
        }
        if (graph) CK(cudaGraphLaunch(it->second.exec, r0.c->stream));
    }
    if (!graph) {
        tl_eager = true;
        try {
            if (kind == K_PCG) dist_pcg(d, cp);
            else dist_bicg(d, cp);
        } catch (...) {
            tl_eager = false;
            throw;
        }
        tl_eager = false;
    }
    for (auto &r : d->R) CK(cudaEventRecord(r.c->ev1, r.c->stream));
    DevState hs;
    for (auto &r : d->R) {
        double *dst = d->local ? x + r.lo : x;
        CK(cudaMemcpyAsync(dst, r.c->kv[KX], sizeof(double) * static_cast<size_t>(r.hi - r.lo),
                           device_ptrs ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, r.c->stream));
    }
    CK(cudaMemcpyAsync(&hs, r0.c->st, sizeof(hs), cudaMemcpyDeviceToHost, r0.c->stream));
    float ms_max = 0.f;
    for (auto &r : d->R) {
        CK(cudaStreamSynchronize(r.c->stream));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, r.c->ev0, r.c->ev1));
        ms_max = std::max(ms_max, ms);
    }
    d->last_ms = ms_max;
    d->last_launches = r0.c->launch_count;
    if (graph) {  // kernels the graph executed on this rank (LaunchPlan, as run_solve)
        const LaunchPlan &P = d->cache.begin()->second.plan;
        const bool entered = hs.iter > 0;
        const int skipped = kind == K_BICG ? hs.half : (hs.iter > 0 ? 1 : 0);
        d->last_launches = static_cast<int>(P.pre + P.post + (entered ? P.once : 0) + int64_t(hs.iter) * P.per_it +
                                            std::max<int64_t>(0, int64_t(hs.iter) - skipped) * P.per_it_cond);
    }
    if (rep) {
        rep->iterations = hs.iter;
        rep->termination = hs.term;
        rep->true_residual = hs.true_res;
        rep->hist_len = hs.iter + 1;
        const int m = std::min(rep->hist_len, std::max(rep->hist_cap, 0));
        if (m > 0 && rep->residual_history)
            CK(cudaMemcpy(rep->residual_history, r0.c->hist_r, sizeof(double) * m, cudaMemcpyDeviceToHost));
        if (m > 0 && rep->time_history)
            CK(cudaMemcpy(rep->time_history, r0.c->hist_t, sizeof(double) * m, cudaMemcpyDeviceToHost));
        rep->wall_time = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    }
    return SB_OK;
}

} // namespace sb

extern "C" {

int sb_nccl_unique_id(unsigned char *out) {
    return guard([&] {
        ncclUniqueId id;
        NC(nccl().GetUniqueId(&id));
        std::memcpy(out, id.internal, sizeof(id.internal));
    });
}

int sb_dist_create(sb_hier hh, int rank, int nranks, const unsigned char *nccl_id, int64_t gather_rows,
                   const sb_device_opts *opts, sb_dist *out) {
    sb_dist d = nullptr;
    const int rc = guard([&] {
        Hier *h = hier_of(hh);
        if (!h || !out || !nccl_id) throw invalid_argument("sb_dist_create: null argument");
        sb_device_opts o{0, 1, -1, 0};
        if (opts) o = *opts;
        d = new sb_dist_s;
        d->nranks = nranks;
        d->local = false;
        d->R.resize(1);
        build_rank(d, d->R[0], *h, rank, gather_rows, o);
        ncclUniqueId id;
        std::memcpy(id.internal, nccl_id, sizeof(id.internal));
        CK(cudaSetDevice(o.device));
        NC(nccl().CommInitRank(&d->comm, nranks, id, rank));
        *out = d;
    });
    if (rc != SB_OK && d) sb_dist_destroy(d);
    return rc;
}

int sb_dist_create_local(sb_hier hh, int nranks, int64_t gather_rows, const sb_device_opts *opts, sb_dist *out) {
    sb_dist d = nullptr;
    const int rc = guard([&] {
        Hier *h = hier_of(hh);
        if (!h || !out || nranks < 1) throw invalid_argument("sb_dist_create_local: bad argument");
        sb_device_opts o{0, 1, -1, 0};
        if (opts) o = *opts;
        d = new sb_dist_s;
        d->nranks = nranks;
        d->local = true;
        d->R.resize(static_cast<size_t>(nranks));
        for (int r = 0; r < nranks; ++r) build_rank(d, d->R[static_cast<size_t>(r)], *h, r, gather_rows, o);
        std::vector<double *> parts(static_cast<size_t>(nranks));
        for (int r = 0; r < nranks; ++r) parts[static_cast<size_t>(r)] = d->R[static_cast<size_t>(r)].c->st->part;
        for (auto &r : d->R) {
            r.part_ptrs = dalloc<double *>(r.c, nranks, false);
            CK(cudaMemcpy(r.part_ptrs, parts.data(), sizeof(double *) * parts.size(), cudaMemcpyHostToDevice));
        }
        *out = d;
    });
    if (rc != SB_OK && d) sb_dist_destroy(d);
    return rc;
}

// In-process ranks over the peer-memory transport (the peers' buffers are
// plain device pointers here): the P2P protocol and kernels on one GPU.
int sb_dist_create_local_p2p(sb_hier hh, int nranks, int64_t gather_rows, const sb_device_opts *opts,
                             sb_dist *out) {
    sb_dist d = nullptr;
    const int rc = guard([&] {
        Hier *h = hier_of(hh);
        if (!h || !out || nranks < 1) throw invalid_argument("sb_dist_create_local_p2p: bad argument");
        sb_device_opts o{0, 1, -1, 0};
        if (opts) o = *opts;
        d = new sb_dist_s;
        d->nranks = nranks;
        d->local = true;
        d->p2p = true;
        d->R.resize(static_cast<size_t>(nranks));
        for (int r = 0; r < nranks; ++r) build_rank(d, d->R[static_cast<size_t>(r)], *h, r, gather_rows, o);
        for (auto &r : d->R) p2p_register(d, r);
        std::vector<const unsigned long long *> ep;
        std::vector<const double *> sl;
        for (auto &q : d->R) {
            ep.push_back(q.epoch);
            sl.push_back(q.pslots);
        }
        for (auto &r : d->R) {
            p2p_plans(r, [&](int q) -> const Partition & { return d->R[static_cast<size_t>(q)].P; });
            p2p_tables(r, ep, sl);
            r.peer_own.assign(r.exported_own.size(), std::vector<const double *>(static_cast<size_t>(nranks)));
            for (size_t id = 0; id < r.exported_own.size(); ++id)
                for (int q = 0; q < nranks; ++q)
                    r.peer_own[id][static_cast<size_t>(q)] = d->R[static_cast<size_t>(q)].exported_own[id];
        }
        d->connected = true;
        *out = d;
    });
    if (rc != SB_OK && d) sb_dist_destroy(d);
    return rc;
}

// One rank per process over peer memory: create, export the IPC handles of the
// buffers peers read (sb_dist_p2p_export), exchange the blobs out of band (every
// rank needs every rank's), then sb_dist_p2p_connect with all of them in rank order.
int sb_dist_create_p2p(sb_hier hh, int rank, int nranks, int64_t gather_rows, const sb_device_opts *opts,
                       sb_dist *out) {
    sb_dist d = nullptr;
    const int rc = guard([&] {
        Hier *h = hier_of(hh);
        if (!h || !out || nranks < 1 || rank < 0 || rank >= nranks)
            throw invalid_argument("sb_dist_create_p2p: bad argument");
        sb_device_opts o{0, 1, -1, 0};
        if (opts) o = *opts;
        d = new sb_dist_s;
        d->nranks = nranks;
        d->local = false;
        d->p2p = true;
        d->R.resize(1);
        RankDev &R = d->R[0];
        build_rank(d, R, *h, rank, gather_rows, o);
        p2p_register(d, R);
        std::map<int, Partition> peers;  // the partitions of the ranks this rank receives from
        p2p_plans(R, [&](int q) -> const Partition & {
            if (q == rank) return R.P;
            auto it = peers.find(q);
            if (it == peers.end()) it = peers.emplace(q, build_partition(*h, q, nranks, gather_rows)).first;
            return it->second;
        });
        *out = d;
    });
    if (rc != SB_OK && d) sb_dist_destroy(d);
    return rc;
}

// blob: int32 count, then per exported buffer (ids in order, then the epoch):
// int64 own-row-0 offset + cudaIpcMemHandle_t
int sb_dist_p2p_export(sb_dist d, unsigned char *buf, int64_t cap, int64_t *len) {
    return guard([&] {
        if (!d || !d->p2p || d->local || !len) throw invalid_argument("sb_dist_p2p_export: not a P2P rank");
        RankDev &R = d->R[0];
        CK(cudaSetDevice(R.c->device));
        const int n = static_cast<int>(R.exported.size()) + 1;
        const int64_t need = 4 + static_cast<int64_t>(n) * (8 + static_cast<int64_t>(sizeof(cudaIpcMemHandle_t)));
        *len = need;
        if (!buf) return;
        if (cap < need) throw invalid_argument("sb_dist_p2p_export: buffer too small");
        std::memcpy(buf, &n, 4);
        unsigned char *p = buf + 4;
        for (int i = 0; i < n; ++i) {
            void *base = i + 1 < n ? R.exported[static_cast<size_t>(i)].first : static_cast<void *>(R.epoch);
            const int64_t off = i + 1 < n ? R.exported[static_cast<size_t>(i)].second : 0;
            cudaIpcMemHandle_t hnd;
            CK(cudaIpcGetMemHandle(&hnd, base));
            std::memcpy(p, &off, 8);
            std::memcpy(p + 8, &hnd, sizeof(hnd));
            p += 8 + sizeof(hnd);
        }
    });
}

int sb_dist_p2p_connect(sb_dist d, const unsigned char *blobs, int64_t len_each) {
    return guard([&] {
        if (!d || !d->p2p || d->local || !blobs) throw invalid_argument("sb_dist_p2p_connect: not a P2P rank");
        RankDev &R = d->R[0];
        CK(cudaSetDevice(R.c->device));
        const size_t nid = R.exported.size();
        R.peer_own.assign(nid, std::vector<const double *>(static_cast<size_t>(d->nranks)));
        std::vector<const unsigned long long *> ep(static_cast<size_t>(d->nranks));
        std::vector<const double *> sl(static_cast<size_t>(d->nranks));
        const int slot_id = R.buf_id.at(R.pslots);
        for (int q = 0; q < d->nranks; ++q) {
            if (q == R.rank) {
                for (size_t id = 0; id < nid; ++id) R.peer_own[id][static_cast<size_t>(q)] = R.exported_own[id];
                ep[static_cast<size_t>(q)] = R.epoch;
                sl[static_cast<size_t>(q)] = R.pslots;
                continue;
            }
            const unsigned char *p = blobs + static_cast<int64_t>(q) * len_each;
            int n = 0;
            std::memcpy(&n, p, 4);
            if (n != static_cast<int>(nid) + 1) throw invalid_argument("sb_dist_p2p_connect: blob of another layout");
            p += 4;
            for (int i = 0; i < n; ++i) {
                int64_t off = 0;
                cudaIpcMemHandle_t hnd;
                std::memcpy(&off, p, 8);
                std::memcpy(&hnd, p + 8, sizeof(hnd));
                p += 8 + sizeof(hnd);
                void *mp = nullptr;
                CK(cudaIpcOpenMemHandle(&mp, hnd, cudaIpcMemLazyEnablePeerAccess));
                R.opened.push_back(mp);
                const char *own = static_cast<const char *>(mp) + off;
                if (i + 1 < n) R.peer_own[static_cast<size_t>(i)][static_cast<size_t>(q)] = reinterpret_cast<const double *>(own);
                else ep[static_cast<size_t>(q)] = reinterpret_cast<const unsigned long long *>(own);
            }
            sl[static_cast<size_t>(q)] = R.peer_own[static_cast<size_t>(slot_id)][static_cast<size_t>(q)];
        }
        p2p_tables(R, ep, sl);
        d->connected = true;
    });
}

void sb_dist_destroy(sb_dist d) {
    if (!d) return;
    for (auto &r : d->R)
        for (void *p : r.opened) cudaIpcCloseMemHandle(p);
    for (auto &kv : d->cache) {
        if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
        if (kv.second.g) cudaGraphDestroy(kv.second.g);
    }
    if (d->comm) nccl().CommDestroy(d->comm);
    for (auto &r : d->R) {
        if (r.ready) cudaEventDestroy(r.ready);
        if (r.ev_fork) cudaEventDestroy(r.ev_fork);
        if (r.ev_join) cudaEventDestroy(r.ev_join);
        if (r.s2) cudaStreamDestroy(r.s2);
        if (r.done) cudaEventDestroy(r.done);
        if (r.c) sb_destroy(r.c);
    }
    delete d;
}

int sb_dist_rows(sb_dist d, int local_rank, int64_t *lo, int64_t *hi, int *first_replicated) {
    return guard([&] {
        if (!d || local_rank < 0 || local_rank >= static_cast<int>(d->R.size()))
            throw invalid_argument("sb_dist_rows: bad rank");
        *lo = d->R[static_cast<size_t>(local_rank)].lo;
        *hi = d->R[static_cast<size_t>(local_rank)].hi;
        if (first_replicated) *first_replicated = d->fr;
    });
}

int sb_dist_pcg(sb_dist d, const sb_cycle *cp, const double *b, double *x, double tol, int max_iters,
                sb_report *rep, int device_ptrs) {
    return guard([&] { run_dist(d, K_PCG, cp, b, x, tol, max_iters, rep, device_ptrs != 0); });
}

int sb_dist_pbicgstab(sb_dist d, const sb_cycle *cp, const double *b, double *x, double tol, int max_iters,
                      sb_report *rep, int device_ptrs) {
    return guard([&] { run_dist(d, K_BICG, cp, b, x, tol, max_iters, rep, device_ptrs != 0); });
}

int sb_dist_vcycle(sb_dist d, const sb_cycle *cpa, const double *f, double *x) {
    return guard([&] {
        Cyc cp;
        for (auto &r : d->R) cp = check_cycle(r.c, cpa, "vcycle");
        const size_t N = d->R.size();
        std::vector<const double *> fv(N);
        std::vector<double *> xv(N);
        for (size_t i = 0; i < N; ++i) {
            RankDev &r = d->R[i];
            CK(cudaSetDevice(r.c->device));
            const double *src = d->local ? f + r.lo : f;
            CK(cudaMemcpyAsync(r.c->kv[KB], src, sizeof(double) * static_cast<size_t>(r.hi - r.lo),
                               cudaMemcpyHostToDevice, r.s));
            fv[i] = r.c->kv[KB];
            xv[i] = r.c->kv[KZ];
        }
        dist_vcycle(d, cp, 0, fv, xv, true);
        for (size_t i = 0; i < N; ++i) {
            RankDev &r = d->R[i];
            double *dst = d->local ? x + r.lo : x;
            CK(cudaMemcpyAsync(dst, r.c->kv[KZ], sizeof(double) * static_cast<size_t>(r.hi - r.lo),
                               cudaMemcpyDeviceToHost, r.s));
        }
        for (auto &r : d->R) CK(cudaStreamSynchronize(r.s));
    });
}

double sb_dist_last_solve_ms(sb_dist d) { return d ? d->last_ms : 0.0; }
int sb_dist_last_launches(sb_dist d) { return d ? d->last_launches : 0; }

} // extern "C"
