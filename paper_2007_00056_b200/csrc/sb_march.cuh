// Plane-marching row-pattern sweep ("RPAT-M"), included by sb_runtime.cu after sb_rowpat.cuh.
//
// On a row-pattern level whose most frequent pattern is a 27-point box --
// offsets dz*P + dy*N + dx with dx, dy, dz in {-1, 0, 1}, P a multiple of N
// (every level of the 27-point hierarchies) -- rows are viewed
// as (plane q, line y, column c) with r = q*P + y*N + c. A CTA owns a tile of
// 8 lines x 32 columns (warp = line, lane = column) and marches it through K
// planes:
//  * the x values of each plane the tile touches (10 lines x 36 doubles: the
//    8 lines, one halo line either side, one halo column either side, rounded
//    out to 16 bytes) arrive in a shared-memory ring by asynchronous copies
//    (cp.async, 16 bytes per thread, completion counted on one mbarrier per
//    ring slot), issued up to D planes ahead and
//    streamed across the CTA's consecutive tiles, so HBM latency is hidden
//    without registers;
//  * every row keeps its gathered values in registers and rolls them by one
//    plane per step (three 9-value plane arrays rotated by identity over an
//    unrolled-by-3 loop), so a step reads only the 9 values of the plane that
//    enters the window from shared memory, and x_i is the window's centre.
// It was written against the row-pattern kernel's bound on 27-point levels (L1
// wavefronts of 27 x gathers per row, 90% of peak). Measured on B200 it cuts
// the L1 traffic 3x but is slower (27-point 256^3 L0 sweep 235 us vs 212 us):
// one row per thread leaves ~240 instructions per warp-step and a 27-long
// dependent DADD chain (the reference's summation order) with 16 warps/SM
// (124 registers), so it is issue/latency-bound. Opt-in (SB_MARCH=1), parity
// tested; DESIGN.md §3.3.
//
// Bit-exactness: the sum is sum_k v_k x[i + o_k] in slot (= CSR) order from 0.0
// with __dmul_rn/__dadd_rn (inc/csr.hpp:185-191). A row whose pattern is not
// the main one is "embedded" into the main slot order when its offsets are a
// subsequence of the main ones: absent slots carry +0.0 and
// sum + (+-0) == sum bit for bit (sum is never -0), unless the x read there is
// inf/NaN -- then the sum is not finite and the row is replayed exactly from its
// own pattern. Warps holding a non-embeddable row, tiles whose copies would
// leave [0, n), and the first and last planes run the plain per-row path.

constexpr int kMarchThreads = 256;  // 8 warps = 8 lines of a tile
constexpr int kMarchLines = kMarchThreads / 32;
#ifndef SB_MARCH_K
#define SB_MARCH_K 16
#endif
#ifndef SB_MARCH_D
#define SB_MARCH_D 16
#endif
constexpr int kMarchK = SB_MARCH_K;  // planes per tile
constexpr int kMarchD = SB_MARCH_D;  // ring slots (planes; a power of two): D - 3 staged ahead
constexpr int kLineW = 36;          // doubles per staged line (32 + halo, 16-byte rounded)
constexpr int kPlaneW = (kMarchLines + 2) * kLineW;  // doubles per staged plane
constexpr int kChunks = kPlaneW / 2;                 // 16-byte chunks per staged plane

// Slot geometry: W main slots in CSR order, centre C, (dz, dy, dx) of slot k,
// src(k): the slot of the previous plane's row holding slot k's value, or -1.
// (Only the box is instantiated; a 7-point cross variant measured slower too.)
template <int G> struct Geo;
template <> struct Geo<0> {  // 27-point box, slots in (dz, dy, dx) lexicographic order
    static constexpr int W = 27, C = 13;
    __host__ __device__ static constexpr int dz(int k) { return k / 9 - 1; }
    __host__ __device__ static constexpr int dy(int k) { return (k / 3) % 3 - 1; }
    __host__ __device__ static constexpr int dx(int k) { return k % 3 - 1; }
    __host__ __device__ static constexpr int src(int k) { return k < 18 ? k + 9 : -1; }
};

template <int W> struct MarchPat {
    double v[W];  // main pattern values (slot order)
    double d, r;  // a_ii, RN(1/a_ii)
    int p;        // main pattern id
    int P, N, NY; // plane stride, line stride, lines per plane (P / N)
    int nqf;      // full planes (n / P)
    int nxb, nyb, ntiles;
};

// march table (after the RPAT table in shared memory): f64 ev[np][WE] (each
// pattern's values placed at the main slots, +0.0 elsewhere) | uint8 emb[np]
__host__ __device__ __forceinline__ size_t march_table_bytes(int np, int w) {
    const size_t we = (w + 1) & ~1;
    return (static_cast<size_t>(np) * we * 8 + static_cast<size_t>(np) + 15) & ~size_t(15);
}
__host__ __device__ __forceinline__ size_t march_smem_bytes(size_t tb, size_t mtb) {
    return sizeof(double) * kMarchD * kPlaneW + 8 * kMarchD + tb + mtb;
}

// exact sum of pattern p's own slots (CSR order, no padding)
template <int WP>
__device__ __forceinline__ double wide_row_sum_masked(const SmemTab<WP> &T, int p, const double *__restrict__ xr) {
    double sum = 0.0;
    const int len = T.l(p);
    for (int k = 0; k < len; ++k) sum = __dadd_rn(sum, __dmul_rn(T.v(p, k), __ldg(xr + T.o(p, k))));
    return sum;
}

// tile t -> (first plane q0, planes kt, first line y0, first column x0); fast
// tiles stage planes q0 - 1 .. q0 + kt, every line copy inside [0, n_even)
template <int W> struct MarchTile {
    int q0, kt, y0, x0;
    bool fast;
    __device__ __forceinline__ MarchTile(const MarchPat<W> &m, int t, int n) {
        const int xb = t % m.nxb, r1 = t / m.nxb;
        const int yb = r1 % m.nyb, qb = r1 / m.nyb;
        x0 = xb * 32;
        y0 = yb * kMarchLines;
        q0 = 1 + qb * kMarchK;                      // plane 0 is done by the per-row pass
        kt = min(kMarchK, m.nqf - 1 - q0);           // planes >= nqf - 1 likewise
        const int64_t amin = static_cast<int64_t>(q0 - 1) * m.P + static_cast<int64_t>(y0 - 1) * m.N + x0 - 2;
        const int64_t amax = static_cast<int64_t>(q0 + kt) * m.P + static_cast<int64_t>(y0 + kMarchLines) * m.N + x0 +
                             kLineW;
        fast = kt > 0 && amin >= 0 && amax <= (n & ~1);
    }
};

template <int MODE>
__device__ __forceinline__ double march_out(double xi, double fi, double omega, double sum, double dg, double ry) {
    if constexpr (MODE == M_SPMV) return sum;
    else if constexpr (MODE == M_RESID) return __dsub_rn(fi, sum);
    else return __dadd_rn(xi, div_rn(__dmul_rn(omega, __dsub_rn(fi, sum)), dg, ry));
}

template <int MODE, int NV, int G, int WP, bool EV>
__global__ void __launch_bounds__(kMarchThreads, G == 0 ? 2 : 3)
    k_march(int n, const uint8_t *__restrict__ pid, int np, const unsigned char *__restrict__ table, int tb,
            const unsigned char *__restrict__ mtable, int mtb, const __grid_constant__ MarchPat<Geo<G>::W> mp,
            const double *__restrict__ x, const double *__restrict__ f, double *__restrict__ out, double omega,
            const int *skip, Red red) {
    static_assert(G == 0, "the marching kernel is specialised for the 27-point box");
    constexpr int W = Geo<G>::W, WE = (W + 1) & ~1;
    extern __shared__ __align__(16) unsigned char smem[];
    double *ring = reinterpret_cast<double *>(smem);
    uint64_t *bar = reinterpret_cast<uint64_t *>(ring + kMarchD * kPlaneW);
    unsigned char *tabs = reinterpret_cast<unsigned char *>(bar + kMarchD);
    {  // constant tables: before the dependency wait
        const uint4 *s0 = reinterpret_cast<const uint4 *>(table);
        uint4 *d0 = reinterpret_cast<uint4 *>(tabs);
        for (int i = threadIdx.x; i < tb / 16; i += blockDim.x) d0[i] = s0[i];
        const uint4 *s1 = reinterpret_cast<const uint4 *>(mtable);
        uint4 *d1 = reinterpret_cast<uint4 *>(tabs + tb);
        for (int i = threadIdx.x; i < mtb / 16; i += blockDim.x) d1[i] = s1[i];
        if (threadIdx.x == 0) {
            for (int i = 0; i < kMarchD; ++i) mbar_init(&bar[i], kChunks);
            fence_mbar_init();
        }
    }
    __syncthreads();
    SmemTab<WP> T;
    T.val = reinterpret_cast<const double *>(tabs);
    T.dg = T.val + static_cast<size_t>(np) * SmemTab<WP>::WV;
    T.ry = T.dg + np;
    T.off = reinterpret_cast<const int32_t *>(T.ry + np);
    T.len = reinterpret_cast<const uint8_t *>(T.off + static_cast<size_t>(np) * SmemTab<WP>::WO);
    const double *ev = reinterpret_cast<const double *>(tabs + tb);
    const uint8_t *emb = reinterpret_cast<const uint8_t *>(ev + static_cast<size_t>(np) * WE);

    double acc[NV > 0 ? NV : 1];
#pragma unroll
    for (int v = 0; v < (NV > 0 ? NV : 1); ++v) acc[v] = 0.0;
    auto emit = [&](int row, double o, double fi, double xi) {
        out[row] = o;
        if (NV >= 1) acc[0] += o * (red.w0 ? (red.w0 == f ? fi : red.w0 == x ? xi : red.w0[row]) : o);
        if (NV >= 2) acc[NV >= 2 ? 1 : 0] += o * (red.w1 ? (red.w1 == x ? xi : red.w1[row]) : o);
    };
    auto plain_row = [&](int row) {  // the row-pattern kernel's per-row path
        const int p = pid[row];
        const double *xr = x + row;
        const double xi = __ldg(xr);
        const double fi = (MODE == M_SPMV) ? 0.0 : __ldg(f + row);
        const double sum = wide_row_sum<WP>(SrcTab<WP>{T, p}, xr, xi);
        emit(row, march_out<MODE>(xi, fi, omega, sum, T.d(p), T.r(p)), fi, xi);
    };
    auto lean_row = [&](int row) {  // the same, one gather at a time (inside the march: few registers)
        const int p = pid[row];
        const double xi = __ldg(x + row);
        const double fi = (MODE == M_SPMV) ? 0.0 : __ldg(f + row);
        emit(row, march_out<MODE>(xi, fi, omega, wide_row_sum_masked<WP>(T, p, x + row), T.d(p), T.r(p)), fi, xi);
    };

    const int lane = threadIdx.x & 31, wy = threadIdx.x >> 5;
    pdl_wait();
    if (!(skip && *skip)) {
        {  // plane 0 and planes >= nqf - 1 (their windows leave [0, n)): per row
            const int64_t lo_end = n < mp.P ? n : mp.P;
            const int64_t hb = static_cast<int64_t>(max(mp.nqf - 1, 1)) * mp.P;
            const int64_t hi_beg = hb > lo_end ? hb : lo_end;
            const int64_t cnt = lo_end + (n - hi_beg);
            for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < cnt;
                 i += static_cast<int64_t>(gridDim.x) * blockDim.x)
                plain_row(static_cast<int>(i < lo_end ? i : hi_beg + (i - lo_end)));
        }
        // producer (every thread, identically): next tile / plane to stage,
        // items issued; items are the staged planes of the CTA's fast tiles in
        // order, item g in ring slot g % D, its mbarrier phase (g / D) & 1.
        // Threads 0..179 each copy one 16-byte chunk of a plane (cp.async,
        // completion tracked by the slot's mbarrier: 180 arrivals per phase).
        int pt = blockIdx.x, pj = 0, issued = 0;
        int freed = 0, base = 0;  // items released / items of the tiles before this one
        const int li = threadIdx.x / (kLineW / 2), ch = threadIdx.x - li * (kLineW / 2);
        // the producer's tile, decoded once: stage it (fast), planes, first plane,
        // this thread's line start minus one (x0 - 1 + (y0 - 1 + li) N)
        bool pfast = false;
        int pkt = 0, pq0 = 0;
        int64_t ploff = 0;
        auto decode = [&]() {
            const MarchTile<W> tl(mp, pt, n);
            pfast = tl.fast;
            pkt = tl.kt;
            pq0 = tl.q0;
            ploff = static_cast<int64_t>(tl.y0 - 1 + li) * mp.N + tl.x0 - 1 + 2 * ch;
        };
        if (pt < mp.ntiles) decode();
        auto pump = [&]() {
            while (issued < freed + kMarchD && pt < mp.ntiles) {
                if (!pfast || pj >= pkt + 2) {
                    pt += gridDim.x;
                    pj = 0;
                    if (pt < mp.ntiles) decode();
                    continue;
                }
                const int slot = issued & (kMarchD - 1);
                if (threadIdx.x < kChunks) {
                    const int64_t a = static_cast<int64_t>(pq0 - 1 + pj) * mp.P + ploff;  // line start + 2 ch - 1
                    const double *src = x + ((a - 2 * ch) & ~int64_t(1)) + 2 * ch;
                    double *dst = ring + slot * kPlaneW + li * kLineW + 2 * ch;
                    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
                    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&bar[slot]))
                                 : "memory");
                }
                ++issued;
                ++pj;
            }
        };
        pump();
        for (int t = blockIdx.x; t < mp.ntiles; t += gridDim.x) {
            const MarchTile<W> tl(mp, t, n);
            if (t + static_cast<int>(gridDim.x) >= mp.ntiles) pdl_trigger();
            const int y = tl.y0 + wy, c = tl.x0 + lane;
            const bool act = y < mp.NY && c < mp.N;
            if (!tl.fast) {
                if (act)
                    for (int k = 0; k < kMarchK; ++k) {
                        const int q = tl.q0 + k;
                        if (q >= mp.nqf - 1) break;
                        lean_row(q * mp.P + y * mp.N + c);
                    }
                continue;
            }
            // the window: three planes of 9 values ((dy, dx) order), rotated by
            // array identity over an unrolled-by-3 step loop (no register moves)
            double A[9], B[9], Cc[9];
            bool have = false;
            const int rrow0 = tl.q0 * mp.P + (act ? y * mp.N + c : 0);
            int pn = pid[rrow0];
            double fn = (MODE == M_SPMV) ? 0.0 : __ldg(f + rrow0);
            // staged values of plane qq (item g) around this thread's row: line
            // wy + dy + 1, column lane + dx + 1 + parity of the line start
            // qq P + (y + dy) N + x0 - 1 (x0 even; 1 when P and N are even)
            auto loadp = [&](double (&Pl)[9], int g, int qq) {
                const double *pb = ring + (g & (kMarchD - 1)) * kPlaneW + wy * kLineW + lane + 1;
#pragma unroll
                for (int dy = -1; dy <= 1; ++dy) {
                    const int sh = EV ? 1 : ((qq * mp.P + (y + dy) * mp.N + 1) & 1);
                    const double *lp = pb + (dy + 1) * kLineW + sh;
#pragma unroll
                    for (int dx = -1; dx <= 1; ++dx) Pl[(dy + 1) * 3 + dx + 1] = lp[dx];
                }
            };
            auto step = [&](double (&Pm)[9], double (&P0)[9], double (&Pp)[9], int k) {
                const int q = tl.q0 + k;
                const int row = rrow0 + k * mp.P;
                const int p = pn;
                const double fi = fn;
                if (k + 1 < tl.kt) {  // next step's pattern byte and rhs, loaded a step ahead
                    pn = pid[row + mp.P];
                    if (MODE != M_SPMV) fn = __ldg(f + row + mp.P);
                }
                // planes q - 1, q, q + 1 = items base + k, +1, +2
                const int g = base + k + 1;
                if (k == 0) {
                    mbar_wait(&bar[(g - 1) & (kMarchD - 1)], ((g - 1) / kMarchD) & 1);
                    mbar_wait(&bar[g & (kMarchD - 1)], (g / kMarchD) & 1);
                }
                mbar_wait(&bar[(g + 1) & (kMarchD - 1)], ((g + 1) / kMarchD) & 1);
                if (__all_sync(0xffffffffu, !act || emb[p])) {
                    if (!have) {
                        loadp(Pm, g - 1, q - 1);
                        loadp(P0, g, q);
                    }
                    loadp(Pp, g + 1, q + 1);
                    have = true;
                    const double xi = P0[4];
                    double sum = 0.0, dg, ry;
                    if (__all_sync(0xffffffffu, !act || p == mp.p)) {
#pragma unroll
                        for (int j = 0; j < 9; ++j) sum = __dadd_rn(sum, __dmul_rn(mp.v[j], Pm[j]));
#pragma unroll
                        for (int j = 0; j < 9; ++j) sum = __dadd_rn(sum, __dmul_rn(mp.v[9 + j], P0[j]));
#pragma unroll
                        for (int j = 0; j < 9; ++j) sum = __dadd_rn(sum, __dmul_rn(mp.v[18 + j], Pp[j]));
                        dg = mp.d;
                        ry = mp.r;
                    } else {
                        const double *e = ev + p * WE;
                        auto wv = [&](int j) { return j < 9 ? Pm[j] : j < 18 ? P0[j - 9] : Pp[j - 18]; };
#pragma unroll
                        for (int j = 0; j < W; j += 2) {
                            const double2 v2 = *reinterpret_cast<const double2 *>(e + j);
                            sum = __dadd_rn(sum, __dmul_rn(v2.x, wv(j)));
                            if (j + 1 < W) sum = __dadd_rn(sum, __dmul_rn(v2.y, wv(j + 1 < W ? j + 1 : 0)));
                        }
                        dg = T.d(p);
                        ry = T.r(p);
                        if (act && p != mp.p && !isfinite(sum))  // an absent slot read inf/NaN: exact replay
                            sum = wide_row_sum_masked<WP>(T, p, x + row);
                    }
                    if (act) emit(row, march_out<MODE>(xi, fi, omega, sum, dg, ry), fi, xi);
                } else {
                    have = false;
                    if (act) lean_row(row);
                }
                __syncthreads();  // every warp is done with plane q - 1
                freed = (k + 1 == tl.kt) ? base + tl.kt + 2 : base + k + 1;
                pump();
            };
#pragma unroll 1
            for (int k = 0; k < tl.kt; k += 3) {
                step(A, B, Cc, k);
                if (k + 1 < tl.kt) step(B, Cc, A, k + 1);
                if (k + 2 < tl.kt) step(Cc, A, B, k + 2);
            }
            base += tl.kt + 2;
        }
    }
    if constexpr (NV > 0) finish_reduction<NV>(red, acc);
}
