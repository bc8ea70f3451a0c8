// Row-pattern format ("RPAT"), included by sb_runtime.cu after the SELL-G kernel.
//
// A level whose rows repeat a small set of (column - row offsets, values)
// sequences -- <= 256 distinct rows, which every level of the structured-grid
// hierarchies has (27 distinct rows at every level of C2/C3/C4, 9 for C1) --
// is stored as ONE byte per row: the index of its pattern. The pattern table
// (offsets, values in the row's CSR order, a_ii and RN(1/a_ii)) sits in shared
// memory. The encoding is lossless (bit-exact values, CSR entry order): the
// sums are the reference's (inc/csr.hpp:185-191). Levels with more patterns use
// SELL-G. Per row the sweep streams 1 B of matrix + the vectors, so the pass is
// bound by x / f / x_new (24 B/row) instead of the matrix.
//
// Table layout (bytes, built on the host, copied into shared memory by every
// CTA before the dependency wait): f64 val[np][WV] | f64 diag[np] |
// f64 rdiag[np] | int32 off[np][WO] | uint8 len[np] (padded to 16); WV = W
// rounded up to 2, WO = W rounded up to 4 (16-byte rows).

constexpr int kPatThreads = 256;

// base + off (doubles) as ONE 32x32->64 multiply-add (IMAD.WIDE): the
// compiler otherwise re-associates (row + off) into 64-bit index arithmetic
// (4 instructions per gather)
__device__ __forceinline__ const double *at_off(const double *base, int off) {
    const double *r;
    asm("mad.wide.s32 %0, %1, 8, %2;" : "=l"(r) : "r"(off), "l"(base));
    return r;
}
// rows per thread per iteration (their gathers in flight together)
#ifndef SB_PAT_ROWS
#define SB_PAT_ROWS 2
#endif
template <int W> struct PatRows { static constexpr int value = W <= 8 ? SB_PAT_ROWS : 1; };

__host__ __device__ __forceinline__ size_t pat_table_bytes(int np, int w) {
    const size_t wv = (w + 1) & ~1, wo = (w + 3) & ~3;
    return (static_cast<size_t>(np) * (wv * 8 + wo * 4) + static_cast<size_t>(np) * 17 + 15) & ~size_t(15);
}

#ifndef SB_PAT_MINB_WIDE
#define SB_PAT_MINB_WIDE 3
#endif
#ifndef SB_PAT_MINB
#define SB_PAT_MINB 4
#endif
// Pattern table view over the shared-memory copy. (Passing the table as a
// kernel parameter, read with constant-cache loads, measured 5-15% slower: the
// lanes of a warp index different patterns at grid boundaries.)
template <int W> struct SmemTab {
    static constexpr int WV = (W + 1) & ~1;  // value row stride (doubles): 16-byte rows
    static constexpr int WO = (W + 3) & ~3;  // offset row stride (int32): 16-byte rows
    const double *val, *dg, *ry;
    const int32_t *off;
    const uint8_t *len;
    __device__ __forceinline__ double v(int p, int k) const { return val[p * WV + k]; }
    __device__ __forceinline__ int o(int p, int k) const { return off[p * WO + k]; }
    __device__ __forceinline__ double d(int p) const { return dg[p]; }
    __device__ __forceinline__ double r(int p) const { return ry[p]; }
    __device__ __forceinline__ int l(int p) const { return len[p]; }
    // a whole row of offsets / values with 16-byte shared-memory loads (one
    // wavefront per load when the warp's rows share the pattern)
    __device__ __forceinline__ void offs(int p, int (&o)[W]) const {
        const int32_t *b = off + p * WO;
#pragma unroll
        for (int k = 0; k < W; k += 4) {
            const int4 t = *reinterpret_cast<const int4 *>(b + k);
            o[k] = t.x;
            if (k + 1 < W) o[k + 1 < W ? k + 1 : 0] = t.y;
            if (k + 2 < W) o[k + 2 < W ? k + 2 : 0] = t.z;
            if (k + 3 < W) o[k + 3 < W ? k + 3 : 0] = t.w;
        }
    }
    __device__ __forceinline__ void vals(int p, double (&v)[W]) const {
        const double *b = val + p * WV;
#pragma unroll
        for (int k = 0; k < W; k += 2) {
            const double2 t = *reinterpret_cast<const double2 *>(b + k);
            v[k] = t.x;
            if (k + 1 < W) v[k + 1 < W ? k + 1 : 0] = t.y;
        }
    }
};

template <int W>
__device__ __forceinline__ SmemTab<W> smem_tab(unsigned char *smem, const unsigned char *table, int np) {
    const int tb = static_cast<int>(pat_table_bytes(np, W));
    {  // constant table: before the dependency wait (overlaps the predecessor's tail)
        const uint4 *src = reinterpret_cast<const uint4 *>(table);
        uint4 *dst = reinterpret_cast<uint4 *>(smem);
        for (int i = threadIdx.x; i < tb / 16; i += blockDim.x) dst[i] = src[i];
    }
    __syncthreads();
    SmemTab<W> T;
    T.val = reinterpret_cast<const double *>(smem);
    T.dg = T.val + static_cast<size_t>(np) * SmemTab<W>::WV;
    T.ry = T.dg + np;
    T.off = reinterpret_cast<const int32_t *>(T.ry + np);
    T.len = reinterpret_cast<const uint8_t *>(T.off + static_cast<size_t>(np) * SmemTab<W>::WO);
    return T;
}

// The level's most frequent pattern, passed by value as a kernel parameter:
// a warp whose rows all have it reads offsets and values as constant-bank
// operands (no shared-memory loads; the table reads otherwise cost as many L1
// wavefronts as the x gathers on 27-point levels).
template <int W> struct MainPat {
    double v[W];
    double d, r;
    int o[W];
    int p, len;
};
template <int W> struct SrcMain {  // row source: the main pattern (kernel parameter)
    const MainPat<W> &m;
    __device__ __forceinline__ void offs(int (&o)[W]) const {
#pragma unroll
        for (int k = 0; k < W; ++k) o[k] = m.o[k];
    }
    __device__ __forceinline__ void vals(double (&v)[W]) const {
#pragma unroll
        for (int k = 0; k < W; ++k) v[k] = m.v[k];
    }
    __device__ __forceinline__ double v1(int k) const { return m.v[k]; }
    __device__ __forceinline__ int o1(int k) const { return m.o[k]; }
    __device__ __forceinline__ double d() const { return m.d; }
    __device__ __forceinline__ double r() const { return m.r; }
    __device__ __forceinline__ int l() const { return m.len; }
};
template <int W> struct SrcTab {  // row source: pattern p of the shared-memory table
    const SmemTab<W> &T;
    int p;
    __device__ __forceinline__ void offs(int (&o)[W]) const { T.offs(p, o); }
    __device__ __forceinline__ void vals(double (&v)[W]) const { T.vals(p, v); }
    __device__ __forceinline__ double v1(int k) const { return T.v(p, k); }
    __device__ __forceinline__ int o1(int k) const { return T.o(p, k); }
    __device__ __forceinline__ double d() const { return T.d(p); }
    __device__ __forceinline__ double r() const { return T.r(p); }
    __device__ __forceinline__ int l() const { return T.l(p); }
};

// sum_k v_k x[i + o_k] of one wide row in slot order (padding slots add +0.0;
// replayed with masked slots when the row's own x is not finite, see below)
template <int W, typename S>
__device__ __forceinline__ double wide_row_sum(const S &src, const double *__restrict__ xr, double xi) {
    int o[W];
    src.offs(o);
    double xv[W];
#pragma unroll
    for (int k = 0; k < W; ++k) xv[k] = __ldg(at_off(xr, o[k]));
    double v[W];
    src.vals(v);
    double sum = 0.0;
#pragma unroll
    for (int k = 0; k < W; ++k) sum = __dadd_rn(sum, __dmul_rn(v[k], xv[k]));
    const int len = src.l();
    if (len < W && !isfinite(xi)) {
        sum = 0.0;
        for (int k = 0; k < len; ++k) sum = __dadd_rn(sum, __dmul_rn(src.v1(k), __ldg(xr + src.o1(k))));
    }
    return sum;
}

// wide rows (27-point levels) keep all W gathers in flight: more registers, 3 CTAs/SM
template <int MODE, int NV, int W>
__device__ __forceinline__ void rowpat_body(const SmemTab<W> &T, const MainPat<W> &mp, int n, const uint8_t *__restrict__ pid,
                                            const double *__restrict__ x, const double *__restrict__ f,
                                            double *__restrict__ out, double omega, const int *skip, Aux aux,
                                            Red red) {
    double acc[NV > 0 ? NV : 1];
#pragma unroll
    for (int v = 0; v < (NV > 0 ? NV : 1); ++v) acc[v] = 0.0;
    constexpr int kPatRows = PatRows<W>::value;
    const int stride = gridDim.x * kPatThreads * kPatRows;
    // the pattern bytes of the next iteration are loaded one iteration ahead,
    // so the x gathers do not wait behind a dependent DRAM load; the first
    // ones (constant data) before the dependency wait
    int pn[kPatRows];
#pragma unroll
    for (int q = 0; q < kPatRows; ++q) {
        const int r = blockIdx.x * kPatThreads * kPatRows + threadIdx.x + q * kPatThreads;
        pn[q] = pid[r < n ? r : n - 1];  // out-of-range threads replay row n-1 (valid gathers)
    }
    pdl_wait();
    if constexpr (W > 8 && (MODE == M_JACOBI || MODE == M_RESID || MODE == M_SPMV)) {
        // wide rows (27-point levels): one row per thread, all W gathers in
        // flight, sums in slot order
        if (!(skip && *skip)) {
            for (int base = blockIdx.x * kPatThreads; base < n; base += stride) {
                if (base + stride >= n) pdl_trigger();
                const int row = base + threadIdx.x;
                const int p = pn[0];
                { const int r = row + stride; pn[0] = pid[r < n ? r : n - 1]; }
                const int rq = row < n ? row : n - 1;
                const double *xr = x + rq;
                const double fi = (MODE == M_SPMV) ? 0.0 : __ldg(f + rq);
                const double xi = __ldg(xr);
                double sum, dg, ry;
                if (__all_sync(0xffffffffu, p == mp.p)) {
                    sum = wide_row_sum<W>(SrcMain<W>{mp}, xr, xi);
                    dg = mp.d;
                    ry = mp.r;
                } else {
                    sum = wide_row_sum<W>(SrcTab<W>{T, p}, xr, xi);
                    dg = T.d(p);
                    ry = T.r(p);
                }
                if (row < n) {
                    double o;
                    if constexpr (MODE == M_SPMV) o = sum;
                    else if constexpr (MODE == M_RESID) o = __dsub_rn(fi, sum);
                    else o = __dadd_rn(xi, div_rn(__dmul_rn(omega, __dsub_rn(fi, sum)), dg, ry));
                    out[row] = o;
                    if (NV >= 1) acc[0] += o * (red.w0 ? (red.w0 == f ? fi : red.w0[row]) : o);
                    if (NV >= 2) acc[NV >= 2 ? 1 : 0] += o * (red.w1 ? red.w1[row] : o);
                }
            }
        }
    } else if (!(skip && *skip)) {
        for (int base = blockIdx.x * kPatThreads * kPatRows; base < n; base += stride) {
            if (base + stride >= n) pdl_trigger();
            int row[kPatRows], p[kPatRows];
            double xv[kPatRows][W];
#pragma unroll
            for (int q = 0; q < kPatRows; ++q) {
                row[q] = base + threadIdx.x + q * kPatThreads;
                p[q] = pn[q];
                const int r = row[q] + stride;
                pn[q] = pid[r < n ? r : n - 1];
            }
            // one iteration with the rows' table source: the main pattern for
            // a warp whose rows all have it, else the shared-memory table
            auto iter = [&](auto src) {
                double fv[kPatRows], xo[kPatRows];  // rhs and own iterate, loaded with the gathers
#pragma unroll
                for (int q = 0; q < kPatRows; ++q) {
                    const int rq = row[q] < n ? row[q] : n - 1;
                    const double *xr = x + rq;
                    int o[W];
                    src(q).offs(o);
#pragma unroll
                    for (int k = 0; k < W; ++k) {
                        const int off = o[k];
                        if constexpr (MODE == M_JACOBI || MODE == M_RESID || MODE == M_SPMV) xv[q][k] = __ldg(at_off(xr, off));
                        else xv[q][k] = xval<MODE, false>(rq + off, x, f, aux, omega);
                    }
                    fv[q] = (MODE == M_SPMV) ? 0.0 : __ldg(f + rq);
                    xo[q] = (MODE >= M_JACOBI) ? xval<MODE, false>(rq, x, f, aux, omega) : 0.0;
                }
#pragma unroll
                for (int q = 0; q < kPatRows; ++q) {
                    if (row[q] >= n) continue;
                    const int len = src(q).l();
                    // Padding slots hold value +0.0 at offset 0 (the row itself): 0 * x_i
                    // is +-0 and sum + (+-0) == sum bit for bit (sum is never -0), so
                    // the unmasked sum equals the reference's unless x_i is inf / NaN
                    // (0 * inf = NaN); only then replay the row with masked slots.
                    double v[W];
                    src(q).vals(v);
                    double sum = 0.0;
#pragma unroll
                    for (int k = 0; k < W; ++k) sum = __dadd_rn(sum, __dmul_rn(v[k], xv[q][k]));
                    if (len < W && !isfinite(xv[q][W - 1])) {
                        sum = 0.0;
#pragma unroll
                        for (int k = 0; k < W; ++k) add_if(sum, __dmul_rn(v[k], xv[q][k]), k < len);
                    }
                    double o;
                    if constexpr (MODE == M_SPMV) {
                        o = sum;
                    } else if constexpr (MODE == M_RESID) {
                        o = __dsub_rn(fv[q], sum);
                    } else {
                        o = __dadd_rn(xo[q], div_rn(__dmul_rn(omega, __dsub_rn(fv[q], sum)), src(q).d(), src(q).r()));
                    }
                    out[row[q]] = o;
                    if (NV >= 1) acc[0] += o * (red.w0 ? (red.w0 == f ? fv[q] : red.w0[row[q]]) : o);
                    if (NV >= 2) acc[NV >= 2 ? 1 : 0] += o * (red.w1 ? red.w1[row[q]] : o);
                }
            };
            bool uni = true;
#pragma unroll
            for (int q = 0; q < kPatRows; ++q) uni = uni && p[q] == mp.p;
            if (__all_sync(0xffffffffu, uni)) iter([&](int) { return SrcMain<W>{mp}; });
            else iter([&](int q) { return SrcTab<W>{T, p[q]}; });
        }
    }
    if constexpr (NV > 0) finish_reduction<NV>(red, acc);
}

template <int MODE, int NV, int W>
__global__ void __launch_bounds__(kPatThreads, W <= 8 ? SB_PAT_MINB : SB_PAT_MINB_WIDE)
    k_rowpat(int n, const uint8_t *__restrict__ pid, int np, const unsigned char *__restrict__ table,
             const __grid_constant__ MainPat<W> mp, const double *__restrict__ x, const double *__restrict__ f,
             double *__restrict__ out, double omega, const int *skip, Aux aux, Red red) {
    extern __shared__ __align__(16) unsigned char smem[];
    const SmemTab<W> T = smem_tab<W>(smem, table, np);
    rowpat_body<MODE, NV, W>(T, mp, n, pid, x, f, out, omega, skip, aux, red);
}

// Residual + restriction fused for a row-pattern level (one launch and no r
// vector): thread c evaluates r_m = f_m - A_m x for the members m0 < m1 of
// coarse row c in the reference's order and writes f_c = (0 + r_m0) + r_m1
// (csr.hpp:267-274 then the unit-P spmv_transpose, csr.hpp:232-239); with
// xc0, also the coarse level's first sweep from 0, x0_c = 0 + (w f_c) / a_cc.
template <int W>
__device__ __forceinline__ double pat_resid_row(int m, int p, const SmemTab<W> &T, const double *__restrict__ x,
                                                const double *__restrict__ f) {
    int o[W];
    T.offs(p, o);
    double xv[W];
#pragma unroll
    for (int k = 0; k < W; ++k) xv[k] = __ldg(at_off(x + m, o[k]));
    const double fm = f[m];
    double v[W];
    T.vals(p, v);
    double sum = 0.0;
#pragma unroll
    for (int k = 0; k < W; ++k) sum = __dadd_rn(sum, __dmul_rn(v[k], xv[k]));
    const int len = T.l(p);
    if (len < W && !isfinite(xv[W - 1])) {  // see k_rowpat: exact replay for a non-finite own x
        sum = 0.0;
#pragma unroll
        for (int k = 0; k < W; ++k) add_if(sum, __dmul_rn(v[k], xv[k]), k < len);
    }
    return __dsub_rn(fm, sum);
}

template <int W>
__global__ void __launch_bounds__(kPatThreads, W <= 8 ? SB_PAT_MINB : SB_PAT_MINB_WIDE)
    k_pat_resid_restrict(int nc, const int2 *__restrict__ mem, const uint8_t *__restrict__ pid, int np,
                         const unsigned char *__restrict__ table, const double *__restrict__ x,
                         const double *__restrict__ f, double *__restrict__ fc, const double *__restrict__ dc,
                         double *__restrict__ xc0, double omega) {
    extern __shared__ __align__(16) unsigned char smem[];
    const SmemTab<W> T = smem_tab<W>(smem, table, np);
    const int c0 = blockIdx.x * blockDim.x + threadIdx.x;
    int2 mm = make_int2(0, -1);
    int p0 = 0, p1 = 0;
    double d = 0.0;
    if (c0 < nc) {  // constant data before the dependency wait
        mm = mem[c0];
        p0 = pid[mm.x];
        if (mm.y >= 0) p1 = pid[mm.y];
        if (xc0) d = dc[c0];
    }
    pdl_wait();
    pdl_trigger_single(nc);
    for (int c = c0; c < nc; c += gridDim.x * blockDim.x) {
        if (c != c0) {
            mm = mem[c];
            p0 = pid[mm.x];
            if (mm.y >= 0) p1 = pid[mm.y];
            if (xc0) d = dc[c];
        }
        double s = __dadd_rn(0.0, pat_resid_row<W>(mm.x, p0, T, x, f));
        if (mm.y >= 0) s = __dadd_rn(s, pat_resid_row<W>(mm.y, p1, T, x, f));
        fc[c] = s;
        if (xc0) xc0[c] = __dadd_rn(0.0, __ddiv_rn(__dmul_rn(omega, s), d));
    }
}

// Row pairs on 27-point box levels (k_boxpair). A thread owns rows 2q, 2q + 1
// (P and N even, so for every run (dz, dy) of three consecutive columns the
// base r + dz P + dy N is even): the six x values both rows need from a run,
// x[r + d - 1 .. r + d + 2] (and d - 2 for alignment), come from three
// 16-byte loads instead of six 8-byte gathers, the rhs / output / pattern
// bytes of the pair in one vector access each, and the two rows' sums are two
// independent dependent chains (ILP 2 for the reference's sequential order).
// Warps whose 64 rows are not all the main pattern, or whose reads would leave
// [0, n), run the row-pattern per-row path. L1 wavefronts per 32 rows: ~58 vs
// ~79 for k_rowpat's wide path, which is L1-bound (ncu: 87% of peak).
#ifndef SB_BOX_THREADS
#define SB_BOX_THREADS 128  // measured: 128 x 5 CTAs/SM (<= 102 registers) 176 us vs 212 at 256 x 2 (27-pt 256^3 L0)
#endif
#ifndef SB_BOX_MINB
#define SB_BOX_MINB 5
#endif
constexpr int kBoxThreads = SB_BOX_THREADS;
template <int MODE, int NV>
__global__ void __launch_bounds__(kBoxThreads, SB_BOX_MINB)
    k_boxpair(int n, const uint8_t *__restrict__ pid, int np, const unsigned char *__restrict__ table,
              const uint32_t *__restrict__ rmask, const __grid_constant__ MainPat<28> mp,
              const double *__restrict__ x, const double *__restrict__ f, double *__restrict__ out, double omega,
              const int *skip, Red red) {
    extern __shared__ __align__(16) unsigned char smem[];
    const SmemTab<28> T = smem_tab<28>(smem, table, np);
    double acc[NV > 0 ? NV : 1];
#pragma unroll
    for (int v = 0; v < (NV > 0 ? NV : 1); ++v) acc[v] = 0.0;
    const int npairs = n >> 1;
    const int stride = gridDim.x * kBoxThreads;
    const int lo = -mp.o[0] + 2, hi = n - (mp.o[26] + 3);  // pairs starting in [lo, hi) read inside [0, n)
    auto accum = [&](int row, double o, double fi, double xi) {
        if (NV >= 1) acc[0] += o * (red.w0 ? (red.w0 == f ? fi : red.w0 == x ? xi : red.w0[row]) : o);
        if (NV >= 2) acc[NV >= 2 ? 1 : 0] += o * (red.w1 ? (red.w1 == x ? xi : red.w1[row]) : o);
    };
    auto emit = [&](int row, double o, double fi, double xi) {
        out[row] = o;
        accum(row, o, fi, xi);
    };
    auto fin = [&](double xi, double fi, double sum, double dg, double ry) -> double {
        if constexpr (MODE == M_SPMV) return sum;
        else if constexpr (MODE == M_RESID) return __dsub_rn(fi, sum);
        else return __dadd_rn(xi, div_rn(__dmul_rn(omega, __dsub_rn(fi, sum)), dg, ry));
    };
    // the pattern bytes are constant: the first pair's before the dependency
    // wait, later ones one iteration ahead
    auto pair_of = [&](int qq) {
        return static_cast<uint32_t>(*reinterpret_cast<const uint16_t *>(pid + 2 * min(qq, npairs - 1)));
    };
    uint32_t ppn = npairs > 0 ? pair_of(blockIdx.x * kBoxThreads + threadIdx.x) : 0u;
    pdl_wait();
    if (!(skip && *skip)) {
        for (int q = blockIdx.x * kBoxThreads + threadIdx.x, base = blockIdx.x * kBoxThreads; base < npairs;
             q += stride, base += stride) {
            if (base + stride >= npairs) pdl_trigger();
            const bool in = q < npairs;
            const unsigned inm = __ballot_sync(0xffffffffu, in);
            const uint32_t ppc = ppn;
            if (base + stride < npairs) ppn = pair_of(q + stride);
            if (!inm) continue;
            // lanes past the end shadow the warp's first pair (in bounds, not stored)
            const int src = __ffs(inm) - 1;
            const int r0w = __shfl_sync(0xffffffffu, 2 * q, src);
            const uint32_t pps = __shfl_sync(0xffffffffu, ppc, src);
            const int r = in ? 2 * q : r0w;
            const uint32_t pp = in ? ppc : pps;
            const int p0 = pp & 0xff, p1 = pp >> 8;
            // restriction masks: the pattern is the main one with some slots absent
            // and the same values elsewhere (0: not a restriction)
            const uint32_t m0 = __ldg(rmask + p0), m1 = __ldg(rmask + p1);
            const bool fast = m0 && m1 && r >= lo && r < hi;
            if (__all_sync(0xffffffffu, fast)) {
                const double2 fv = (MODE == M_SPMV) ? make_double2(0.0, 0.0) : __ldg(reinterpret_cast<const double2 *>(f + r));
                double s0 = 0.0, s1 = 0.0, xi0 = 0.0, xi1 = 0.0;
                double2 A[9], B[9], Cc[9];
#pragma unroll
                for (int j = 0; j < 9; ++j) {  // run j: slots 3j .. 3j+2, base offset o[3j+1] (even)
                    const double2 *b = reinterpret_cast<const double2 *>(at_off(x + r, mp.o[3 * j + 1]));
                    A[j] = __ldg(b - 1);
                    B[j] = __ldg(b);
                    Cc[j] = __ldg(b + 1);
                }
                // an absent slot adds +0.0 (no product: inf / NaN there never enter),
                // sum + (+0) == sum bit for bit, so the sums are the rows' own CSR sums
                if (__all_sync(0xffffffffu, (m0 & m1) == 0x7ffffffu)) {
#pragma unroll
                    for (int j = 0; j < 9; ++j) {
                        s0 = __dadd_rn(s0, __dmul_rn(mp.v[3 * j], A[j].y));
                        s1 = __dadd_rn(s1, __dmul_rn(mp.v[3 * j], B[j].x));
                        s0 = __dadd_rn(s0, __dmul_rn(mp.v[3 * j + 1], B[j].x));
                        s1 = __dadd_rn(s1, __dmul_rn(mp.v[3 * j + 1], B[j].y));
                        s0 = __dadd_rn(s0, __dmul_rn(mp.v[3 * j + 2], B[j].y));
                        s1 = __dadd_rn(s1, __dmul_rn(mp.v[3 * j + 2], Cc[j].x));
                    }
                } else {
                    auto t = [&](uint32_t m, int k, double v, double xv) {
                        return ((m >> k) & 1u) ? __dmul_rn(v, xv) : 0.0;
                    };
#pragma unroll
                    for (int j = 0; j < 9; ++j) {
                        s0 = __dadd_rn(s0, t(m0, 3 * j, mp.v[3 * j], A[j].y));
                        s1 = __dadd_rn(s1, t(m1, 3 * j, mp.v[3 * j], B[j].x));
                        s0 = __dadd_rn(s0, t(m0, 3 * j + 1, mp.v[3 * j + 1], B[j].x));
                        s1 = __dadd_rn(s1, t(m1, 3 * j + 1, mp.v[3 * j + 1], B[j].y));
                        s0 = __dadd_rn(s0, t(m0, 3 * j + 2, mp.v[3 * j + 2], B[j].y));
                        s1 = __dadd_rn(s1, t(m1, 3 * j + 2, mp.v[3 * j + 2], Cc[j].x));
                    }
                }
                xi0 = B[4].x;
                xi1 = B[4].y;
                if (in) {
                    const double o0 = fin(xi0, fv.x, s0, mp.d, mp.r), o1 = fin(xi1, fv.y, s1, mp.d, mp.r);
                    if constexpr (NV == 0) {
                        *reinterpret_cast<double2 *>(out + r) = make_double2(o0, o1);
                    } else {
                        emit(r, o0, fv.x, xi0);
                        emit(r + 1, o1, fv.y, xi1);
                    }
                }
            } else if (in) {  // the row-pattern per-row path for both rows
#pragma unroll 1
                for (int h = 0; h < 2; ++h) {
                    const int row = r + h, p = h ? p1 : p0;
                    const double *xr = x + row;
                    const double xi = __ldg(xr);
                    const double fi = (MODE == M_SPMV) ? 0.0 : __ldg(f + row);
                    const double sum = (p == mp.p) ? wide_row_sum<28>(SrcMain<28>{mp}, xr, xi)
                                                   : wide_row_sum<28>(SrcTab<28>{T, p}, xr, xi);
                    const double dg = (p == mp.p) ? mp.d : T.d(p), ry = (p == mp.p) ? mp.r : T.r(p);
                    emit(row, fin(xi, fi, sum, dg, ry), fi, xi);
                }
            }
        }
    }
    if constexpr (NV > 0) finish_reduction<NV>(red, acc);
}

// Row pairs on 7-point (W = 7: -P, -N, -1, 0, 1, N, P) and 5-point (W = 5:
// -N, -1, 0, 1, N) cross levels with even strides: k_boxpair's scheme for the
// cross. Per pair: one 16-byte load for each of the +-P / +-N neighbour pairs,
// three for the -1 .. +2 run, one for the rhs, one store; the two rows' sums
// are independent chains; restriction masks (W bits) keep boundary rows on the
// vector path (absent slot: +0.0, no product).
#ifndef SB_CROSS_THREADS
#define SB_CROSS_THREADS 256
#endif
#ifndef SB_CROSS_MINB
#define SB_CROSS_MINB 6  // measured (C2 / 256^3 L0 sweeps): 256 x 6 best of 256 x 4,5,6,8, 128 x 8,10,12, 512 x 2
                         // (256 x 8 = 32 registers spills: 256^3 L0 110 vs 79 us cold)
#endif
#ifndef SB_CROSS_MINB_NV
#define SB_CROSS_MINB_NV 4  // fused-dot variants (SpMV + dot, last sweep + dot): room for the reduction state
#endif
constexpr int kCrossThreads = SB_CROSS_THREADS;
template <int MODE, int NV, int W, bool RG = false>
__global__ void __launch_bounds__(kCrossThreads, NV > 0 ? SB_CROSS_MINB_NV : SB_CROSS_MINB)
    k_crosspair(int n, const uint8_t *__restrict__ pid, int np, const unsigned char *__restrict__ table,
                const uint32_t *__restrict__ rmask, const __grid_constant__ MainPat<W> mp,
                const double *__restrict__ x, const double *__restrict__ f, double *__restrict__ out, double omega,
                const int *skip, Red red, int q_lo_, int q_hi_) {
    // RG: only the pairs [q_lo_, q_hi_) (the partitioned path sweeps its
    // interior while the halo is in flight, then the rest); else every pair.
    // (Separate instantiation: the range bounds as runtime values cost the
    // whole-level sweep ~20% at 256^3, measured.)
    static_assert(W == 7 || W == 5, "cross geometries");
    constexpr int C = W / 2;  // centre slot (offset 0)
    extern __shared__ __align__(16) unsigned char smem[];
    const SmemTab<W> T = smem_tab<W>(smem, table, np);
    double acc[NV > 0 ? NV : 1];
#pragma unroll
    for (int v = 0; v < (NV > 0 ? NV : 1); ++v) acc[v] = 0.0;
    const int npairs = n >> 1;
    const int q_lo = RG ? q_lo_ : 0, q_hi = RG ? q_hi_ : npairs;
    const int stride = gridDim.x * kCrossThreads;
    const int lo = -mp.o[0] + 2, hi = n - (mp.o[W - 1] + 3);
    // M_RESID_RESTRICT (coarse row q = fine rows 2q, 2q + 1; red.w0 = a_cc or
    // red.pid / red.pdg the coarse pattern's, red.w1 = the coarse first-sweep
    // destination or null): f_c = (0 + r0) + r1 (csr.hpp:267-274 then the
    // unit-P spmv_transpose, csr.hpp:232-239) and x0_c = 0 + (w f_c) / a_cc,
    // the operation order of k_pat_resid_restrict
    auto restrict_pair = [&](int qc, double r0, double r1) {
        const double s = __dadd_rn(__dadd_rn(0.0, r0), r1);
        out[qc] = s;
        if (red.w1) {
            const double d = red.pid ? __ldg(red.pdg + red.pid[qc]) : __ldg(red.w0 + qc);
            const_cast<double *>(red.w1)[qc] = __dadd_rn(0.0, __ddiv_rn(__dmul_rn(omega, s), d));
        }
    };
    auto accum = [&](int row, double o, double fi, double xi) {
        if (NV >= 1) acc[0] += o * (red.w0 ? (red.w0 == f ? fi : red.w0 == x ? xi : red.w0[row]) : o);
        if (NV >= 2) acc[NV >= 2 ? 1 : 0] += o * (red.w1 ? (red.w1 == x ? xi : red.w1[row]) : o);
    };
    auto emit = [&](int row, double o, double fi, double xi) {
        out[row] = o;
        accum(row, o, fi, xi);
    };
    auto fin = [&](double xi, double fi, double sum, double dg, double ry) -> double {
        if constexpr (MODE == M_SPMV) return sum;
        else if constexpr (MODE == M_RESID || MODE == M_RESID_RESTRICT) return __dsub_rn(fi, sum);
        else return __dadd_rn(xi, div_rn(__dmul_rn(omega, __dsub_rn(fi, sum)), dg, ry));
    };
    // the pattern bytes are constant: the first pair's before the dependency
    // wait, later ones one iteration ahead
    auto pair_of = [&](int qq) {
        return static_cast<uint32_t>(*reinterpret_cast<const uint16_t *>(pid + 2 * min(qq, npairs - 1)));
    };
    uint32_t ppn = q_hi > q_lo ? pair_of(q_lo + blockIdx.x * kCrossThreads + threadIdx.x) : 0u;
#ifdef SB_XP_TRACE
    const unsigned long long t_in = gtime();
    unsigned long long t_ld = 0;
#endif
    pdl_wait();
#ifdef SB_XP_TRACE
    const unsigned long long t_w = gtime();
#endif
    if (!(skip && *skip)) {
        for (int q = q_lo + blockIdx.x * kCrossThreads + threadIdx.x, base = q_lo + blockIdx.x * kCrossThreads;
             base < q_hi; q += stride, base += stride) {
            if (base + stride >= q_hi) pdl_trigger();
            const bool in = q < q_hi;
            const unsigned inm = __ballot_sync(0xffffffffu, in);
            const uint32_t ppc = ppn;
            if (base + stride < q_hi) ppn = pair_of(q + stride);
            if (!inm) continue;
            const int src = __ffs(inm) - 1;
            const int r0w = __shfl_sync(0xffffffffu, 2 * q, src);
            const uint32_t pps = __shfl_sync(0xffffffffu, ppc, src);
            const int r = in ? 2 * q : r0w;
            const uint32_t pp = in ? ppc : pps;
            const int p0 = pp & 0xff, p1 = pp >> 8;
            const uint32_t m0 = __ldg(rmask + p0), m1 = __ldg(rmask + p1);
            const bool fast = m0 && m1 && r >= lo && r < hi;
            if (__all_sync(0xffffffffu, fast)) {
                const double2 fv = (MODE == M_SPMV) ? make_double2(0.0, 0.0) : __ldg(reinterpret_cast<const double2 *>(f + r));
                const double *xr = x + r;
                // x values per slot for row r (a) and row r + 1 (b)
                double a[W], b[W];
                {
                    const double2 A = __ldg(reinterpret_cast<const double2 *>(xr - 2));
                    const double2 B = __ldg(reinterpret_cast<const double2 *>(xr));
                    const double2 Cc = __ldg(reinterpret_cast<const double2 *>(xr + 2));
                    a[C - 1] = A.y; a[C] = B.x; a[C + 1] = B.y;
                    b[C - 1] = B.x; b[C] = B.y; b[C + 1] = Cc.x;
                }
#pragma unroll
                for (int k = 0; k < W; ++k) {
                    if (k >= C - 1 && k <= C + 1) continue;
                    const double2 v2 = __ldg(reinterpret_cast<const double2 *>(at_off(xr, mp.o[k])));
                    a[k] = v2.x;
                    b[k] = v2.y;
                }
                if constexpr (MODE == M_JACOBI_PROLONG) {
                    // x' = x + (0 + x_c[j / 2]) at every row read: rows r-1 | r, r+1 |
                    // r+2 are pairs q-1 | q | q+1, the even offsets' rows pair q + o/2
                    const int qq = r >> 1;
                    const double *xc = red.w0;
                    const double cm = __dadd_rn(0.0, __ldg(xc + qq - 1)), c0 = __dadd_rn(0.0, __ldg(xc + qq)),
                                 cq = __dadd_rn(0.0, __ldg(xc + qq + 1));
                    a[C - 1] = __dadd_rn(a[C - 1], cm);
                    a[C] = __dadd_rn(a[C], c0);
                    a[C + 1] = __dadd_rn(a[C + 1], c0);
                    b[C - 1] = __dadd_rn(b[C - 1], c0);
                    b[C] = __dadd_rn(b[C], c0);
                    b[C + 1] = __dadd_rn(b[C + 1], cq);
#pragma unroll
                    for (int k = 0; k < W; ++k) {
                        if (k >= C - 1 && k <= C + 1) continue;
                        const double ck = __dadd_rn(0.0, __ldg(xc + qq + mp.o[k] / 2));
                        a[k] = __dadd_rn(a[k], ck);
                        b[k] = __dadd_rn(b[k], ck);
                    }
                }
                double s0 = 0.0, s1 = 0.0;
#ifdef SB_XP_TRACE
                {
                    double chk = fv.x;
#pragma unroll
                    for (int k = 0; k < W; ++k) chk += a[k] + b[k];
                    if (chk == 1.2345e300) t_ld = 1;
                    t_ld = max(t_ld, gtime());
                }
#endif
                if (__all_sync(0xffffffffu, (m0 & m1) == (1u << W) - 1u)) {
#pragma unroll
                    for (int k = 0; k < W; ++k) {
                        s0 = __dadd_rn(s0, __dmul_rn(mp.v[k], a[k]));
                        s1 = __dadd_rn(s1, __dmul_rn(mp.v[k], b[k]));
                    }
                } else {
#pragma unroll
                    for (int k = 0; k < W; ++k) {
                        s0 = __dadd_rn(s0, ((m0 >> k) & 1u) ? __dmul_rn(mp.v[k], a[k]) : 0.0);
                        s1 = __dadd_rn(s1, ((m1 >> k) & 1u) ? __dmul_rn(mp.v[k], b[k]) : 0.0);
                    }
                }
                if (in) {
                    const double o0 = fin(a[C], fv.x, s0, mp.d, mp.r), o1 = fin(b[C], fv.y, s1, mp.d, mp.r);
                    if constexpr (MODE == M_RESID_RESTRICT) {
                        restrict_pair(q, o0, o1);
                        continue;
                    }
                    *reinterpret_cast<double2 *>(out + r) = make_double2(o0, o1);
                    if constexpr (NV > 0) {
                        accum(r, o0, fv.x, a[C]);
                        accum(r + 1, o1, fv.y, b[C]);
                    }
                }
            } else if (in) {  // the row-pattern per-row path for both rows
                double o0r = 0.0, o1r = 0.0;
#pragma unroll 1
                for (int h = 0; h < 2; ++h) {
                    const int row = r + h, p = h ? p1 : p0;
                    const double *xrow = x + row;
                    auto xv = [&](int o) {  // x' = x + (0 + x_c[j / 2]) for M_JACOBI_PROLONG
                        if constexpr (MODE == M_JACOBI_PROLONG)
                            return __dadd_rn(__ldg(xrow + o), __dadd_rn(0.0, __ldg(red.w0 + ((row + o) >> 1))));
                        else
                            return __ldg(xrow + o);
                    };
                    const double xi = xv(0);
                    const double fi = (MODE == M_SPMV) ? 0.0 : __ldg(f + row);
                    double sum = 0.0;
                    const int len = T.l(p);
                    for (int k = 0; k < len; ++k) sum = __dadd_rn(sum, __dmul_rn(T.v(p, k), xv(T.o(p, k))));
                    if constexpr (MODE == M_RESID_RESTRICT) (h ? o1r : o0r) = fin(xi, fi, sum, 0.0, 0.0);
                    else emit(row, fin(xi, fi, sum, T.d(p), T.r(p)), fi, xi);
                }
                if constexpr (MODE == M_RESID_RESTRICT) restrict_pair(q, o0r, o1r);
            }
        }
    }
    if constexpr (NV > 0) finish_reduction<NV>(red, acc);
#ifdef SB_XP_TRACE
    const unsigned long long t_end = gtime();
    __shared__ unsigned long long s_ld, s_end;
    if (threadIdx.x == 0) s_ld = s_end = 0;
    __syncthreads();
    atomicMax(&s_ld, t_ld);
    atomicMax(&s_end, t_end);
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned i = atomicAdd(&g_xp_n, 1u);
        if (i < 65536u) {
            g_xp_trace[6 * i] = t_in;
            g_xp_trace[6 * i + 1] = t_w;
            g_xp_trace[6 * i + 2] = s_end;
            g_xp_trace[6 * i + 3] = blockIdx.x;
            g_xp_trace[6 * i + 4] = s_ld;
            g_xp_trace[6 * i + 5] = gtime();
        }
    }
#endif
}

// Residual + restriction (k_pat_resid_restrict) on 7-point cross levels with
// even strides when coarse row c's members are a row pair (2k, 2k + 1): node-HEM
// on a grid pairs each row with its right neighbour, so at the fine levels of
// C2-C4 every aggregate is one. The pair's two residuals come from
// k_crosspair's 16-byte loads; f_c = (0 + r_m0) + r_m1 and the coarse level's
// first sweep x0_c = 0 + (w f_c) / a_cc exactly as k_pat_resid_restrict
// (csr.hpp:267-274, 232-239). Warps with another aggregate or pattern shape
// take the per-member path. Bitwise equal, but measured slower than
// k_pat_resid_restrict (C2 solve 13.92 vs 13.61 ms with the prefetch below): opt-in, SB_CROSS_RR=1.
template <int W>
__global__ void __launch_bounds__(kCrossThreads, SB_CROSS_MINB)
    k_cross_rr(int nc, const int2 *__restrict__ mem, int n, const uint8_t *__restrict__ pid, int np,
               const unsigned char *__restrict__ table, const uint32_t *__restrict__ rmask,
               const __grid_constant__ MainPat<W> mp, const double *__restrict__ x, const double *__restrict__ f,
               double *__restrict__ fc, const double *__restrict__ dc, double *__restrict__ xc0, double omega) {
    constexpr int C = W / 2;
    extern __shared__ __align__(16) unsigned char smem[];
    const SmemTab<W> T = smem_tab<W>(smem, table, np);
    const int lo = -mp.o[0] + 2, hi = n - (mp.o[W - 1] + 3);
    const int stride = gridDim.x * kCrossThreads;
    auto resid = [&](int m, int p) {  // r_m = f_m - A_m x, the reference's order
        double sum = 0.0;
        const int len = T.l(p);
        for (int k = 0; k < len; ++k) sum = __dadd_rn(sum, __dmul_rn(T.v(p, k), __ldg(x + m + T.o(p, k))));
        return __dsub_rn(__ldg(f + m), sum);
    };
    // members and pattern bytes are constant: the first coarse row's before the
    // dependency wait, later ones one iteration ahead
    struct Pre {
        int2 mm;
        uint32_t pp;
    };
    auto pre_of = [&](int cc) {
        Pre q;
        q.mm = __ldg(mem + min(cc, nc - 1));
        const bool pair = q.mm.y == q.mm.x + 1 && (q.mm.x & 1) == 0;
        q.pp = pair ? static_cast<uint32_t>(*reinterpret_cast<const uint16_t *>(pid + q.mm.x)) : 0xffffffffu;
        return q;
    };
    Pre nx = pre_of(blockIdx.x * kCrossThreads + threadIdx.x);
    pdl_wait();
    for (int c = blockIdx.x * kCrossThreads + threadIdx.x, base = blockIdx.x * kCrossThreads; base < nc;
         c += stride, base += stride) {
        if (base + stride >= nc) pdl_trigger();
        const bool in = c < nc;
        const unsigned inm = __ballot_sync(0xffffffffu, in);
        const Pre cur = nx;
        if (base + stride < nc) nx = pre_of(c + stride);
        if (!inm) continue;
        const int src = __ffs(inm) - 1;
        const int2 mw = make_int2(__shfl_sync(0xffffffffu, cur.mm.x, src), __shfl_sync(0xffffffffu, cur.mm.y, src));
        const uint32_t pw = __shfl_sync(0xffffffffu, cur.pp, src);
        const int2 mm = in ? cur.mm : mw;
        const uint32_t pp = in ? cur.pp : pw;
        const int r = mm.x;
        bool fast = pp != 0xffffffffu && r >= lo && r < hi;
        uint32_t m0 = 0u, m1 = 0u;
        if (fast) {
            m0 = __ldg(rmask + (pp & 0xff));
            m1 = __ldg(rmask + (pp >> 8));
            fast = m0 && m1;
        }
        double s;
        if (__all_sync(0xffffffffu, fast)) {
            const double *xr = x + r;
            double a[W], b[W];
            {
                const double2 A = __ldg(reinterpret_cast<const double2 *>(xr - 2));
                const double2 B = __ldg(reinterpret_cast<const double2 *>(xr));
                const double2 Cc = __ldg(reinterpret_cast<const double2 *>(xr + 2));
                a[C - 1] = A.y; a[C] = B.x; a[C + 1] = B.y;
                b[C - 1] = B.x; b[C] = B.y; b[C + 1] = Cc.x;
            }
#pragma unroll
            for (int k = 0; k < W; ++k) {
                if (k >= C - 1 && k <= C + 1) continue;
                const double2 v2 = __ldg(reinterpret_cast<const double2 *>(at_off(xr, mp.o[k])));
                a[k] = v2.x;
                b[k] = v2.y;
            }
            const double2 fv = __ldg(reinterpret_cast<const double2 *>(f + r));
            double s0 = 0.0, s1 = 0.0;
#pragma unroll
            for (int k = 0; k < W; ++k) {
                s0 = __dadd_rn(s0, ((m0 >> k) & 1u) ? __dmul_rn(mp.v[k], a[k]) : 0.0);
                s1 = __dadd_rn(s1, ((m1 >> k) & 1u) ? __dmul_rn(mp.v[k], b[k]) : 0.0);
            }
            s = __dadd_rn(__dadd_rn(0.0, __dsub_rn(fv.x, s0)), __dsub_rn(fv.y, s1));
        } else {
            if (!in) continue;
            s = __dadd_rn(0.0, resid(mm.x, pid[mm.x]));
            if (mm.y >= 0) s = __dadd_rn(s, resid(mm.y, pid[mm.y]));
        }
        if (in) {
            fc[c] = s;
            if (xc0) xc0[c] = __dadd_rn(0.0, __ddiv_rn(__dmul_rn(omega, s), __ldg(dc + c)));
        }
    }
}
