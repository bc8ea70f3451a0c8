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
// CTA before the dependency wait): f64 val[np][W] | f64 diag[np] |
// f64 rdiag[np] | int32 off[np][W] | uint8 len[np] (padded to 16).

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
    return (static_cast<size_t>(np) * w * 12 + static_cast<size_t>(np) * 16 + static_cast<size_t>(np) + 15) & ~size_t(15);
}

#ifndef SB_PAT_MINB_WIDE
#define SB_PAT_MINB_WIDE 2
#endif
#ifndef SB_PAT_CHUNK
#define SB_PAT_CHUNK 28
#endif
#ifndef SB_PAT_MINB
#define SB_PAT_MINB 4
#endif
// wide rows (27-point levels) keep all W gathers in flight: more registers, 3 CTAs/SM
template <int MODE, int NV, int W>
__global__ void __launch_bounds__(kPatThreads, W <= 8 ? SB_PAT_MINB : SB_PAT_MINB_WIDE)
    k_rowpat(int n, const uint8_t *__restrict__ pid, int np, const unsigned char *__restrict__ table,
             const double *__restrict__ x, const double *__restrict__ f, double *__restrict__ out, double omega,
             const int *skip, Aux aux, Red red) {
    extern __shared__ __align__(16) unsigned char smem[];
    double acc[NV > 0 ? NV : 1];
#pragma unroll
    for (int v = 0; v < (NV > 0 ? NV : 1); ++v) acc[v] = 0.0;
    const int tb = static_cast<int>(pat_table_bytes(np, W));
    {  // constant table: before the dependency wait (overlaps the predecessor's tail)
        const uint4 *src = reinterpret_cast<const uint4 *>(table);
        uint4 *dst = reinterpret_cast<uint4 *>(smem);
        for (int i = threadIdx.x; i < tb / 16; i += blockDim.x) dst[i] = src[i];
    }
    __syncthreads();
    constexpr int kPatRows = PatRows<W>::value;
    const double *sval = reinterpret_cast<const double *>(smem);
    const double *sdg = sval + static_cast<size_t>(np) * W;
    const double *sry = sdg + np;
    const int32_t *soff = reinterpret_cast<const int32_t *>(sry + np);
    const uint8_t *slen = reinterpret_cast<const uint8_t *>(soff + static_cast<size_t>(np) * W);
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
        // wide rows (27-point levels): one row per thread, the gathers in chunks
        // of SB_PAT_CHUNK (registers for more resident warps), sums in slot order
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
                double sum = 0.0;
#pragma unroll
                for (int c0 = 0; c0 < W; c0 += SB_PAT_CHUNK) {
                    double xv[SB_PAT_CHUNK];
#pragma unroll
                    for (int k = 0; k < SB_PAT_CHUNK; ++k)
                        if (c0 + k < W) xv[k] = __ldg(at_off(xr, soff[p * W + c0 + k]));
#pragma unroll
                    for (int k = 0; k < SB_PAT_CHUNK; ++k)
                        if (c0 + k < W) sum = __dadd_rn(sum, __dmul_rn(sval[p * W + c0 + k], xv[k]));
                }
                const int len = slen[p];
                if (len < W && !isfinite(xi)) {  // exact replay for a non-finite own x (see below)
                    sum = 0.0;
                    for (int k = 0; k < len; ++k) sum = __dadd_rn(sum, __dmul_rn(sval[p * W + k], __ldg(xr + soff[p * W + k])));
                }
                if (row < n) {
                    double o;
                    if constexpr (MODE == M_SPMV) o = sum;
                    else if constexpr (MODE == M_RESID) o = __dsub_rn(fi, sum);
                    else o = __dadd_rn(xi, div_rn(__dmul_rn(omega, __dsub_rn(fi, sum)), sdg[p], sry[p]));
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
            double fv[kPatRows], xo[kPatRows];  // rhs and own iterate, loaded with the gathers
#pragma unroll
            for (int q = 0; q < kPatRows; ++q) {
                const int rq = row[q] < n ? row[q] : n - 1;
                const double *xr = x + rq;
#pragma unroll
                for (int k = 0; k < W; ++k) {
                    const int off = soff[p[q] * W + k];
                    if constexpr (MODE == M_JACOBI || MODE == M_RESID || MODE == M_SPMV) xv[q][k] = __ldg(at_off(xr, off));
                    else xv[q][k] = xval<MODE, false>(rq + off, x, f, aux, omega);
                }
                fv[q] = (MODE == M_SPMV) ? 0.0 : __ldg(f + rq);
                xo[q] = (MODE >= M_JACOBI) ? xval<MODE, false>(rq, x, f, aux, omega) : 0.0;
            }
#pragma unroll
            for (int q = 0; q < kPatRows; ++q) {
                if (row[q] >= n) continue;
                const int len = slen[p[q]];
                // Padding slots hold value +0.0 at offset 0 (the row itself): 0 * x_i
                // is +-0 and sum + (+-0) == sum bit for bit (sum is never -0), so
                // the unmasked sum equals the reference's unless x_i is inf / NaN
                // (0 * inf = NaN); only then replay the row with masked slots.
                double sum = 0.0;
#pragma unroll
                for (int k = 0; k < W; ++k) sum = __dadd_rn(sum, __dmul_rn(sval[p[q] * W + k], xv[q][k]));
                if (len < W && !isfinite(xv[q][W - 1])) {
                    sum = 0.0;
#pragma unroll
                    for (int k = 0; k < W; ++k) add_if(sum, __dmul_rn(sval[p[q] * W + k], xv[q][k]), k < len);
                }
                double o;
                if constexpr (MODE == M_SPMV) {
                    o = sum;
                } else if constexpr (MODE == M_RESID) {
                    o = __dsub_rn(fv[q], sum);
                } else {
                    o = __dadd_rn(xo[q], div_rn(__dmul_rn(omega, __dsub_rn(fv[q], sum)), sdg[p[q]], sry[p[q]]));
                }
                out[row[q]] = o;
                if (NV >= 1) acc[0] += o * (red.w0 ? (red.w0 == f ? fv[q] : red.w0[row[q]]) : o);
                if (NV >= 2) acc[NV >= 2 ? 1 : 0] += o * (red.w1 ? red.w1[row[q]] : o);
            }
        }
    }
    if constexpr (NV > 0) finish_reduction<NV>(red, acc);
}

// Residual + restriction fused for a row-pattern level (one launch and no r
// vector): thread c evaluates r_m = f_m - A_m x for the members m0 < m1 of
// coarse row c in the reference's order and writes f_c = (0 + r_m0) + r_m1
// (csr.hpp:267-274 then the unit-P spmv_transpose, csr.hpp:232-239); with
// xc0, also the coarse level's first sweep from 0, x0_c = 0 + (w f_c) / a_cc.
template <int W>
__device__ __forceinline__ double pat_resid_row(int m, int p, const double *sval, const int32_t *soff,
                                                const uint8_t *slen, const double *__restrict__ x,
                                                const double *__restrict__ f) {
    double xv[W];
#pragma unroll
    for (int k = 0; k < W; ++k) xv[k] = __ldg(at_off(x + m, soff[p * W + k]));
    const double fm = f[m];
    double sum = 0.0;
#pragma unroll
    for (int k = 0; k < W; ++k) sum = __dadd_rn(sum, __dmul_rn(sval[p * W + k], xv[k]));
    const int len = slen[p];
    if (len < W && !isfinite(xv[W - 1])) {  // see k_rowpat: exact replay for a non-finite own x
        sum = 0.0;
#pragma unroll
        for (int k = 0; k < W; ++k) add_if(sum, __dmul_rn(sval[p * W + k], xv[k]), k < len);
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
    const int tb = static_cast<int>(pat_table_bytes(np, W));
    {
        const uint4 *src = reinterpret_cast<const uint4 *>(table);
        uint4 *dst = reinterpret_cast<uint4 *>(smem);
        for (int i = threadIdx.x; i < tb / 16; i += blockDim.x) dst[i] = src[i];
    }
    __syncthreads();
    const double *sval = reinterpret_cast<const double *>(smem);
    const double *sdg = sval + static_cast<size_t>(np) * W;
    const double *sry = sdg + np;
    const int32_t *soff = reinterpret_cast<const int32_t *>(sry + np);
    const uint8_t *slen = reinterpret_cast<const uint8_t *>(soff + static_cast<size_t>(np) * W);
    (void)sdg;
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
    for (int c = c0; c < nc; c += gridDim.x * blockDim.x) {
        if (c != c0) {
            mm = mem[c];
            p0 = pid[mm.x];
            if (mm.y >= 0) p1 = pid[mm.y];
            if (xc0) d = dc[c];
        }
        double s = __dadd_rn(0.0, pat_resid_row<W>(mm.x, p0, sval, soff, slen, x, f));
        if (mm.y >= 0) s = __dadd_rn(s, pat_resid_row<W>(mm.y, p1, sval, soff, slen, x, f));
        fc[c] = s;
        if (xc0) xc0[c] = __dadd_rn(0.0, __ddiv_rn(__dmul_rn(omega, s), d));
    }
}
