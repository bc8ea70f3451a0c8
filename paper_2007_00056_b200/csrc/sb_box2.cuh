// Two Jacobi sweeps in one launch on the mid-size structured 7-point levels
// (k_cross_box2), included by sb_runtime.cu after sb_tblock.cuh (whose level
// analysis it shares: the class table, TMA tensor maps). EXPERIMENTAL: bitwise
// equal to two sweeps, but measured slower than two k_crosspair / k_rowpat
// launches at every level (C2 L9: 131 vs 106 us from the level down; the
// in-CTA chain load -> sweep -> barrier -> sweep costs ~6 us per launch
// against ~2.1 us per plain kernel), with the boxes loaded by TMA or by
// plain per-thread loads alike.
//
// The mid levels of the 3-D hierarchies (~32K .. 1M rows) are latency-bound:
// a kernel of the graph costs ~2-3.5 us whatever its size (launch, the
// programmatic-dependency wait, one L2 round trip for the gathers). Here a CTA
// owns a TX x TY x TZ box of the grid. ONE TMA load brings x with a 2-wide
// halo and f with a 1-wide halo (out-of-grid elements zero-filled); the CTA
// computes sweep 1 on the box + 1-wide halo into shared memory, then sweep 2
// on the box, and stores x''. One launch replaces two: the second sweep needs
// no grid-wide dependency, only the CTA's own halo (recomputed redundantly).
//
// Bitwise: as k_cross_tb2 -- every row's sum is its CSR sum in column order
// (-P, -N, -1, 0, 1, N, P); an absent slot is an out-of-grid neighbour whose x
// is the TMA's +0.0 and whose table value is +0.0, so it adds +0 * +0 = +0.0
// to a running sum that is never -0.0; x' of an out-of-grid position is +0.0.

#ifndef SB_BOX2_TMA
#define SB_BOX2_TMA 0  // 1: the boxes arrive by TMA (measured slower: one serial ~1.5 us load per CTA)
#endif

struct BoxGeo {
    int nx, ny, nz;
    int nbx, nby, nbz;  // boxes per axis
};

template <int TX, int TY, int TZ> struct Box2 {
    static constexpr int WX = TX + 4, HX = TY + 4, DX = TZ + 4;  // x box (2-wide halo)
    static constexpr int HF = TY + 2, DF = TZ + 2;               // f and x' boxes: WX x HF x DF
    static constexpr int NX = WX * HX * DX, NF = WX * HF * DF;
    static constexpr int TAB = (kTbTab * 8 + 127) & ~127;
    static constexpr size_t smem() {
        return static_cast<size_t>(TAB + 128 + ((NX * 8 + 127) & ~127) + 2 * ((NF * 8 + 127) & ~127));
    }
};

// K rows of one sweep from a shared-memory box: centres at i[k] (plane stride
// SP, line stride SL), values of class c[k] from the table; operands first,
// then the K dependent sums interleaved.
template <int K>
__device__ __forceinline__ void box_rows(const double *tab, const int (&c)[K], const double *b, const int (&i)[K],
                                         int SP, int SL, const double (&fi)[K], double omega, double (&o)[K]) {
    double x[7][K];
#pragma unroll
    for (int k = 0; k < K; ++k) {
        const int j = i[k];
        x[0][k] = b[j - SP];
        x[1][k] = b[j - SL];
        x[2][k] = b[j - 1];
        x[3][k] = b[j];
        x[4][k] = b[j + 1];
        x[5][k] = b[j + SL];
        x[6][k] = b[j + SP];
    }
    double s[K];
#pragma unroll
    for (int k = 0; k < K; ++k) s[k] = 0.0;
#pragma unroll
    for (int j = 0; j < 7; ++j)
#pragma unroll
        for (int k = 0; k < K; ++k) s[k] = __dadd_rn(s[k], __dmul_rn(tab[c[k] * 9 + j], x[j][k]));
#pragma unroll
    for (int k = 0; k < K; ++k)
        o[k] = __dadd_rn(x[3][k], div_rn(__dmul_rn(omega, __dsub_rn(fi[k], s[k])), tab[c[k] * 9 + 7],
                                         tab[c[k] * 9 + 8]));
}

template <int TX, int TY, int TZ>
__global__ void __launch_bounds__(kTbThreads, 3)
    k_cross_box2(const __grid_constant__ CUtensorMap mx, const __grid_constant__ CUtensorMap mf, const BoxGeo g,
                 const double *__restrict__ ctab, double *__restrict__ out, double omega, const double *xglob,
                 const double *fglob) {
    using B = Box2<TX, TY, TZ>;
    constexpr int WX = B::WX, SXP = B::WX * B::HX, SFP = B::WX * B::HF;  // line / plane strides
    constexpr int N1 = (TX + 2) * (TY + 2) * (TZ + 2), N2 = TX * TY * TZ;
    constexpr int K1 = (N1 + kTbThreads - 1) / kTbThreads, K2 = N2 / kTbThreads;
    static_assert(N2 % kTbThreads == 0, "box rows per thread");
    extern __shared__ __align__(128) unsigned char smem[];
    double *tab = reinterpret_cast<double *>(smem);
    uint64_t *bar = reinterpret_cast<uint64_t *>(smem + B::TAB);
    double *xs = reinterpret_cast<double *>(smem + B::TAB + 128);
    double *fs = xs + (((B::NX * 8 + 127) & ~127) / 8);
    double *ps = fs + (((B::NF * 8 + 127) & ~127) / 8);
    const int bx = blockIdx.x % g.nbx, by = (blockIdx.x / g.nbx) % g.nby, bz = blockIdx.x / (g.nbx * g.nby);
    const int x0 = bx * TX, y0 = by * TY, z0 = bz * TZ;
    for (int i = threadIdx.x; i < kTbTab; i += kTbThreads) tab[i] = ctab[i];
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        fence_mbar_init();
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mx)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mf)) : "memory");
    }
    __syncthreads();
    pdl_wait();  // x and f come from the predecessor
#if SB_BOX2_TMA
    if (threadIdx.x == 0) {
        mbar_expect_tx(bar, static_cast<uint32_t>((B::NX + B::NF) * 8));
        tma_load_3d(xs, &mx, x0 - 2, y0 - 2, z0 - 2, bar);
        tma_load_3d(fs, &mf, x0 - 2, y0 - 1, z0 - 1, bar);
    }
    mbar_wait(bar, 0u);
#else
    // every thread loads its share of both boxes (all loads in flight at once:
    // one L2 round trip), out-of-grid elements +0.0
    {
        const double *xg = xglob;
        const double *fg = fglob;
        constexpr int LX = (B::NX + kTbThreads - 1) / kTbThreads, LF = (B::NF + kTbThreads - 1) / kTbThreads;
        double vx[LX], vf[LF];
#pragma unroll
        for (int k = 0; k < LX; ++k) {
            const int q = threadIdx.x + k * kTbThreads;
            const int u = q % B::WX, v = (q / B::WX) % B::HX, w = q / (B::WX * B::HX);
            const int gx = x0 - 2 + u, gy = y0 - 2 + v, gz = z0 - 2 + w;
            const bool ok = q < B::NX && gx >= 0 && gx < g.nx && gy >= 0 && gy < g.ny && gz >= 0 && gz < g.nz;
            vx[k] = ok ? __ldcg(xg + (static_cast<int64_t>(gz) * g.ny + gy) * g.nx + gx) : 0.0;
        }
#pragma unroll
        for (int k = 0; k < LF; ++k) {
            const int q = threadIdx.x + k * kTbThreads;
            const int u = q % B::WX, v = (q / B::WX) % B::HF, w = q / (B::WX * B::HF);
            const int gx = x0 - 2 + u, gy = y0 - 1 + v, gz = z0 - 1 + w;
            const bool ok = q < B::NF && gx >= 0 && gx < g.nx && gy >= 0 && gy < g.ny && gz >= 0 && gz < g.nz;
            vf[k] = ok ? __ldcg(fg + (static_cast<int64_t>(gz) * g.ny + gy) * g.nx + gx) : 0.0;
        }
#pragma unroll
        for (int k = 0; k < LX; ++k)
            if (threadIdx.x + k * kTbThreads < B::NX) xs[threadIdx.x + k * kTbThreads] = vx[k];
#pragma unroll
        for (int k = 0; k < LF; ++k)
            if (threadIdx.x + k * kTbThreads < B::NF) fs[threadIdx.x + k * kTbThreads] = vf[k];
    }
    __syncthreads();
#endif
    // sweep 1 on the box + 1-wide halo: F-position (u, v, w) <-> grid (x0-1+u,
    // y0-1+v, z0-1+w); x box index (w+1) SXP + (v+1) WX + u+1; f / x' index
    // w SFP + v WX + u+1
#pragma unroll
    for (int k0 = 0; k0 < K1; k0 += 4) {  // batches of 4 rows (registers)
        constexpr int KB = 4;
        int c[KB], ix[KB], jf[KB];
        bool ok[KB], in[KB];
        double fi[KB];
#pragma unroll
        for (int k = 0; k < KB; ++k) {
            const int q = threadIdx.x + (k0 + k) * kTbThreads;
            in[k] = k0 + k < K1 && q < N1;
            const int p = min(q, N1 - 1);
            const int u = p % (TX + 2), v = (p / (TX + 2)) % (TY + 2), w = p / ((TX + 2) * (TY + 2));
            const int gx = x0 - 1 + u, gy = y0 - 1 + v, gz = z0 - 1 + w;
            ok[k] = in[k] && gx >= 0 && gx < g.nx && gy >= 0 && gy < g.ny && gz >= 0 && gz < g.nz;
            c[k] = ok[k] ? tb_cls(gx, g.nx) + 3 * tb_cls(gy, g.ny) + 9 * tb_cls(gz, g.nz) : 13;
            ix[k] = (w + 1) * SXP + (v + 1) * WX + u + 1;
            jf[k] = w * SFP + v * WX + u + 1;
            fi[k] = fs[jf[k]];
        }
        double o[KB];
        box_rows<KB>(tab, c, xs, ix, SXP, WX, fi, omega, o);
#pragma unroll
        for (int k = 0; k < KB; ++k)
            if (in[k]) ps[jf[k]] = ok[k] ? o[k] : 0.0;
    }
    __syncthreads();
    pdl_trigger();
    // sweep 2 on the box -> HBM
    {
        int c[K2], jf[K2];
        bool ok[K2];
        double fi[K2];
        int64_t go[K2];
#pragma unroll
        for (int k = 0; k < K2; ++k) {
            const int p = threadIdx.x + k * kTbThreads;
            const int uu = p % TX, vv = (p / TX) % TY, ww = p / (TX * TY);
            const int gx = x0 + uu, gy = y0 + vv, gz = z0 + ww;
            ok[k] = gx < g.nx && gy < g.ny && gz < g.nz;
            c[k] = ok[k] ? tb_cls(gx, g.nx) + 3 * tb_cls(gy, g.ny) + 9 * tb_cls(gz, g.nz) : 13;
            jf[k] = (ww + 1) * SFP + (vv + 1) * WX + uu + 2;
            fi[k] = fs[jf[k]];
            go[k] = (static_cast<int64_t>(gz) * g.ny + gy) * g.nx + gx;
        }
        double o[K2];
        box_rows<K2>(tab, c, ps, jf, SFP, WX, fi, omega, o);
#pragma unroll
        for (int k = 0; k < K2; ++k)
            if (ok[k]) out[go[k]] = o[k];
    }
}

using Box2Kernel = void (*)(CUtensorMap, CUtensorMap, BoxGeo, const double *, double *, double, const double *,
                           const double *);
// instances: TX = 16 (box 16 x 8 x 8) or 8 (box 8 x 16 x 8), 1024 rows per CTA
static Box2Kernel box2_kernel(int TX) {
#if SB_EXPERIMENTAL
    return TX >= 16 ? k_cross_box2<16, 8, 8> : k_cross_box2<8, 16, 8>;
#else
    (void)TX;
    return nullptr;
#endif
}
static size_t box2_smem(int TX) { return TX >= 16 ? Box2<16, 8, 8>::smem() : Box2<8, 16, 8>::smem(); }
