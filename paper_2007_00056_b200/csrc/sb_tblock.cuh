// Two Jacobi sweeps in ONE pass over HBM on 7-point cross levels (temporal
// blocking), included by sb_runtime.cu after the row-pattern kernels.
//
// A level qualifies when it is a structured nx x ny x nz grid (node m =
// (iz*ny + iy)*nx + ix, main pattern (-P, -N, -1, 0, 1, N, P) with N = nx,
// P = nx*ny) whose row pattern is a function of the row's boundary class
// (low / interior / high in each dimension, 27 classes) and whose absent
// slots are exactly the out-of-grid neighbours. Every level of the 7-point
// BASELINE hierarchies above the coarsest few is one (node-HEM pairs rows
// along one axis at a time; verified row by row on the host, build_tb).
//
// The CTA owns a TX x TY column of the grid and marches it through a chunk of
// z-planes. Each step, TMA (cp.async.bulk.tensor, 3-D tiles, out-of-grid
// elements zero-filled) brings one plane of x with a 2-wide halo and one plane
// of f with a 1-wide halo into shared-memory rings; the CTA computes sweep 1
// (x') on the plane below over the tile + 1-wide halo and sweep 2 (x'') on the
// plane below that over the tile, and stores x'' to HBM. (A TMA tile's first
// innermost element must sit on a 16-byte boundary, so f is loaded with the
// same 2-wide x-halo as x: tiles start at even columns.) Per row the pass
// streams x (8 B) + f (8 B) + x'' (8 B) for TWO sweeps instead of 2 x 25 B.
//
// Bitwise: each row's sum is the reference's CSR sum in column order
// (-P, -N, -1, 0, 1, N, P) with __dmul_rn / __dadd_rn; an absent slot is an
// out-of-grid neighbour whose x is the TMA's +0.0 fill and whose table value
// is +0.0, so it adds +0 * +0 = +0.0 to a running sum that is never -0.0 (it
// starts at +0.0): no bit changes, and an inf / NaN of an in-grid x can never
// meet an absent slot. The update is fin()'s x + RN(w (f - sum) / a_ii).

constexpr int kTbThreads = 256;
constexpr int kTbR = 4;  // ring depth of x, f and x' planes (see the step schedule in k_cross_tb2)
constexpr int kTbClasses = 27;
constexpr int kTbTab = kTbClasses * 9;  // per class: 7 values (CSR order, +0.0 where absent), a_ii, RN(1/a_ii)

struct TbGeo {
    int nx, ny, nz;
    int TX, TY, ZL;  // tile (x, y) of the kernel instance and z-chunk length
    int ntx, nty;    // tiles per plane in x / y
};

__host__ __device__ __forceinline__ int tb_a128(int b) { return (b + 127) & ~127; }
// x slot: (TX + 4) x (TY + 4) from (x0 - 2, y0 - 2); f and x' slots: (TX + 4) x (TY + 2) from (x0 - 2, y0 - 1)
__host__ __device__ __forceinline__ size_t tb_smem_bytes(int TX, int TY) {
    const int sx = tb_a128((TX + 4) * (TY + 4) * 8), sf = tb_a128((TX + 4) * (TY + 2) * 8);
    return static_cast<size_t>(tb_a128(kTbTab * 8) + 128 + kTbR * (sx + 2 * sf));
}

__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *m, int x, int y, int z, uint64_t *bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(x), "r"(y), "r"(z), "r"(smem_u32(bar))
        : "memory");
}

// boundary class of coordinate i on an axis of n points
__device__ __forceinline__ int tb_cls(int i, int n) { return i == 0 ? 0 : (i == n - 1 ? 2 : 1); }

__device__ __forceinline__ double2 lds2(const double *p) { return *reinterpret_cast<const double2 *>(p); }

// One Jacobi row: x values of slots (-P, -N, -1, 0, 1, N, P), CSR order, a = class values.
template <typename A>
__device__ __forceinline__ double tb_eval(const A &a, double xm, double xs, double xw, double xc, double xe,
                                          double xn, double xp, double fi, double omega) {
    double s = 0.0;
    s = __dadd_rn(s, __dmul_rn(a[0], xm));
    s = __dadd_rn(s, __dmul_rn(a[1], xs));
    s = __dadd_rn(s, __dmul_rn(a[2], xw));
    s = __dadd_rn(s, __dmul_rn(a[3], xc));
    s = __dadd_rn(s, __dmul_rn(a[4], xe));
    s = __dadd_rn(s, __dmul_rn(a[5], xn));
    s = __dadd_rn(s, __dmul_rn(a[6], xp));
    return __dadd_rn(xc, div_rn(__dmul_rn(omega, __dsub_rn(fi, s)), a[7], a[8]));
}

// A row pair (columns c, c+1 of a plane triple): m / p = the pair in the planes
// below / above, c2 = the pair itself, w = (c-2, c-1), e = (c+2, c+3), s / n =
// the pair in the lines below / above.
template <typename A, typename B>
__device__ __forceinline__ double2 tb_pair(const A &a0, const B &a1, double2 m, double2 w, double2 c2,
                                           double2 e, double2 sv, double2 nv, double2 p, double2 f, double omega) {
    return make_double2(tb_eval(a0, m.x, sv.x, w.y, c2.x, c2.y, nv.x, p.x, f.x, omega),
                        tb_eval(a1, m.y, sv.y, c2.x, c2.y, e.x, nv.y, p.y, f.y, omega));
}

// TX: tile width (64, 32, 16 or 8), TY = 512 / TX: thread (cp, cv) owns the row
// pair at columns x0 + 2cp, +1 of line y0 + cv in every plane, for both sweeps.
// Step t (one CTA barrier per step):
//   x(t) = x plane z0-2+t arrives (TMA); every thread rolls its own pair of
//   x(t) into registers (planes q-1, q, q+1 of sweep 1 never touch shared
//   memory twice);
//   sweep 1 on plane q = z0-3+t (t >= 2) over the tile + 1-wide halo -> x'
//   slot t (and the thread's x' registers); the halo lines and columns are
//   computed by threads 0 .. 2 TX/2 + 2 (TY + 2);
//   sweep 2 on plane q2 = q - 2 (t >= 5) from x' slots t-3 .. t-1 (own pair
//   from registers) -> HBM; f of q2 comes from registers too.
// Rings of 4: x(j) is read at steps j .. j+2, f(j) at step j+2, x'(j) at steps
// j+1 .. j+3, so after step t the slots of x(t-2) / f(t-2) take x(t+2) / f(t+2).
template <int TX>
__global__ void __launch_bounds__(kTbThreads, 2)
    k_cross_tb2(const __grid_constant__ CUtensorMap mx, const __grid_constant__ CUtensorMap mf, const TbGeo g,
                const double *__restrict__ ctab, double *__restrict__ out, double omega) {
    constexpr int TXP = TX / 2, TY = kTbThreads / TXP;
    constexpr int W = TX + 4;  // row stride (doubles) of every slot
    constexpr int SX = (W * (TY + 4) * 8 + 127) & ~127, SF = (W * (TY + 2) * 8 + 127) & ~127;
    constexpr uint32_t XB = W * (TY + 4) * 8, FB = W * (TY + 2) * 8;
    constexpr int TABB = (kTbTab * 8 + 127) & ~127;
    extern __shared__ __align__(128) unsigned char smem[];
    double *tab = reinterpret_cast<double *>(smem);
    uint64_t *barx = reinterpret_cast<uint64_t *>(smem + TABB);
    uint64_t *barf = barx + kTbR;
    unsigned char *xr = smem + TABB + 128;
    unsigned char *fr = xr + kTbR * SX;
    unsigned char *pr = fr + kTbR * SF;
    auto XS = [&](int step) { return reinterpret_cast<const double *>(xr + (step & (kTbR - 1)) * SX); };
    auto FS = [&](int step) { return reinterpret_cast<const double *>(fr + (step & (kTbR - 1)) * SF); };
    auto PS = [&](int step) { return reinterpret_cast<double *>(pr + (step & (kTbR - 1)) * SF); };

    const int tile = blockIdx.x % (g.ntx * g.nty), chunk = blockIdx.x / (g.ntx * g.nty);
    const int x0 = (tile % g.ntx) * TX, y0 = (tile / g.ntx) * TY;
    const int z0 = chunk * g.ZL, z1 = min(g.nz, z0 + g.ZL);
    const int nx_steps = (z1 - z0) + 4, nf_steps = (z1 - z0) + 2, nsteps = (z1 - z0) + 5;

    for (int i = threadIdx.x; i < kTbTab; i += kTbThreads) tab[i] = ctab[i];
    if (threadIdx.x == 0) {
        for (int i = 0; i < 2 * kTbR; ++i) mbar_init(barx + i, 1);
        fence_mbar_init();
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mx)) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&mf)) : "memory");
    }
    double ci[9];
#pragma unroll
    for (int k = 0; k < 9; ++k) ci[k] = __ldg(ctab + 13 * 9 + k);
    // own pair
    const int cp = threadIdx.x % TXP, cv = threadIdx.x / TXP;
    const int c = 2 * cp + 2;          // slot column of the pair (x, f and x' slots start at x0 - 2)
    const int gx = x0 + 2 * cp, gy = y0 + cv;
    const bool pin = gx < g.nx && gy < g.ny;  // nx even: a pair is all in or all out
    const int cxa = tb_cls(gx, g.nx), cxb = tb_cls(gx + 1, g.nx), cyy = tb_cls(gy, g.ny);
    const bool pint = pin && cxa == 1 && cxb == 1 && cyy == 1;
    const int ox = (cv + 2) * W + c;   // own pair in an x slot (line gy - y0 + 2)
    const int of = (cv + 1) * W + c;   // own pair in an f / x' slot (line gy - y0 + 1)
    // extra sweep-1 work: the halo lines (slot lines 0 and TY + 1) as pairs on
    // threads [0, TX), the halo columns (slot columns 1 and TX + 2) as single
    // rows on threads [TX, TX + 2 (TY + 2))
    const bool ep = threadIdx.x < TX;
    const int el = threadIdx.x < TXP ? 0 : TY + 1;                     // f / x' slot line
    const int egx = x0 + 2 * cp, egy = y0 - 1 + el;
    const bool epin = ep && egx < g.nx && egy >= 0 && egy < g.ny;
    const int ecxy = epin ? tb_cls(egy, g.ny) * 3 : 0;
    const int eh = threadIdx.x - TX;
    const bool hs = eh >= 0 && eh < 2 * (TY + 2);
    const int hl = hs ? eh % (TY + 2) : 0, hcol = hs && eh >= TY + 2 ? TX + 2 : 1;  // slot line / column
    const int hgx = x0 - 2 + hcol, hgy = y0 - 1 + hl;
    const bool hin = hs && hgx >= 0 && hgx < g.nx && hgy >= 0 && hgy < g.ny;
    const int hcxy = hin ? tb_cls(hgx, g.nx) + 3 * tb_cls(hgy, g.ny) : 0;
    const int64_t P = static_cast<int64_t>(g.nx) * g.ny;
    double *outp = out + static_cast<int64_t>(gy) * g.nx + gx;  // + q2 * P
    __syncthreads();
    pdl_wait();  // x and f come from the predecessor
    auto load_x = [&](int step) {
        uint64_t *b = barx + (step & (kTbR - 1));
        mbar_expect_tx(b, XB);
        tma_load_3d(const_cast<double *>(XS(step)), &mx, x0 - 2, y0 - 2, z0 - 2 + step, b);
    };
    auto load_f = [&](int step) {
        uint64_t *b = barf + (step & (kTbR - 1));
        mbar_expect_tx(b, FB);
        tma_load_3d(const_cast<double *>(FS(step)), &mf, x0 - 2, y0 - 1, z0 - 1 + step, b);
    };
    if (threadIdx.x == 0) {  // fill the rings
        for (int j = 0; j < kTbR && j < nx_steps; ++j) load_x(j);
        for (int j = 0; j < kTbR && j < nf_steps; ++j) load_f(j);
    }
    // class values of a row (shared-memory table; the fast paths use ci)
    auto cls_vals = [&](int cls) -> const double * { return tab + cls * 9; };
    double2 xqm = make_double2(0.0, 0.0), xq = xqm;       // own pair, x planes q-1, q
    double2 pr0 = xqm, pr1 = xqm, pr2 = xqm;              // own pair, x' of steps t-3, t-2, t-1
    double2 fr0 = xqm, fr1 = xqm;                         // own pair, f of steps t-2, t-1 (planes q-2, q-1)
    for (int t = 0; t < nsteps; ++t) {
        const bool s1 = t >= 2 && t < nx_steps, s2 = t >= 5;
        const int q = z0 - 3 + t, q2 = q - 2;
        if (t < nx_steps) mbar_wait(barx + (t & (kTbR - 1)), static_cast<uint32_t>((t / kTbR) & 1));
        if (s1) mbar_wait(barf + ((t - 2) & (kTbR - 1)), static_cast<uint32_t>(((t - 2) / kTbR) & 1));
        const double *xa = XS(t - 2), *xb = XS(t - 1), *xn = XS(t);
        const double2 xqp = t < nx_steps ? lds2(xn + ox) : make_double2(0.0, 0.0);
        double2 pnew = make_double2(0.0, 0.0), fq = make_double2(0.0, 0.0);
        if (s1) {
            const double *f1 = FS(t - 2);
            double *po = PS(t);
            const int cz = tb_cls(q, g.nz);
            const bool qin = q >= 0 && q < g.nz;
            fq = lds2(f1 + of);
            const double2 w = lds2(xb + ox - 2), e = lds2(xb + ox + 2), sv = lds2(xb + ox - W), nv = lds2(xb + ox + W);
            if (__all_sync(0xffffffffu, pint && cz == 1)) {
                pnew = tb_pair(ci, ci, xqm, w, xq, e, sv, nv, xqp, fq, omega);
            } else if (qin && pin) {
                pnew = tb_pair(cls_vals(cxa + 3 * cyy + 9 * cz), cls_vals(cxb + 3 * cyy + 9 * cz), xqm, w, xq, e, sv,
                               nv, xqp, fq, omega);
            }
            *reinterpret_cast<double2 *>(po + of) = pnew;
            if (ep) {  // halo line pair
                const int ex = (el + 1) * W + c;
                double2 o = make_double2(0.0, 0.0);
                if (qin && epin) {
                    const int cxe = tb_cls(egx, g.nx), cxf = tb_cls(egx + 1, g.nx);
                    o = tb_pair(cls_vals(cxe + ecxy + 9 * cz), cls_vals(cxf + ecxy + 9 * cz), lds2(xa + ex),
                                lds2(xb + ex - 2), lds2(xb + ex), lds2(xb + ex + 2), lds2(xb + ex - W), lds2(xb + ex + W),
                                lds2(xn + ex), lds2(f1 + el * W + c), omega);
                }
                *reinterpret_cast<double2 *>(po + el * W + c) = o;
            }
            if (hs) {  // halo column row
                const int hx = (hl + 1) * W + hcol;
                double o = 0.0;
                if (qin && hin)
                    o = tb_eval(cls_vals(hcxy + 9 * cz), xa[hx], xb[hx - W], xb[hx - 1], xb[hx], xb[hx + 1], xb[hx + W],
                                xn[hx], f1[hl * W + hcol], omega);
                po[hl * W + hcol] = o;
            }
        }
        if (s2) {  // sweep 2 on plane q2 -> HBM
            const double *pc = PS(t - 2);
            const double2 w = lds2(pc + of - 2), e = lds2(pc + of + 2), sv = lds2(pc + of - W), nv = lds2(pc + of + W);
            const int cz = tb_cls(q2, g.nz);
            double2 o;
            if (__all_sync(0xffffffffu, pint && cz == 1)) {
                o = tb_pair(ci, ci, pr0, w, pr1, e, sv, nv, pr2, fr0, omega);
            } else {
                o = tb_pair(cls_vals(cxa + 3 * cyy + 9 * cz), cls_vals(cxb + 3 * cyy + 9 * cz), pr0, w, pr1, e, sv, nv,
                            pr2, fr0, omega);
            }
            if (pin) *reinterpret_cast<double2 *>(outp + static_cast<int64_t>(q2) * P) = o;
        }
        // roll the own-pair registers
        xqm = xq;
        xq = xqp;
        pr0 = pr1;
        pr1 = pr2;
        pr2 = pnew;
        fr0 = fr1;
        fr1 = fq;
        __syncthreads();
        if (threadIdx.x == 0) {  // x(t-2) and f(t-2) are consumed
            if (t + 2 < nx_steps && t >= 2) load_x(t + 2);
            if (t + 2 < nf_steps && t >= 2) load_f(t + 2);
        }
        if (t + 2 == nsteps) pdl_trigger();
    }
}

using TbKernel = void (*)(CUtensorMap, CUtensorMap, TbGeo, const double *, double *, double);
static TbKernel tb_kernel(int TX) {
#if SB_EXPERIMENTAL
    return TX == 64 ? k_cross_tb2<64> : TX == 32 ? k_cross_tb2<32> : TX == 16 ? k_cross_tb2<16> : k_cross_tb2<8>;
#else
    (void)TX;
    return nullptr;
#endif
}
