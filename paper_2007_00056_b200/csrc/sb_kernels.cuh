// sm_100a kernels of the solve phase. Every kernel is HBM-bound fp64 sparse /
// vector work (arithmetic intensity ~0.13-0.17 flop/B); tensor cores do not
// apply. Design rules:
//  * CSR tiles of <=256 consecutive rows are staged into shared memory with
//    one TMA bulk copy (cp.async.bulk + mbarrier) for values and one for
//    column indices: fully coalesced 16-byte-granular HBM streams with no
//    padding and no format conversion of the reference's CSR.
//  * One thread per row then walks its row sequentially from shared memory in
//    CSR order, sum = 0.0; sum += v*x (explicit __dmul_rn/__dadd_rn: no FMA),
//    exactly the reference's spmv (inc/csr.hpp:185-191), so SpMV, residual
//    and Jacobi sweeps are bit-identical to the reference.
//  * Reductions are deterministic: fixed shuffle tree per block, per-block
//    partials, the last block to finish folds the partials in fixed order and
//    runs the Krylov scalar logic in its epilogue (no extra launch, no atomics
//    on doubles), then sets the CUDA-graph conditional handles that drive the
//    device-side iteration loop.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace sb {

constexpr int kTileRows = 256;   // rows per CSR tile == threads per CTA
constexpr int kVecThreads = 256;

// Krylov / AMG scalar state, device resident (one per context).
struct DevState {
    double tol, r0, rn, rz, pAp, alpha, beta;
    double rho, denom, omega, sn, true_res;
    double part[2];  // multi-rank: this rank's reduction totals
    double red[2];   // multi-rank: allreduced totals
    int iter, max_iters, done, term, status, half, hist_cap;
    int x_pending;  // PCG: x += alpha p of this iteration not applied yet (k_pcg_update_r -> k_xpay_x / k_x_final)
    unsigned long long t0;
    double *hist_r;
    double *hist_t;
};

enum EpOp : int {
    EP_NONE = 0,
    EP_STORE,        // st->true_res = sqrt(a)
    EP_INIT_NORM,    // rn0 = sqrt(a); record; converged?; max_iters == 0?
    EP_PCG_RZ0,      // rz = a
    EP_PCG_PAP,      // pAp = a; breakdown or alpha
    EP_PCG_RN,       // rn, record, stop tests
    EP_PCG_RZ,       // beta = a / rz; rz = a
    EP_BI_RHO0,      // rho = a (+ breakdown test)
    EP_BI_DENOM,     // denom = a; breakdown or alpha
    EP_BI_SN,        // sn = sqrt(a); half-step exit test
    EP_BI_AS,        // a = (As,As), b = (As,s); breakdown or omega
    EP_BI_RN_RHO,    // rn = sqrt(a), rho' = b; stop tests; beta; rho
    EP_AMG_RN,       // amg_solve: rn, record, divergence / convergence
    EP_PARTIAL,      // multi-rank: store this rank's totals (logic runs after the allreduce)
};

// Conditional-handle set performed by a reduction epilogue: every listed
// handle receives !st->done.
struct CondSet {
    unsigned long long h[2];
    int n;
};

struct Red {
    double *partials;   // 2 * gridDim.x
    unsigned *counter;  // zero between uses
    DevState *st;
    int op;
    int nval;           // 0, 1 or 2 reduced values
    const double *w0;   // value 0 = sum out_i * w0_i (or custom, see kernels)
    const double *w1;   // value 1 = sum out_i * w1_i
    CondSet cs;
    // k_crosspair M_RESID_RESTRICT on a row-pattern coarse level: a_cc = pdg[pid[c]]
    const uint8_t *pid = nullptr;
    const double *pdg = nullptr;
};

} // namespace sb
