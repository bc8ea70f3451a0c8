// Internal host-side structures shared by the host setup (sb_host.cpp) and the
// device runtime (sb_runtime.cu). Not part of the C ABI.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "sparsh_b200.h"

namespace sb {

// Reference error classes -> C-ABI status codes (include/sparsh_b200.h).
struct invalid_argument : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct runtime_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};
struct cuda_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

void set_error(const std::string &msg);

// Host CSR with int64 row offsets (int32 columns, f64 values). rp32 mirrors rp
// when nnz fits int32 so sb_hier_level can hand out reference-layout views.
struct HostCsr {
    int64_t n = 0, ncols = 0;
    std::vector<int64_t> rp{0};
    std::vector<int32_t> rp32{0};
    std::vector<int32_t> ci;
    std::vector<double> v;
    int64_t nnz() const { return static_cast<int64_t>(ci.size()); }
    void sync_rp32();
};

struct HostLevel {
    HostCsr A;
    std::vector<int32_t> agg; // fine_to_coarse (empty on the coarsest level)
    int64_t n_coarse = -1;
};

struct Hier {
    std::vector<HostLevel> levels;
    bool stalled = false;
    // Coarsest level: dense LU exactly as the reference factors it
    // (inc/coarse_solver.hpp:129-166) and the inverse built column by column
    // with the reference's solve order (inc/coarse_solver.hpp:168-182).
    int64_t nc = 0;
    std::vector<double> lu;
    std::vector<int32_t> perm;
    std::vector<double> inv; // row-major nc x nc
    long symbolic = 0, numeric = 0;
    mutable long solves = 0;
};

HostCsr csr_from_abi(const sb_csr &A);
void validate_csr(const HostCsr &A);
std::vector<int32_t> node_hem(const HostCsr &A, int64_t *n_coarse);
HostCsr galerkin(const HostCsr &A, const std::vector<int32_t> &agg, int64_t nc, int threads);
// the same product computed on CUDA device `device` (sb_galerkin.cu), bit-identical
HostCsr galerkin_gpu(const HostCsr &A, const std::vector<int32_t> &agg, int64_t nc, int device);
HostCsr stencil27(int64_t nx, int64_t ny, int64_t nz, double diag, double off);
void factor_coarse(Hier &h);
Hier *build_hierarchy(HostCsr A0, const sb_setup_opts &o);
Hier *hier_of(sb_hier h);

// Maps the reference's exception classes onto C-ABI status codes.
template <typename Fn> int guard(Fn &&fn) {
    try {
        fn();
        return SB_OK;
    } catch (const sb::invalid_argument &e) {
        set_error(e.what());
        return SB_EINVAL;
    } catch (const sb::cuda_error &e) {
        set_error(e.what());
        return SB_ECUDA;
    } catch (const std::invalid_argument &e) {
        set_error(e.what());
        return SB_EINVAL;
    } catch (const std::exception &e) {
        set_error(e.what());
        return SB_ERUNTIME;
    }
}

} // namespace sb
