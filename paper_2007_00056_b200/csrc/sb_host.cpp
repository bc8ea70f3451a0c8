// Host setup for the B200 solve phase: CSR validation, node-HEM aggregation,
// the Galerkin coarse operator, the coarse dense LU + inverse, the hierarchy
// loop, and the synthetic problem generators. Everything here must reproduce
// the reference's bits (aggregates, coarse sparsity AND values), because a
// 1-ulp difference flips node-HEM ties on the next level (SURVEY.md §7 "hard
// parts" 1). The arithmetic therefore follows the reference's evaluation order
// entry by entry; parallelism is only used where it cannot change an order
// (independent coarse rows of the Galerkin product).
//
// Build with -ffp-contract=off (the reference is compiled without FMA).

#include <algorithm>
#include <cctype>
#include <fstream>
#include <sstream>
#include <cmath>
#include <cstring>
#include <mutex>
#include <numeric>
#include <random>
#include <thread>

#include "sb_internal.h"

namespace sb {

void HostCsr::sync_rp32() {
    if (nnz() <= INT32_MAX && n < INT32_MAX) {
        rp32.resize(rp.size());
        for (size_t i = 0; i < rp.size(); ++i) rp32[i] = static_cast<int32_t>(rp[i]);
    } else {
        rp32.clear();
    }
}

HostCsr csr_from_abi(const sb_csr &A) {
    if (A.nrows < 0 || A.ncols < 0) throw invalid_argument("CsrMatrix: negative dimension");
    if ((A.row_ptr32 == nullptr) == (A.row_ptr64 == nullptr))
        throw invalid_argument("sb_csr: set exactly one of row_ptr32 / row_ptr64");
    HostCsr M;
    M.n = A.nrows;
    M.ncols = A.ncols;
    M.rp.resize(static_cast<size_t>(A.nrows) + 1);
    for (int64_t i = 0; i <= A.nrows; ++i)
        M.rp[i] = A.row_ptr32 ? static_cast<int64_t>(A.row_ptr32[i]) : A.row_ptr64[i];
    if (M.rp[0] != 0) throw invalid_argument("CsrMatrix: row_ptr[0] != 0");
    const int64_t nnz = M.rp[A.nrows];
    if (nnz < 0) throw invalid_argument("CsrMatrix: row_ptr not monotone");
    if (nnz > 0 && (A.col_idx == nullptr || A.values == nullptr))
        throw invalid_argument("CsrMatrix: col/value arrays missing");
    M.ci.assign(A.col_idx, A.col_idx + nnz);
    M.v.assign(A.values, A.values + nnz);
    validate_csr(M);
    M.sync_rp32();
    return M;
}

// inc/csr.hpp:135-162 — same checks, same messages.
void validate_csr(const HostCsr &A) {
    if (static_cast<int64_t>(A.rp.size()) != A.n + 1)
        throw invalid_argument("CsrMatrix: row_ptr length mismatch");
    if (A.rp.front() != 0) throw invalid_argument("CsrMatrix: row_ptr[0] != 0");
    if (A.rp.back() != A.nnz()) throw invalid_argument("CsrMatrix: row_ptr[nrows] != nnz");
    if (A.ci.size() != A.v.size()) throw invalid_argument("CsrMatrix: col/value length mismatch");
    for (int64_t i = 0; i < A.n; ++i) {
        if (A.rp[i + 1] < A.rp[i]) throw invalid_argument("CsrMatrix: row_ptr not monotone");
        for (int64_t k = A.rp[i]; k < A.rp[i + 1]; ++k) {
            if (A.ci[k] < 0 || A.ci[k] >= A.ncols)
                throw invalid_argument("CsrMatrix: column index out of range in row " +
                                       std::to_string(i));
            if (k > A.rp[i] && A.ci[k] <= A.ci[k - 1])
                throw invalid_argument("CsrMatrix: columns not strictly increasing in row " +
                                       std::to_string(i));
        }
    }
}

// Node-based heavy-edge matching, ascending visit (inc/coarsen.hpp:31-73):
// a node pairs with its unassigned neighbour of largest |a_ij| (stored zeros
// never match, ties keep the lowest column because the scan is ascending and
// the test is strict), coarse ids in discovery order.
std::vector<int32_t> node_hem(const HostCsr &A, int64_t *n_coarse) {
    if (A.n != A.ncols) throw invalid_argument("coarsen_node_hem: matrix must be square");
    std::vector<int32_t> f2c(static_cast<size_t>(A.n), -1);
    int32_t next = 0;
    for (int64_t i = 0; i < A.n; ++i) {
        if (f2c[i] >= 0) continue;
        int64_t best = -1;
        double best_w = 0.0;
        for (int64_t k = A.rp[i]; k < A.rp[i + 1]; ++k) {
            const int32_t j = A.ci[k];
            if (j == i || f2c[j] >= 0) continue;
            const double w = std::fabs(A.v[k]);
            if (w != 0.0 && (best < 0 || w > best_w)) {
                best = j;
                best_w = w;
            }
        }
        f2c[i] = next;
        if (best >= 0) f2c[best] = next;
        ++next;
    }
    *n_coarse = next;
    return f2c;
}

// Galerkin product for the unit piecewise-constant P (inc/aggregation.hpp:92-152).
// Coarse row k accumulates, member by member in ascending fine order and entry
// by entry in CSR order, into one running sum per coarse column; touched
// columns come out sorted and every touched column is stored (even a 0.0 sum).
// Coarse rows are independent, so chunks of them run on separate threads with
// identical per-row arithmetic.
HostCsr galerkin(const HostCsr &A, const std::vector<int32_t> &agg, int64_t nc, int threads) {
    const int64_t n = A.n;
    std::vector<int64_t> mptr(static_cast<size_t>(nc) + 1, 0);
    for (int32_t c : agg) {
        if (c < 0 || c >= nc)
            throw invalid_argument("Aggregation: coarse index " + std::to_string(c) +
                                   " outside [0, " + std::to_string(nc) + ")");
        ++mptr[static_cast<size_t>(c) + 1];
    }
    for (int64_t c = 0; c < nc; ++c) {
        const int64_t sz = mptr[c + 1];
        if (sz < 1 || sz > 2)
            throw invalid_argument("Aggregation: coarse node " + std::to_string(c) + " has " +
                                   std::to_string(sz) + " fine nodes");
    }
    for (int64_t c = 0; c < nc; ++c) mptr[c + 1] += mptr[c];
    std::vector<int32_t> mem(static_cast<size_t>(n));
    {
        std::vector<int64_t> next(mptr.begin(), mptr.end() - 1);
        for (int64_t i = 0; i < n; ++i) mem[next[agg[i]]++] = static_cast<int32_t>(i);
    }

    if (threads <= 0) threads = static_cast<int>(std::max(1u, std::thread::hardware_concurrency()));
    if (nc < 65536) threads = 1;
    struct Chunk {
        int64_t k0, k1;
        std::vector<int64_t> rowlen;
        std::vector<int32_t> ci;
        std::vector<double> v;
    };
    std::vector<Chunk> chunks(static_cast<size_t>(threads));
    auto work = [&](Chunk &ch) {
        std::vector<int32_t> cols;
        std::vector<double> acc;
        std::vector<int32_t> order;
        ch.rowlen.reserve(static_cast<size_t>(ch.k1 - ch.k0));
        for (int64_t k = ch.k0; k < ch.k1; ++k) {
            cols.clear();
            acc.clear();
            for (int64_t m = mptr[k]; m < mptr[k + 1]; ++m) {
                const int32_t i = mem[m];
                for (int64_t e = A.rp[i]; e < A.rp[i + 1]; ++e) {
                    const int32_t l = agg[A.ci[e]];
                    size_t t = 0;
                    while (t < cols.size() && cols[t] != l) ++t;
                    if (t == cols.size()) {
                        cols.push_back(l);
                        acc.push_back(0.0); // the reference's SPA slot starts at 0.0
                    }
                    acc[t] += A.v[e];
                }
            }
            order.resize(cols.size());
            std::iota(order.begin(), order.end(), 0);
            std::sort(order.begin(), order.end(),
                      [&](int32_t a, int32_t b) { return cols[a] < cols[b]; });
            for (int32_t t : order) {
                ch.ci.push_back(cols[t]);
                ch.v.push_back(acc[t]);
            }
            ch.rowlen.push_back(static_cast<int64_t>(cols.size()));
        }
    };
    const int64_t per = (nc + threads - 1) / threads;
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t) {
        chunks[t].k0 = std::min<int64_t>(nc, t * per);
        chunks[t].k1 = std::min<int64_t>(nc, (t + 1) * per);
        if (threads == 1) work(chunks[t]);
        else pool.emplace_back(work, std::ref(chunks[t]));
    }
    for (auto &th : pool) th.join();

    HostCsr C;
    C.n = C.ncols = nc;
    C.rp.assign(static_cast<size_t>(nc) + 1, 0);
    int64_t total = 0;
    for (auto &ch : chunks) total += static_cast<int64_t>(ch.ci.size());
    C.ci.reserve(static_cast<size_t>(total));
    C.v.reserve(static_cast<size_t>(total));
    int64_t row = 0;
    for (auto &ch : chunks) {
        for (int64_t len : ch.rowlen) {
            C.rp[row + 1] = C.rp[row] + len;
            ++row;
        }
        C.ci.insert(C.ci.end(), ch.ci.begin(), ch.ci.end());
        C.v.insert(C.v.end(), ch.v.begin(), ch.v.end());
        std::vector<int32_t>().swap(ch.ci);
        std::vector<double>().swap(ch.v);
    }
    C.sync_rp32();
    return C;
}

// Dense LU with partial pivoting of the coarsest matrix, exactly the reference's
// loop order (inc/coarse_solver.hpp:129-166), then the explicit inverse: column
// j is the reference's permuted forward/backward substitution of e_j
// (inc/coarse_solver.hpp:168-182). The device applies the inverse as a GEMV.
void factor_coarse(Hier &h) {
    const HostCsr &A = h.levels.back().A;
    if (A.n > 2000)
        throw invalid_argument("CoarseFactorization: coarsest level has " + std::to_string(A.n) +
                               " rows; the device path supports the dense LU (<= 2000) only");
    const size_t n = static_cast<size_t>(A.n);
    h.nc = A.n;
    h.lu.assign(n * n, 0.0);
    h.perm.resize(n);
    double max_abs = 0.0;
    for (size_t i = 0; i < n; ++i)
        for (int64_t k = A.rp[i]; k < A.rp[i + 1]; ++k) {
            h.lu[i * n + static_cast<size_t>(A.ci[k])] = A.v[k];
            max_abs = std::max(max_abs, std::fabs(A.v[k]));
        }
    std::iota(h.perm.begin(), h.perm.end(), 0);
    const double tol = 1e-14 * max_abs;
    for (size_t k = 0; k < n; ++k) {
        size_t p = k;
        for (size_t i = k + 1; i < n; ++i)
            if (std::fabs(h.lu[i * n + k]) > std::fabs(h.lu[p * n + k])) p = i;
        const double pivot = h.lu[p * n + k];
        if (pivot == 0.0 || std::fabs(pivot) < tol)
            throw runtime_error("CoarseFactorization: singular pivot in row " + std::to_string(k));
        if (p != k) {
            for (size_t j = 0; j < n; ++j) std::swap(h.lu[p * n + j], h.lu[k * n + j]);
            std::swap(h.perm[p], h.perm[k]);
        }
        for (size_t i = k + 1; i < n; ++i) {
            const double m = h.lu[i * n + k] / pivot;
            h.lu[i * n + k] = m;
            for (size_t j = k + 1; j < n; ++j) h.lu[i * n + j] -= m * h.lu[k * n + j];
        }
    }
    h.inv.assign(n * n, 0.0);
    std::vector<double> b(n), y(n);
    for (size_t col = 0; col < n; ++col) {
        std::fill(b.begin(), b.end(), 0.0);
        b[col] = 1.0;
        for (size_t i = 0; i < n; ++i) {
            double s = b[static_cast<size_t>(h.perm[i])];
            for (size_t j = 0; j < i; ++j) s -= h.lu[i * n + j] * y[j];
            y[i] = s;
        }
        for (size_t i = n; i-- > 0;) {
            double s = y[i];
            for (size_t j = i + 1; j < n; ++j) s -= h.lu[i * n + j] * y[j];
            y[i] = s / h.lu[i * n + i];
        }
        for (size_t i = 0; i < n; ++i) h.inv[i * n + col] = y[i];
    }
    h.symbolic += 1;
    h.numeric += 1;
}

// inc/hierarchy.hpp:51-76
Hier *build_hierarchy(HostCsr A0, const sb_setup_opts &o) {
    if (A0.n != A0.ncols) throw invalid_argument("Hierarchy: matrix must be square");
    if (o.coarse_target < 1) throw invalid_argument("SolverConfig: coarse_target must be >= 1");
    if (o.max_levels < 1) throw invalid_argument("SolverConfig: max_levels must be >= 1");
    if (o.coarsening != 0)
        throw invalid_argument("sb_setup: only node_hem coarsening is provided (edge_hem is not on the device path)");
    if (o.coarse_solver != 0 && o.coarse_solver != -1)
        throw invalid_argument("sb_setup: coarse_solver=cg is not supported on the device path; use direct");
    auto h = std::make_unique<Hier>();
    h->levels.push_back(HostLevel{std::move(A0), {}, -1});
    while (h->levels.back().A.n > o.coarse_target &&
           static_cast<int>(h->levels.size()) < o.max_levels) {
        const HostCsr &Af = h->levels.back().A;
        int64_t nc = 0;
        std::vector<int32_t> agg = node_hem(Af, &nc);
        if (nc == Af.n) {
            h->stalled = true;
            break;
        }
        HostCsr Ac = o.galerkin_gpu ? galerkin_gpu(Af, agg, nc, o.gpu_device) : galerkin(Af, agg, nc, o.threads);
        h->levels.back().agg = std::move(agg);
        h->levels.back().n_coarse = nc;
        h->levels.push_back(HostLevel{std::move(Ac), {}, -1});
    }
    if (o.coarse_solver == 0) factor_coarse(*h);
    return h.release();
}

} // namespace sb

// ---------------------------------------------------------------------------
// C ABI: host setup + generators
// ---------------------------------------------------------------------------
using namespace sb;


struct sb_hier_s {
    sb::Hier *h;
};

namespace sb {
Hier *hier_of(sb_hier h) { return h ? h->h : nullptr; }
} // namespace sb

extern "C" {

int sb_setup(const sb_csr *A, const sb_setup_opts *opts, sb_hier *out) {
    return guard([&] {
        if (!A || !out) throw invalid_argument("sb_setup: null argument");
        sb_setup_opts o{0, 500, 10, 0, 0, 0, 0};
        if (opts) o = *opts;
        HostCsr M = csr_from_abi(*A);
        *out = new sb_hier_s{build_hierarchy(std::move(M), o)};
    });
}

int sb_hier_from_levels(int nlevels, const sb_csr *levels, const int32_t *const *f2c, sb_hier *out) {
    return guard([&] {
        if (nlevels < 1 || !levels || !out) throw invalid_argument("sb_hier_from_levels: bad arguments");
        auto h = std::make_unique<Hier>();
        for (int k = 0; k < nlevels; ++k) {
            HostLevel L;
            L.A = csr_from_abi(levels[k]);
            if (L.A.n != L.A.ncols) throw invalid_argument("Hierarchy: matrix must be square");
            if (k + 1 < nlevels) {
                if (!f2c || !f2c[k]) throw invalid_argument("sb_hier_from_levels: missing aggregation");
                L.agg.assign(f2c[k], f2c[k] + L.A.n);
                L.n_coarse = levels[k + 1].nrows;
                // Aggregation::validate (inc/aggregation.hpp:42-58): a surjection
                // with 1 or 2 fine nodes per coarse node (the device restriction
                // stores at most two members per aggregate)
                std::vector<int32_t> count(static_cast<size_t>(L.n_coarse), 0);
                for (int32_t c : L.agg) {
                    if (c < 0 || c >= L.n_coarse)
                        throw invalid_argument("Aggregation: coarse index " + std::to_string(c) +
                                               " outside [0, " + std::to_string(L.n_coarse) + ")");
                    ++count[static_cast<size_t>(c)];
                }
                for (int64_t c = 0; c < L.n_coarse; ++c)
                    if (count[c] < 1 || count[c] > 2)
                        throw invalid_argument("Aggregation: coarse node " + std::to_string(c) + " has " +
                                               std::to_string(count[c]) + " fine nodes");
            }
            h->levels.push_back(std::move(L));
        }
        factor_coarse(*h);
        *out = new sb_hier_s{h.release()};
    });
}

void sb_hier_free(sb_hier h) {
    if (!h) return;
    delete h->h;
    delete h;
}
int sb_hier_nlevels(sb_hier h) { return h ? static_cast<int>(h->h->levels.size()) : 0; }
int sb_hier_stalled(sb_hier h) { return h && h->h->stalled ? 1 : 0; }

int sb_hier_level(sb_hier h, int k, sb_csr *A, const int32_t **f2c, int64_t *n_coarse) {
    return guard([&] {
        if (!h || k < 0 || k >= static_cast<int>(h->h->levels.size()))
            throw invalid_argument("sb_hier_level: level out of range");
        const HostLevel &L = h->h->levels[static_cast<size_t>(k)];
        if (A) {
            A->nrows = L.A.n;
            A->ncols = L.A.ncols;
            A->row_ptr32 = L.A.rp32.empty() ? nullptr : L.A.rp32.data();
            A->row_ptr64 = L.A.rp32.empty() ? L.A.rp.data() : nullptr;
            A->col_idx = L.A.ci.data();
            A->values = L.A.v.data();
        }
        if (f2c) *f2c = L.agg.empty() ? nullptr : L.agg.data();
        if (n_coarse) *n_coarse = L.n_coarse;
    });
}

int sb_hier_coarse_counts(sb_hier h, long *symbolic, long *numeric, long *solves) {
    return guard([&] {
        if (!h) throw invalid_argument("sb_hier_coarse_counts: null hierarchy");
        if (symbolic) *symbolic = h->h->symbolic;
        if (numeric) *numeric = h->h->numeric;
        if (solves) *solves = h->h->solves;
    });
}

// ---- generators -------------------------------------------------------------

static void emit(HostCsr &M, sb_csr *out) {
    M.sync_rp32();
    const size_t n1 = M.rp.size();
    out->nrows = M.n;
    out->ncols = M.ncols;
    if (!M.rp32.empty()) {
        auto *rp = static_cast<int32_t *>(std::malloc(sizeof(int32_t) * n1));
        std::memcpy(rp, M.rp32.data(), sizeof(int32_t) * n1);
        out->row_ptr32 = rp;
        out->row_ptr64 = nullptr;
    } else {
        auto *rp = static_cast<int64_t *>(std::malloc(sizeof(int64_t) * n1));
        std::memcpy(rp, M.rp.data(), sizeof(int64_t) * n1);
        out->row_ptr64 = rp;
        out->row_ptr32 = nullptr;
    }
    auto *ci = static_cast<int32_t *>(std::malloc(sizeof(int32_t) * (M.ci.size() + 1)));
    auto *v = static_cast<double *>(std::malloc(sizeof(double) * (M.v.size() + 1)));
    std::memcpy(ci, M.ci.data(), sizeof(int32_t) * M.ci.size());
    std::memcpy(v, M.v.data(), sizeof(double) * M.v.size());
    out->col_idx = ci;
    out->values = v;
}

// read_matrix_market / write_matrix_market — inc/mm_io.hpp:35-135 restated:
// coordinate real general|symmetric, 1-based indices, symmetric entries
// mirrored, then the reference's from_triplets (inc/csr.hpp:57-95: std::sort
// by (row, col), duplicates summed from 0.0 in the sorted order).
int sb_read_matrix_market(const char *path, sb_csr *out) {
    return guard([&] {
        if (!path || !out) throw invalid_argument("sb_read_matrix_market: null argument");
        const std::string p(path);
        std::ifstream in(p);
        if (!in) throw runtime_error("read_matrix_market: cannot open '" + p + "'");
        auto lower = [](std::string s) {
            for (char &ch : s) ch = static_cast<char>(std::tolower(static_cast<unsigned char>(ch)));
            return s;
        };
        std::string banner;
        if (!std::getline(in, banner)) throw runtime_error("read_matrix_market: '" + p + "' is empty");
        std::istringstream hdr(banner);
        std::string tag, object, format, field, symmetry;
        hdr >> tag >> object >> format >> field >> symmetry;
        if (lower(tag) != "%%matrixmarket" || lower(object) != "matrix")
            throw runtime_error("read_matrix_market: '" + p + "': malformed header '" + banner + "'");
        if (lower(format) != "coordinate")
            throw runtime_error("read_matrix_market: '" + p + "': only coordinate format is supported");
        if (lower(field) != "real")
            throw runtime_error("read_matrix_market: '" + p + "': field '" + field + "' is not real");
        const std::string sym = lower(symmetry);
        if (sym != "general" && sym != "symmetric")
            throw runtime_error("read_matrix_market: '" + p + "': symmetry '" + symmetry +
                                "' is not general or symmetric");
        std::string line;
        auto next_data_line = [&](std::string &o) {
            while (std::getline(in, o)) {
                const auto pos = o.find_first_not_of(" \t\r\n");
                if (pos == std::string::npos || o[pos] == '%') continue;
                return true;
            }
            return false;
        };
        if (!next_data_line(line)) throw runtime_error("read_matrix_market: '" + p + "': missing size line");
        long long nrows = 0, ncols = 0, nnz = 0;
        {
            std::istringstream sz(line);
            if (!(sz >> nrows >> ncols >> nnz) || nrows < 0 || ncols < 0 || nnz < 0)
                throw runtime_error("read_matrix_market: '" + p + "': malformed size line '" + line + "'");
        }
        struct Trip {
            int32_t row, col;
            double value;
        };
        std::vector<Trip> ent;
        ent.reserve(static_cast<size_t>(sym == "symmetric" ? 2 * nnz : nnz));
        for (long long e = 0; e < nnz; ++e) {
            if (!next_data_line(line))
                throw runtime_error("read_matrix_market: '" + p + "': expected " + std::to_string(nnz) +
                                    " entries, found " + std::to_string(e));
            std::istringstream es(line);
            long long i = 0, j = 0;
            double v = 0.0;
            if (!(es >> i >> j >> v)) throw runtime_error("read_matrix_market: '" + p + "': malformed entry '" + line + "'");
            if (i < 1 || i > nrows || j < 1 || j > ncols)
                throw runtime_error("read_matrix_market: '" + p + "': index (" + std::to_string(i) + ", " +
                                    std::to_string(j) + ") out of bounds for " + std::to_string(nrows) + "x" +
                                    std::to_string(ncols));
            ent.push_back({static_cast<int32_t>(i - 1), static_cast<int32_t>(j - 1), v});
            if (sym == "symmetric" && i != j) ent.push_back({static_cast<int32_t>(j - 1), static_cast<int32_t>(i - 1), v});
        }
        std::sort(ent.begin(), ent.end(),
                  [](const Trip &a, const Trip &b) { return a.row != b.row ? a.row < b.row : a.col < b.col; });
        HostCsr M;
        M.n = nrows;
        M.ncols = ncols;
        M.rp.assign(static_cast<size_t>(nrows) + 1, 0);
        size_t k = 0;
        while (k < ent.size()) {
            const int32_t r = ent[k].row, cc = ent[k].col;
            double sum = 0.0;
            while (k < ent.size() && ent[k].row == r && ent[k].col == cc) sum += ent[k++].value;
            M.ci.push_back(cc);
            M.v.push_back(sum);
            M.rp[static_cast<size_t>(r) + 1] = static_cast<int64_t>(M.ci.size());
        }
        for (long long r = 0; r < nrows; ++r)
            M.rp[static_cast<size_t>(r) + 1] = std::max(M.rp[static_cast<size_t>(r) + 1], M.rp[static_cast<size_t>(r)]);
        emit(M, out);
    });
}

int sb_write_matrix_market(const char *path, const sb_csr *A) {
    return guard([&] {
        if (!path || !A) throw invalid_argument("sb_write_matrix_market: null argument");
        const HostCsr M = csr_from_abi(*A);
        std::ofstream out(path);
        if (!out) throw runtime_error(std::string("write_matrix_market: cannot open '") + path + "'");
        out << "%%MatrixMarket matrix coordinate real general\n";
        out << M.n << " " << M.ncols << " " << M.nnz() << "\n";
        out.precision(17);
        for (int64_t i = 0; i < M.n; ++i)
            for (int64_t e = M.rp[static_cast<size_t>(i)]; e < M.rp[static_cast<size_t>(i) + 1]; ++e)
                out << (i + 1) << " " << (M.ci[static_cast<size_t>(e)] + 1) << " " << M.v[static_cast<size_t>(e)] << "\n";
        if (!out) throw runtime_error(std::string("write_matrix_market: write to '") + path + "' failed");
    });
}

int sb_galerkin_gpu(const sb_csr *A, const int32_t *f2c, int64_t n_coarse, int device, sb_csr *out) {
    return guard([&] {
        if (!A || !f2c || !out) throw invalid_argument("sb_galerkin_gpu: null argument");
        HostCsr M = csr_from_abi(*A);
        if (M.n != M.ncols) throw invalid_argument("galerkin_product: matrix must be square");
        if (n_coarse < 1 || n_coarse > M.n) throw invalid_argument("sb_galerkin_gpu: bad n_coarse");
        std::vector<int32_t> agg(f2c, f2c + M.n);
        HostCsr C = galerkin_gpu(M, agg, n_coarse, device);
        emit(C, out);
    });
}

void sb_free_csr(sb_csr *m) {
    if (!m) return;
    std::free(const_cast<int32_t *>(m->row_ptr32));
    std::free(const_cast<int64_t *>(m->row_ptr64));
    std::free(const_cast<int32_t *>(m->col_idx));
    std::free(const_cast<double *>(m->values));
    m->row_ptr32 = nullptr;
    m->row_ptr64 = nullptr;
    m->col_idx = nullptr;
    m->values = nullptr;
}

// A value stored through the reference's from_triplets is `0.0 + v`
// (inc/csr.hpp:79-83); keep that (it maps -0.0 to +0.0).
static inline double stored(double v) {
    double s = 0.0;
    s += v;
    return s;
}

} // extern "C"
namespace sb {
// 3D 27-point operator (diag, `off` to every neighbour), Dirichlet, rows in
// (iz*ny + iy)*nx + ix order, columns ascending: built straight into the
// host CSR (int64 offsets; nnz may exceed int32: C5 512^3 has 3.6e9).
HostCsr stencil27(int64_t nx, int64_t ny, int64_t nz, double diag, double off) {
    if (nx < 1 || ny < 1 || nz < 1) throw invalid_argument("stencil27: grid dims must be >= 1");
    if (nx * ny * nz > INT32_MAX) throw invalid_argument("stencil27: grid too large for int32 columns");
    HostCsr M;
    M.n = M.ncols = nx * ny * nz;
    M.rp.assign(static_cast<size_t>(M.n) + 1, 0);
    const int64_t nnz = (3 * nx - 2) * (3 * ny - 2) * (3 * nz - 2);
    M.ci.reserve(static_cast<size_t>(nnz));
    M.v.reserve(static_cast<size_t>(nnz));
    const double sd = stored(diag), so = stored(off);
    for (int64_t iz = 0; iz < nz; ++iz)
        for (int64_t iy = 0; iy < ny; ++iy)
            for (int64_t ix = 0; ix < nx; ++ix) {
                const int64_t m = (iz * ny + iy) * nx + ix;
                for (int dz = -1; dz <= 1; ++dz)
                    for (int dy = -1; dy <= 1; ++dy)
                        for (int dx = -1; dx <= 1; ++dx) {
                            const int64_t jx = ix + dx, jy = iy + dy, jz = iz + dz;
                            if (jx < 0 || jy < 0 || jz < 0 || jx >= nx || jy >= ny || jz >= nz) continue;
                            const int64_t col = (jz * ny + jy) * nx + jx;
                            M.ci.push_back(static_cast<int32_t>(col));
                            M.v.push_back(col == m ? sd : so);
                        }
                M.rp[static_cast<size_t>(m) + 1] = static_cast<int64_t>(M.ci.size());
            }
    M.sync_rp32();
    return M;
}
} // namespace sb
extern "C" {

// inc/problems.hpp:28-57, same expressions in the same order; rows come out
// sorted (south, west, diag, east, north) as from_triplets would sort them.
int sb_gen_convdiff2d(int64_t nx, int64_t ny, double bx, double by, double c, sb_csr *out) {
    return guard([&] {
        if (nx < 2 || ny < 2)
            throw invalid_argument("convdiff2d: grid dims must be >= 2, got " + std::to_string(nx) +
                                   "x" + std::to_string(ny));
        if (nx * ny > INT32_MAX) throw invalid_argument("convdiff2d: grid too large");
        const double hx = 1.0 / (static_cast<double>(nx) + 1.0);
        const double hy = 1.0 / (static_cast<double>(ny) + 1.0);
        const double diag = 2.0 * hy / hx + 2.0 * hx / hy + std::abs(bx) * hy +
                            std::abs(by) * hx + c * hx * hy;
        const double west = -hy / hx - std::max(bx, 0.0) * hy;
        const double east = -hy / hx + std::min(bx, 0.0) * hy;
        const double south = -hx / hy - std::max(by, 0.0) * hx;
        const double north = -hx / hy + std::min(by, 0.0) * hx;
        HostCsr M;
        M.n = M.ncols = nx * ny;
        M.rp.assign(static_cast<size_t>(M.n) + 1, 0);
        M.ci.reserve(static_cast<size_t>(5 * M.n));
        M.v.reserve(static_cast<size_t>(5 * M.n));
        for (int64_t iy = 0; iy < ny; ++iy)
            for (int64_t ix = 0; ix < nx; ++ix) {
                const int64_t m = iy * nx + ix;
                auto put = [&](int64_t col, double val) {
                    M.ci.push_back(static_cast<int32_t>(col));
                    M.v.push_back(stored(val));
                };
                if (iy > 0) put(m - nx, south);
                if (ix > 0) put(m - 1, west);
                put(m, diag);
                if (ix < nx - 1) put(m + 1, east);
                if (iy < ny - 1) put(m + nx, north);
                M.rp[m + 1] = static_cast<int64_t>(M.ci.size());
            }
        emit(M, out);
    });
}

// 3D 7-point stencil on an nx*ny*nz grid, node m = (iz*ny + iy)*nx + ix,
// Dirichlet boundaries (out-of-grid neighbours dropped). off = {x-, x+, y-, y+, z-, z+}.
int sb_gen_stencil7(int64_t nx, int64_t ny, int64_t nz, double diag, const double off[6],
                    sb_csr *out) {
    return guard([&] {
        if (nx < 1 || ny < 1 || nz < 1) throw invalid_argument("stencil7: grid dims must be >= 1");
        if (nx * ny * nz > INT32_MAX) throw invalid_argument("stencil7: grid too large for int32 columns");
        HostCsr M;
        M.n = M.ncols = nx * ny * nz;
        M.rp.assign(static_cast<size_t>(M.n) + 1, 0);
        M.ci.reserve(static_cast<size_t>(7 * M.n));
        M.v.reserve(static_cast<size_t>(7 * M.n));
        const int64_t sxy = nx * ny;
        for (int64_t iz = 0; iz < nz; ++iz)
            for (int64_t iy = 0; iy < ny; ++iy)
                for (int64_t ix = 0; ix < nx; ++ix) {
                    const int64_t m = (iz * ny + iy) * nx + ix;
                    auto put = [&](int64_t col, double val) {
                        M.ci.push_back(static_cast<int32_t>(col));
                        M.v.push_back(stored(val));
                    };
                    if (iz > 0) put(m - sxy, off[4]);
                    if (iy > 0) put(m - nx, off[2]);
                    if (ix > 0) put(m - 1, off[0]);
                    put(m, diag);
                    if (ix < nx - 1) put(m + 1, off[1]);
                    if (iy < ny - 1) put(m + nx, off[3]);
                    if (iz < nz - 1) put(m + sxy, off[5]);
                    M.rp[m + 1] = static_cast<int64_t>(M.ci.size());
                }
        emit(M, out);
    });
}

// -lap(u) + b.grad(u) + c u on (0,1)^3, first-order upwinding, every entry
// scaled by the cell volume hx*hy*hz — the 3D extension of convdiff2d
// (inc/problems.hpp:28-41) used for config C4.
int sb_gen_convdiff3d(int64_t nx, int64_t ny, int64_t nz, double bx, double by, double bz,
                      double c, sb_csr *out) {
    const double hx = 1.0 / (static_cast<double>(nx) + 1.0);
    const double hy = 1.0 / (static_cast<double>(ny) + 1.0);
    const double hz = 1.0 / (static_cast<double>(nz) + 1.0);
    const double ax = hy * hz / hx, ay = hx * hz / hy, az = hx * hy / hz;
    const double diag = 2.0 * (ax + ay + az) + std::abs(bx) * hy * hz + std::abs(by) * hx * hz +
                        std::abs(bz) * hx * hy + c * hx * hy * hz;
    const double off[6] = {-ax - std::max(bx, 0.0) * hy * hz, -ax + std::min(bx, 0.0) * hy * hz,
                           -ay - std::max(by, 0.0) * hx * hz, -ay + std::min(by, 0.0) * hx * hz,
                           -az - std::max(bz, 0.0) * hx * hy, -az + std::min(bz, 0.0) * hx * hy};
    return sb_gen_stencil7(nx, ny, nz, diag, off, out);
}

int sb_gen_stencil27(int64_t nx, int64_t ny, int64_t nz, double diag, double off, sb_csr *out) {
    return guard([&] {
        HostCsr M = sb::stencil27(nx, ny, nz, diag, off);
        emit(M, out);
    });
}

int sb_setup_stencil27(int64_t nx, int64_t ny, int64_t nz, double diag, double off, const sb_setup_opts *opts,
                       sb_hier *out) {
    return guard([&] {
        if (!out) throw invalid_argument("sb_setup_stencil27: null argument");
        sb_setup_opts o{0, 500, 10, 0, 0, 0, 0};
        if (opts) o = *opts;
        *out = new sb_hier_s{build_hierarchy(sb::stencil27(nx, ny, nz, diag, off), o)};
    });
}

int sb_gen_rhs_random(int64_t n, unsigned seed, double *out) {
    return guard([&] {
        if (n < 0 || (n > 0 && !out)) throw invalid_argument("rhs_random: bad arguments");
        std::mt19937 gen(seed);
        std::uniform_real_distribution<double> dist(0.0, 1.0);
        for (int64_t i = 0; i < n; ++i) out[i] = dist(gen);
    });
}

} // extern "C"
