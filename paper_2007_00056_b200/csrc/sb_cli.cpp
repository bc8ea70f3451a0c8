// sparsh_b200 — command-line front end over the C ABI, mirroring the
// reference's `sparsh run` / `gen` / `coarsen-info` (tools/sparsh.cpp:241-330):
// same flags, same report text, same convergence CSV
// ("iter,residual_l2,cumulative_seconds", tools/sparsh.cpp:135-149), same exit
// codes (0 converged / done, 1 not converged or numerical failure, 2 usage or
// I/O error). The solve runs on the GPU; deviations: the smoother defaults to
// weighted Jacobi and Gauss-Seidel is rejected (sequential), --threads is
// accepted and ignored, extra generated problems (3D) and device placement
// flags (--device, --host-levels-from, --galerkin-gpu) are available.
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iomanip>
#include <iostream>
#include <map>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "sparsh_b200.h"

namespace {

struct usage_error : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct numeric_error : std::runtime_error {
    using std::runtime_error::runtime_error;
};

void ck(int rc) {
    if (rc == SB_OK) return;
    const std::string msg = sb_last_error();
    if (rc == SB_EINVAL) throw usage_error(msg);
    if (rc == SB_ERUNTIME) throw numeric_error(msg);
    throw std::runtime_error(msg);
}

std::vector<std::string> split(const std::string &s, char sep) {
    std::vector<std::string> parts;
    std::string item;
    std::istringstream in(s);
    while (std::getline(in, item, sep)) parts.push_back(item);
    return parts;
}

long parse_long(const std::string &s, const std::string &what) {
    size_t pos = 0;
    long v = 0;
    try {
        v = std::stol(s, &pos);
    } catch (const std::exception &) {
        pos = std::string::npos;
    }
    if (pos != s.size() || s.empty()) throw usage_error("bad " + what + " '" + s + "'");
    return v;
}

double parse_double(const std::string &s, const std::string &what) {
    size_t pos = 0;
    double v = 0.0;
    try {
        v = std::stod(s, &pos);
    } catch (const std::exception &) {
        pos = std::string::npos;
    }
    if (pos != s.size() || s.empty()) throw usage_error("bad " + what + " '" + s + "'");
    return v;
}

// poisson2d:NXxNY | convdiff2d:NXxNY:BX,BY,C (the reference's) and
// poisson3d:NXxNYxNZ | aniso3d:NXxNYxNZ:EPS | convdiff3d:NXxNYxNZ:BX,BY,BZ,C | stencil27:NXxNYxNZ
sb_csr build_problem(const std::string &text) {
    const std::string usage =
        " (expected poisson2d:NXxNY, convdiff2d:NXxNY:BX,BY,C, poisson3d:NXxNYxNZ, aniso3d:NXxNYxNZ:EPS, "
        "convdiff3d:NXxNYxNZ:BX,BY,BZ,C or stencil27:NXxNYxNZ)";
    const auto parts = split(text, ':');
    if (parts.size() < 2) throw usage_error("bad --problem '" + text + "'" + usage);
    const auto dims = split(parts[1], 'x');
    std::vector<long> d;
    for (const auto &s : dims) d.push_back(parse_long(s, "grid dimension"));
    sb_csr A{};
    const std::string &k = parts[0];
    auto coeffs = [&](size_t want) {
        if (parts.size() != 3) throw usage_error("bad --problem '" + text + "'" + usage);
        const auto c = split(parts[2], ',');
        if (c.size() != want) throw usage_error("bad --problem '" + text + "'" + usage);
        std::vector<double> v;
        for (const auto &s : c) v.push_back(parse_double(s, "coefficient"));
        return v;
    };
    if (k == "poisson2d" && d.size() == 2 && parts.size() == 2) {
        ck(sb_gen_convdiff2d(d[0], d[1], 0.0, 0.0, 0.0, &A));
    } else if (k == "convdiff2d" && d.size() == 2) {
        const auto c = coeffs(3);
        ck(sb_gen_convdiff2d(d[0], d[1], c[0], c[1], c[2], &A));
    } else if (k == "poisson3d" && d.size() == 3 && parts.size() == 2) {
        const double off[6] = {-1, -1, -1, -1, -1, -1};
        ck(sb_gen_stencil7(d[0], d[1], d[2], 6.0, off, &A));
    } else if (k == "aniso3d" && d.size() == 3) {
        const auto c = coeffs(1);
        const double off[6] = {-1, -1, -1, -1, -c[0], -c[0]};
        ck(sb_gen_stencil7(d[0], d[1], d[2], 4.0 + 2.0 * c[0], off, &A));
    } else if (k == "convdiff3d" && d.size() == 3) {
        const auto c = coeffs(4);
        ck(sb_gen_convdiff3d(d[0], d[1], d[2], c[0], c[1], c[2], c[3], &A));
    } else if (k == "stencil27" && d.size() == 3 && parts.size() == 2) {
        ck(sb_gen_stencil27(d[0], d[1], d[2], 26.0, -1.0, &A));
    } else {
        throw usage_error("bad --problem '" + text + "'" + usage);
    }
    return A;
}

std::vector<double> build_rhs(const std::string &mode, int64_t n, unsigned seed) {
    if (mode == "ones") return std::vector<double>(static_cast<size_t>(n), 1.0);
    if (mode == "random") {
        std::vector<double> v(static_cast<size_t>(n));
        ck(sb_gen_rhs_random(n, seed, v.data()));
        return v;
    }
    if (mode.rfind("file:", 0) == 0) {  // read_vector (problems.hpp:78-89)
        const std::string path = mode.substr(5);
        std::ifstream in(path);
        if (!in) throw std::runtime_error("read_vector: cannot open '" + path + "'");
        std::vector<double> v;
        double x = 0.0;
        while (in >> x) v.push_back(x);
        if (!in.eof())
            throw std::runtime_error("read_vector: malformed value in '" + path + "' near entry " +
                                     std::to_string(v.size()));
        if (static_cast<int64_t>(v.size()) != n)
            throw usage_error("rhs file has " + std::to_string(v.size()) + " entries but the system has " +
                              std::to_string(n));
        return v;
    }
    throw usage_error("bad --rhs '" + mode + "' (expected ones, random or file:PATH)");
}

struct Opts {
    std::string problem, matrix, solver = "amg", coarsening = "node_hem", smoother = "jacobi",
                         coarse_solver = "direct", rhs = "ones", out, config;
    double omega = 2.0 / 3.0, tol = 1e-8;
    int pre = 6, post = 6, max_levels = 10, max_iters = 1000, threads = 1, device = 0, galerkin_gpu = 0;
    long coarse_target = 500, host_levels_from = -1;
    unsigned seed = 42;
};

void set_opt(Opts &o, const std::string &key, const std::string &v) {
    if (key == "problem") o.problem = v;
    else if (key == "matrix") o.matrix = v;
    else if (key == "solver") o.solver = v;
    else if (key == "coarsening") o.coarsening = v;
    else if (key == "smoother") o.smoother = v;
    else if (key == "coarse-solver") o.coarse_solver = v;
    else if (key == "omega") o.omega = parse_double(v, "omega");
    else if (key == "pre") o.pre = static_cast<int>(parse_long(v, "pre"));
    else if (key == "post") o.post = static_cast<int>(parse_long(v, "post"));
    else if (key == "coarse-target") o.coarse_target = parse_long(v, "coarse-target");
    else if (key == "max-levels") o.max_levels = static_cast<int>(parse_long(v, "max-levels"));
    else if (key == "tol") o.tol = parse_double(v, "tol");
    else if (key == "max-iters") o.max_iters = static_cast<int>(parse_long(v, "max-iters"));
    else if (key == "rhs") o.rhs = v;
    else if (key == "seed") o.seed = static_cast<unsigned>(parse_long(v, "seed"));
    else if (key == "out") o.out = v;
    else if (key == "threads") o.threads = static_cast<int>(parse_long(v, "threads"));
    else if (key == "config") o.config = v;
    else if (key == "device") o.device = static_cast<int>(parse_long(v, "device"));
    else if (key == "host-levels-from") o.host_levels_from = parse_long(v, "host-levels-from");
    else if (key == "galerkin-gpu") o.galerkin_gpu = static_cast<int>(parse_long(v, "galerkin-gpu"));
    else throw usage_error("unknown option --" + key);
}

// key=value file, command-line flags win (tools/sparsh.cpp:382-445)
void apply_config(Opts &o, const std::map<std::string, std::string> &given) {
    if (o.config.empty()) return;
    std::ifstream in(o.config);
    if (!in) throw std::runtime_error("cannot open config file '" + o.config + "'");
    std::string line;
    int lineno = 0;
    auto trim = [](const std::string &s) {
        const auto b = s.find_first_not_of(" \t\r\n");
        if (b == std::string::npos) return std::string();
        return s.substr(b, s.find_last_not_of(" \t\r\n") - b + 1);
    };
    while (std::getline(in, line)) {
        ++lineno;
        const auto hash = line.find('#');
        if (hash != std::string::npos) line.erase(hash);
        line = trim(line);
        if (line.empty()) continue;
        const auto eq = line.find('=');
        if (eq == std::string::npos)
            throw usage_error(o.config + ":" + std::to_string(lineno) + ": expected key=value, got '" + line + "'");
        const std::string key = trim(line.substr(0, eq)), value = trim(line.substr(eq + 1));
        if (key.empty()) throw usage_error(o.config + ":" + std::to_string(lineno) + ": empty key");
        if (key == "config") throw usage_error(o.config + ": config files cannot nest");
        if (given.count(key)) continue;
        set_opt(o, key, value);
    }
}

sb_csr load_system(const Opts &o) {
    if (o.problem.empty() == o.matrix.empty()) throw usage_error("exactly one of --problem and --matrix is required");
    sb_csr A{};
    if (o.matrix.empty()) return build_problem(o.problem);
    if (sb_read_matrix_market(o.matrix.c_str(), &A) != SB_OK)
        throw std::runtime_error(sb_last_error());  // an I/O error: exit 2
    return A;
}

int smoother_code(const std::string &s) {
    if (s == "jacobi" || s == "weighted_jacobi") return SB_SMOOTHER_JACOBI;
    if (s == "gs_forward" || s == "gs_backward" || s == "gs_symmetric")
        throw usage_error("smoother '" + s + "' is sequential Gauss-Seidel: not provided on the GPU (use jacobi)");
    throw usage_error("bad --smoother '" + s + "'");
}

struct LevelStat {
    int64_t size, nnz;
};

std::vector<LevelStat> level_stats(sb_hier h) {
    std::vector<LevelStat> s;
    for (int k = 0; k < sb_hier_nlevels(h); ++k) {
        sb_csr a{};
        const int32_t *agg = nullptr;
        int64_t nc = 0;
        ck(sb_hier_level(h, k, &a, &agg, &nc));
        s.push_back({a.nrows, a.row_ptr32 ? a.row_ptr32[a.nrows] : a.row_ptr64[a.nrows]});
    }
    return s;
}

// print_levels (tools/sparsh.cpp:151-176)
void print_levels(std::ostream &out, const std::vector<LevelStat> &s, bool stalled) {
    out << std::setw(6) << "level" << std::setw(12) << "size" << std::setw(14) << "nnz" << std::setw(9) << "ratio"
        << '\n';
    double nnz = 0, rows = 0;
    for (size_t i = 0; i < s.size(); ++i) {
        out << std::setw(6) << i << std::setw(12) << s[i].size << std::setw(14) << s[i].nnz;
        if (i == 0) out << std::setw(9) << "-";
        else
            out << std::setw(9) << std::fixed << std::setprecision(2)
                << static_cast<double>(s[i - 1].size) / static_cast<double>(s[i].size) << std::defaultfloat;
        out << '\n';
        nnz += static_cast<double>(s[i].nnz);
        rows += static_cast<double>(s[i].size);
    }
    out << "operator complexity: " << std::setprecision(4) << nnz / static_cast<double>(s[0].nnz) << '\n';
    out << "grid complexity:     " << std::setprecision(4) << rows / static_cast<double>(s[0].size) << '\n';
    if (stalled) out << "warning: coarsening stalled above the coarse-size target\n";
}

const char *term_name(int t) {
    switch (t) {
    case SB_CONVERGED: return "converged";
    case SB_MAX_ITERS: return "max_iters";
    case SB_BREAKDOWN: return "breakdown";
    default: return "diverged";
    }
}

sb_setup_opts setup_opts(const Opts &o, bool hierarchy) {
    if (o.coarsening != "node_hem") {
        if (o.coarsening == "edge_hem") throw usage_error("coarsening 'edge_hem' is not provided on the device path");
        throw usage_error("bad --coarsening '" + o.coarsening + "'");
    }
    if (o.coarse_solver != "direct")
        throw usage_error("coarse solver '" + o.coarse_solver + "' is not provided on the device path (use direct)");
    sb_setup_opts so{0, o.coarse_target, o.max_levels, hierarchy ? 0 : -1, 0, o.galerkin_gpu, o.device};
    if (!hierarchy) {
        so.max_levels = 1;
        so.coarse_target = 1;
    }
    return so;
}

int cmd_run(const Opts &o) {
    const bool needs_h = o.solver == "amg" || o.solver == "pcg" || o.solver == "pbicgstab";
    if (!needs_h && o.solver != "cg" && o.solver != "bicgstab")
        throw usage_error("bad --solver '" + o.solver + "' (expected amg, cg, pcg, bicgstab or pbicgstab)");
    sb_cycle cp{o.pre, o.post, smoother_code(o.smoother), o.omega};
    sb_csr A = load_system(o);
    const std::vector<double> b = build_rhs(o.rhs, A.nrows, o.seed);
    const sb_setup_opts so = setup_opts(o, needs_h);
    sb_hier h = nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    const int rs = sb_setup(&A, &so, &h);
    sb_free_csr(&A);
    if (rs == SB_ERUNTIME) {
        std::cerr << "error: " << sb_last_error() << '\n';
        return 1;
    }
    ck(rs);
    sb_ctx ctx = nullptr;
    const sb_device_opts dopt{o.device, 1, o.host_levels_from, 0};
    ck(sb_create(h, &dopt, &ctx));
    const double setup_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    std::vector<double> x(b.size(), 0.0), hr(static_cast<size_t>(std::max(o.max_iters, 0)) + 2),
        ht(hr.size());
    sb_report rep{0, 0, 0, 0, 0, static_cast<int>(hr.size()), hr.data(), ht.data()};
    int rc = SB_OK;
    if (o.solver == "amg") rc = sb_amg_solve(ctx, &cp, b.data(), x.data(), o.tol, o.max_iters, &rep);
    else if (o.solver == "pcg") rc = sb_pcg(ctx, &cp, b.data(), x.data(), o.tol, o.max_iters, &rep);
    else if (o.solver == "cg") rc = sb_pcg(ctx, nullptr, b.data(), x.data(), o.tol, o.max_iters, &rep);
    else if (o.solver == "pbicgstab") rc = sb_pbicgstab(ctx, &cp, b.data(), x.data(), o.tol, o.max_iters, &rep);
    else rc = sb_pbicgstab(ctx, nullptr, b.data(), x.data(), o.tol, o.max_iters, &rep);
    if (rc == SB_ERUNTIME) {
        std::cerr << "error: " << sb_last_error() << '\n';
        sb_destroy(ctx);
        sb_hier_free(h);
        return 1;
    }
    ck(rc);
    const int hl = std::min(rep.hist_len, rep.hist_cap);
    if (!o.out.empty()) {  // write_report_csv (tools/sparsh.cpp:135-149)
        std::ofstream out(o.out);
        if (!out) throw std::runtime_error("cannot open '" + o.out + "' for writing");
        out << "iter,residual_l2,cumulative_seconds\n";
        char num[40];
        for (int k = 0; k < hl; ++k) {
            std::snprintf(num, sizeof num, "%.17g", hr[static_cast<size_t>(k)]);
            out << k << ',' << num << ',';
            std::snprintf(num, sizeof num, "%.9g", ht[static_cast<size_t>(k)]);
            out << num << '\n';
        }
        if (!out) throw std::runtime_error("write to '" + o.out + "' failed");
    }
    std::cout << "solver: " << o.solver << '\n';
    if (needs_h) print_levels(std::cout, level_stats(h), sb_hier_stalled(h) != 0);
    std::cout << std::setprecision(6) << std::fixed << "setup seconds: " << setup_s << '\n'
              << "solve seconds: " << rep.wall_time << '\n'
              << std::defaultfloat << "iterations: " << rep.iterations << '\n'
              << "termination: " << term_name(rep.termination) << '\n'
              << "final residual: " << std::setprecision(6) << (hl > 0 ? hr[static_cast<size_t>(hl - 1)] : 0.0)
              << " (true " << rep.true_residual << ")\n";
    sb_destroy(ctx);
    sb_hier_free(h);
    if (rep.termination != SB_CONVERGED) {
        std::cerr << "solver did not converge: " << term_name(rep.termination) << '\n';
        return 1;
    }
    return 0;
}

int cmd_gen(const std::string &problem, const std::string &out) {
    sb_csr A = build_problem(problem);
    const std::string path = out.empty() ? "/dev/stdout" : out;
    ck(sb_write_matrix_market(path.c_str(), &A));
    if (!out.empty()) {
        const int64_t nnz = A.row_ptr32 ? A.row_ptr32[A.nrows] : A.row_ptr64[A.nrows];
        std::cerr << "wrote " << A.nrows << "x" << A.ncols << " matrix (" << nnz << " nonzeros) to " << out << '\n';
    }
    sb_free_csr(&A);
    return 0;
}

int cmd_coarsen_info(const Opts &o) {
    sb_csr A = load_system(o);
    sb_setup_opts so = setup_opts(o, true);
    so.coarse_solver = -1;  // only the level structure (tools/sparsh.cpp:322-324)
    sb_hier h = nullptr;
    const int rs = sb_setup(&A, &so, &h);
    sb_free_csr(&A);
    if (rs == SB_ERUNTIME) {
        std::cerr << "error: " << sb_last_error() << '\n';
        return 1;
    }
    ck(rs);
    print_levels(std::cout, level_stats(h), sb_hier_stalled(h) != 0);
    sb_hier_free(h);
    return 0;
}

int usage() {
    std::cerr << "usage: sparsh_b200 {run|gen|coarsen-info} [--key value ...]\n"
                 "  run          --problem SPEC | --matrix FILE [--solver amg|cg|pcg|bicgstab|pbicgstab]\n"
                 "               [--smoother jacobi] [--omega W] [--pre N] [--post N] [--coarse-target N]\n"
                 "               [--max-levels N] [--tol T] [--max-iters N] [--rhs ones|random|file:PATH]\n"
                 "               [--seed S] [--out CSV] [--config FILE] [--device D] [--host-levels-from K]\n"
                 "               [--galerkin-gpu 0|1]\n"
                 "  gen          --problem SPEC [--out FILE]\n"
                 "  coarsen-info --problem SPEC | --matrix FILE [--coarse-target N] [--max-levels N]\n";
    return 2;
}

} // namespace

int main(int argc, char **argv) {
    if (argc < 2) return usage();
    const std::string cmd = argv[1];
    try {
        Opts o;
        std::map<std::string, std::string> given;
        std::string gen_problem, gen_out;
        for (int i = 2; i < argc; ++i) {
            std::string a = argv[i];
            if (a.rfind("--", 0) != 0) throw usage_error("unexpected argument '" + a + "'");
            a = a.substr(2);
            std::string v;
            const auto eq = a.find('=');
            if (eq != std::string::npos) {
                v = a.substr(eq + 1);
                a = a.substr(0, eq);
            } else {
                if (i + 1 >= argc) throw usage_error("option --" + a + " needs a value");
                v = argv[++i];
            }
            given[a] = v;
            if (cmd == "gen") {
                if (a == "problem") gen_problem = v;
                else if (a == "out") gen_out = v;
                else throw usage_error("unknown option --" + a);
            } else {
                set_opt(o, a, v);
            }
        }
        if (cmd == "gen") {
            if (gen_problem.empty()) throw usage_error("--problem is required");
            return cmd_gen(gen_problem, gen_out);
        }
        apply_config(o, given);
        if (cmd == "run") return cmd_run(o);
        if (cmd == "coarsen-info") return cmd_coarsen_info(o);
        return usage();
    } catch (const usage_error &e) {
        std::cerr << "error: " << e.what() << '\n';
        return 2;
    } catch (const numeric_error &e) {
        std::cerr << "error: " << e.what() << '\n';
        return 1;
    } catch (const std::exception &e) {
        std::cerr << "error: " << e.what() << '\n';
        return 2;
    }
}
