// oracle/ref_driver.cpp — TEST INFRASTRUCTURE ONLY (the checker, never the product).
//
// Drives the UNMODIFIED reference library (compiled from /root/reference by
// oracle/Makefile into oracle/_ref/) and prints machine-readable results:
//
//   ref_driver dump  --beta 1/2 --n 64 --bits 2048 --k 8 --workers 8
//       The reference pipeline stage by stage, exactly as hankel::compute
//       sequences it (proj/src/pipeline.cpp:41-66), plus — outside the timed
//       stages — the k x k block of H^{-1} kept in FIXED POINT: a restatement
//       of assemble_truncated_inverse (proj/src/inversion.cpp:244-262) that
//       stops before the binary64 cast at :258, so a >=20-digit eigenvalue can
//       be taken from it (SURVEY.md §0.3, §8c "20-digit λ").
//       Output: one JSON object with D (hex mantissas at K fractional bits),
//       the block (hex mantissas at 2K), the reference's binary64 lambdas and
//       the RunRecord-style stage timings.
//
//   ref_driver time  --beta 1/2 --n 256 --bits 2048 --k 8 --workers 8
//       hankel::compute() itself (proj/src/pipeline.cpp:26-72) and its
//       to_json(RunRecord) (pipeline.cpp:213-232): the CPU baseline arm.
//
//   ref_driver record  < records
//       The reference's RunRecord writers on given records (byte-level parity
//       of the product's to_csv_row / to_json): per stdin line
//         n bnum bden bits k workers required_bits nl l_1..l_nl nt t_1..t_nt
//         wall ldlt transpose invL invL_arith invL_comm invH eigen
//       (doubles as C99 hex floats) prints to_csv_row (pipeline.cpp:150-160),
//       then to_json (pipeline.cpp:213-232), then a line "@@".
#include "hankel/errors.hpp"
#include "hankel/inversion.hpp"
#include "hankel/jacobi.hpp"
#include "hankel/ldlt.hpp"
#include "hankel/moments.hpp"
#include "hankel/pipeline.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <iostream>
#include <sstream>
#include <string>
#include <thread>

using namespace hankel;
using Clock = std::chrono::steady_clock;

namespace {

double since(Clock::time_point t0) { return std::chrono::duration<double>(Clock::now() - t0).count(); }

struct Args {
    std::string mode;
    unsigned bnum = 1, bden = 2;
    int n = 2;
    long bits = 64;
    int k = 8;
    int workers = 1;
};

Args parse(int argc, char** argv) {
    Args a;
    if (argc < 2) throw std::invalid_argument("usage: ref_driver dump|time --beta a/b --n N --bits K --k k --workers W");
    a.mode = argv[1];
    for (int i = 2; i + 1 < argc; i += 2) {
        const std::string f = argv[i], v = argv[i + 1];
        if (f == "--beta") {
            const auto s = v.find('/');
            a.bnum = unsigned(std::stoul(v.substr(0, s)));
            a.bden = s == std::string::npos ? 1u : unsigned(std::stoul(v.substr(s + 1)));
        } else if (f == "--n") a.n = std::stoi(v);
        else if (f == "--bits") a.bits = std::stol(v);
        else if (f == "--k") a.k = std::stoi(v);
        else if (f == "--workers") a.workers = std::stoi(v);
        else throw std::invalid_argument("unknown flag " + f);
    }
    if (a.workers <= 0) a.workers = int(std::max(1u, std::thread::hardware_concurrency()));
    return a;
}

std::string num(double v) {
    if (std::isnan(v) || std::isinf(v)) return "null";
    std::ostringstream os;
    os.precision(17);
    os << v;
    return os.str();
}

std::string hex(const FixScalar& x) {
    const mpz_class& m = x.mantissa();
    return m.get_str(16);
}

int run_dump(const Args& a) {
    const WeightSpec beta = WeightSpec::make(a.bnum, a.bden);
    const int k = std::min(a.k, a.n);
    std::ostringstream js;
    const auto t_wall = Clock::now();
    const MomentTable table = build_hankel(beta, a.n, a.bits);
    const ColumnAssignment asg = assign_columns(a.n, a.workers);
    auto t0 = Clock::now();
    const LdltFactors f = decompose_parallel(table, asg);
    const double ldlt_s = since(t0);
    t0 = Clock::now();
    const RowDistributedL rows = transpose_redistribute(f);
    const double transpose_s = since(t0);
    t0 = Clock::now();
    const PartialInverse inv = invert_L_partial_parallel(rows, k);
    const double invL_s = since(t0);
    t0 = Clock::now();
    const TruncatedInverse block = assemble_truncated_inverse(inv, k);
    const double invH_s = since(t0);
    t0 = Clock::now();
    const SmallestEigResult eig = smallest_eigs_of_H(block, std::min(3, k));
    const double eigen_s = since(t0);
    const double wall_s = since(t_wall);

    // Fixed-point block, restating proj/src/inversion.cpp:244-262 without the
    // binary64 cast of :258.  Same term order (l ascending from max(j,c)), same
    // exact product (:255), same RNE division by D_l at 2K (:256), exact sum.
    const long K = inv.frac_bits, WK = 2 * K;
    const FixScalar one = FixScalar::from_integer(1, K);
    auto lv = [&](int l, int col) -> const FixScalar& { return l == col ? one : inv.rows[size_t(l)][size_t(col)]; };
    std::vector<FixScalar> M(size_t(k) * size_t(k));
    for (int j = 0; j < k; ++j)
        for (int c = j; c < k; ++c) {
            FixScalar acc = FixScalar::from_integer(0, WK);
            for (int l = std::max(j, c); l < a.n; ++l) acc = acc + (lv(l, j) * lv(l, c)).div(inv.D[size_t(l)], WK);
            M[size_t(j) * size_t(k) + size_t(c)] = acc;
            M[size_t(c) * size_t(k) + size_t(j)] = acc;
        }

    js << "{\"n\":" << a.n << ",\"beta\":\"" << a.bnum << "/" << a.bden << "\",\"bits\":" << a.bits
       << ",\"k\":" << k << ",\"workers\":" << a.workers << ",\"update_count\":" << f.update_count;
    js << ",\"D\":[";
    for (int i = 0; i < a.n; ++i) js << (i ? "," : "") << "\"" << hex(f.D[size_t(i)]) << "\"";
    js << "],\"L_col0\":[";
    for (size_t r = 0; r < f.L[0].size(); ++r) js << (r ? "," : "") << "\"" << hex(f.L[0][r]) << "\"";
    js << "],\"Linv\":[";
    for (int r = 0; r < (a.n <= 128 ? a.n : 0); ++r) {  // bulky: only for small orders
        js << (r ? "," : "") << "[";
        for (size_t c = 0; c < inv.rows[size_t(r)].size(); ++c) js << (c ? "," : "") << "\"" << hex(inv.rows[size_t(r)][c]) << "\"";
        js << "]";
    }
    js << "],\"block_frac_bits\":" << WK << ",\"block\":[";
    for (size_t i = 0; i < M.size(); ++i) js << (i ? "," : "") << "\"" << hex(M[i]) << "\"";
    js.precision(17);
    js << "],\"lambda\":[";
    for (size_t i = 0; i < eig.lambda.size(); ++i) js << (i ? "," : "") << num(eig.lambda[i]);
    js << "],\"trunc_err\":[";
    for (size_t i = 0; i < eig.trunc_err.size(); ++i) js << (i ? "," : "") << num(eig.trunc_err[i]);
    js << "],\"timing\":{\"wall_s\":" << wall_s << ",\"ldlt_s\":" << ldlt_s << ",\"transpose_s\":" << transpose_s
       << ",\"invL_s\":" << invL_s << ",\"invH_s\":" << invH_s << ",\"eigen_s\":" << eigen_s << "}}";
    std::cout << js.str() << std::endl;
    return 0;
}

int run_time(const Args& a) {
    ComputeOptions o;
    o.n = a.n;
    o.beta = WeightSpec::make(a.bnum, a.bden);
    o.bits = a.bits;
    o.k = a.k;
    o.workers = a.workers;
    const RunRecord r = compute(o);
    std::string s = to_json(r);
    for (auto& ch : s)
        if (ch == '\n') ch = ' ';
    std::cout << s << std::endl;
    return 0;
}

} // namespace

int run_record() {
    std::string line;
    while (std::getline(std::cin, line)) {
        if (line.empty()) continue;
        std::istringstream is(line);
        auto dbl = [&]() {
            std::string t;
            is >> t;
            return std::strtod(t.c_str(), nullptr);
        };
        RunRecord r;
        unsigned bn = 1, bd = 2;
        is >> r.n >> bn >> bd >> r.bits >> r.k >> r.workers >> r.required_bits;
        r.beta = WeightSpec::make(bn, bd);
        size_t nl = 0, nt = 0;
        is >> nl;
        for (size_t i = 0; i < nl; ++i) r.lambda.push_back(dbl());
        is >> nt;
        for (size_t i = 0; i < nt; ++i) r.trunc_err.push_back(dbl());
        for (double* f : {&r.wall_s, &r.ldlt_s, &r.transpose_s, &r.invL_s, &r.invL_arith_s, &r.invL_comm_s, &r.invH_s,
                          &r.eigen_s})
            *f = dbl();
        std::cout << to_csv_row(r) << "\n" << to_json(r) << "\n@@" << std::endl;
    }
    return 0;
}

int main(int argc, char** argv) {
    try {
        if (argc >= 2 && std::string(argv[1]) == "record") return run_record();
        const Args a = parse(argc, argv);
        if (a.mode == "dump") return run_dump(a);
        if (a.mode == "time") return run_time(a);
        std::cerr << "unknown mode " << a.mode << "\n";
        return 3;
    } catch (const precision_error& e) {
        std::cerr << "precision_error: " << e.what() << "\n";
        return 2;
    } catch (const std::invalid_argument& e) {
        std::cerr << "invalid_argument: " << e.what() << "\n";
        return 3;
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
}
