// test_facade.cpp — the reference's own unit-test cases, re-run through the
// C++ entry points of include/hankel_b200.hpp (namespace hankel::b200).
//
// Host-only cases (moments, assignment, Jacobi, CSV/JSON) always run.  Device
// cases run when a CUDA device is usable; `--require-gpu` makes their absence
// a failure (the -m gpu pytest), otherwise they are reported as skipped.
// Each case cites the reference test it mirrors (proj/tests/*.cpp).
#include "hankel_b200.hpp"

#include <cstdio>
#include <cstring>
#include <sstream>
#include <string>

namespace hb = hankel::b200;

static int g_pass = 0, g_fail = 0;
#define CHECK(c)                                                                                                      \
    do {                                                                                                              \
        if (c)                                                                                                        \
            ++g_pass;                                                                                                 \
        else {                                                                                                        \
            ++g_fail;                                                                                                 \
            std::fprintf(stderr, "%s:%d: CHECK failed: %s\n", __FILE__, __LINE__, #c);                                \
        }                                                                                                             \
    } while (0)
#define CHECK_THROWS_AS(expr, T)                                                                                      \
    do {                                                                                                              \
        bool ok_ = false;                                                                                             \
        try {                                                                                                         \
            (void)(expr);                                                                                             \
        } catch (const T&) {                                                                                          \
            ok_ = true;                                                                                               \
        } catch (...) {                                                                                               \
        }                                                                                                             \
        CHECK(ok_ && #T);                                                                                             \
    } while (0)
static bool approx(double a, double b, double rel) { return std::fabs(a - b) <= rel * std::max(std::fabs(a), std::fabs(b)); }

// ------------------------------------------------------------------ host

static void host_cases() {
    // test_ldlt.cpp (assign_columns): boustrophedon, counts within one
    const auto a = hb::assign_columns(10, 3);
    const std::vector<int> want{0, 1, 2, 2, 1, 0, 0, 1, 2, 2};
    CHECK(a.owner == want);
    for (int w = 0; w < 3; ++w) CHECK(std::abs(int(a.owned(w).size()) - 10 / 3) <= 1);
    CHECK_THROWS_AS(hb::assign_columns(0, 2), std::invalid_argument);
    CHECK_THROWS_AS(hb::assign_columns(4, 0), std::invalid_argument);

    // test_moments.cpp:46-67: exact integer moments; WeightSpec::make validation
    CHECK_THROWS_AS(hb::WeightSpec::make(0, 1), std::invalid_argument);
    CHECK_THROWS_AS(hb::WeightSpec::make(4, 1), std::invalid_argument);
    const auto half = hb::WeightSpec::make(1, 2), one = hb::WeightSpec::make(1, 1), third = hb::WeightSpec::make(1, 3);
    double f = 1; // (2j+1)!
    for (int j = 0; j < 8; ++j) {
        f *= (j == 0 ? 1.0 : double(2 * j) * double(2 * j + 1));
        CHECK(hb::moment(half, unsigned(j), 4).to_double() == 2.0 * f); // mu_j = 2 (2j+1)!
    }
    CHECK(hb::moment(one, 5, 2).to_double() == 120.0);                 // 5!
    CHECK(hb::moment(third, 1, 2).to_double() == 3.0 * 120.0);          // 3 (3+2)!
    const auto tab = hb::build_hankel(one, 6, 4);
    CHECK(tab.exact() && tab.order() == 6 && tab.entry(2, 3) == tab.mu(5));
    CHECK(!hb::build_hankel(half, 64, 2).exact()); // 2 (253)! does not fit 64 bits
    {   // odd 2/beta: half-integer Gamma values, correctly rounded (test_moments.cpp:23-28 sqrt(pi) digits)
        const auto t2 = hb::build_hankel(hb::WeightSpec::make(2, 1), 4, 4); // beta = 2: mu_k = Gamma((k+1)/2) / 2
        CHECK(!t2.exact());
        CHECK(std::fabs(t2.mu(0).to_double() - 0.88622692545275801365) < 1e-16); // sqrt(pi) / 2
        CHECK(t2.mu(1).to_double() == 0.5);                                        // Gamma(1) / 2
        CHECK(std::fabs(t2.mu(2).to_double() - 0.44311346272637900682) < 1e-16); // sqrt(pi) / 4
        CHECK_THROWS_AS(hb::WeightSpec::make(3, 1), std::invalid_argument);     // 2/beta not an integer
    }
    CHECK(hb::moment_bits(one, 3) == 5);                                 // mu_4 = 24

    // MpFloat <-> binary64
    for (double x : {1.0, -3.5, 1e-300, 6.02214076e23, 0.1})
        CHECK(hb::MpFloat::from_double(x, 3).to_double() == x);

    // test_jacobi.cpp:24-44
    auto ev = hb::jacobi_eigenvalues({2, 1, 1, 2}, 2);
    CHECK(approx(ev[0], 1.0, 1e-14) && approx(ev[1], 3.0, 1e-14));
    ev = hb::jacobi_eigenvalues({5, 0, 0, 0, -1, 0, 0, 0, 2}, 3);
    CHECK((ev == std::vector<double>{-1, 2, 5}));
    const double A = 240.0 / 336.0, B = -12.0 / 336.0, C = 2.0 / 336.0;
    ev = hb::jacobi_eigenvalues({A, B, B, C}, 2);
    CHECK(approx(ev[1], 0.716081879923010796, 1e-14));
    CHECK(approx(ev[0], 0.00415621531508444244, 1e-12));
    CHECK_THROWS_AS(hb::jacobi_eigenvalues({1, 2, 3}, 2), std::invalid_argument);
    CHECK_THROWS_AS(hb::jacobi_eigenvalues({}, 0), std::invalid_argument);

    // test_jacobi.cpp:103-111: smallest eigenvalues of H from a binary64 block
    hb::TruncatedInverse blk;
    blk.k = 2;
    blk.M = {A, B, B, C};
    blk.M_minus = {A};
    const auto r = hb::smallest_eigs_of_H(blk, 1);
    CHECK(approx(r.lambda[0], 1.39648834586837266, 1e-13));
    CHECK(r.trunc_err[0] < 0);
    CHECK_THROWS_AS(hb::smallest_eigs_of_H(blk, 3), std::invalid_argument);
    hb::TruncatedInverse one_blk;
    one_blk.k = 1;
    one_blk.M = {0.5};
    const auto r1 = hb::smallest_eigs_of_H(one_blk, 1);
    CHECK(r1.lambda[0] == 2.0 && std::isnan(r1.trunc_err[0]));

    // test_pipeline.cpp (CSV / JSON shape): 20 columns, NaN rows, required_bits only when set
    hb::RunRecord rec;
    rec.n = 7;
    rec.bits = 1024;
    rec.k = 3;
    rec.workers = 2;
    rec.lambda = {0.25};
    rec.trunc_err = {-1e-20};
    const std::string row = hb::to_csv_row(rec);
    CHECK(std::count(row.begin(), row.end(), ',') == 19);
    CHECK(row.rfind("7,1/2,1024,3,2,0.25,", 0) == 0);
    CHECK(row.find("nan") != std::string::npos);
    std::ostringstream csv;
    hb::write_scan_csv(csv, {rec, rec});
    const std::string csv_s = csv.str();
    CHECK(std::count(csv_s.begin(), csv_s.end(), '\n') == 3);
    const std::string js = hb::to_json(rec);
    CHECK(js.find("\"N\": 7") != std::string::npos && js.find("required_bits") == std::string::npos);
    rec.required_bits = 2048;
    CHECK(hb::to_json(rec).find("\"required_bits\": 2048") != std::string::npos);

    // compute() argument checks happen before any device work (pipeline.cpp:27-30)
    hb::ComputeOptions bad;
    bad.n = 0;
    CHECK_THROWS_AS(hb::compute(bad), std::invalid_argument);
    bad.n = 4;
    bad.k = 0;
    CHECK_THROWS_AS(hb::compute(bad), std::invalid_argument);
}

// ---------------------------------------------------------------- device

static bool device_available() {
    try {
        hb::Device d(1);
        return true;
    } catch (const std::runtime_error&) {
        return false;
    }
}

static void device_cases() {
    const auto half = hb::WeightSpec::make(1, 2), one = hb::WeightSpec::make(1, 1);
    {   // test_ldlt.cpp:80-87: serial LDLT on the 2x2 case
        const auto table = hb::build_hankel(half, 2, 2);
        const auto f = hb::decompose_serial(table);
        CHECK(f.D.to_double(0) == 2.0);
        CHECK(f.D.to_double(1) == 168.0);
        CHECK(f.l_entry(1, 0).to_double() == 6.0);
        CHECK(f.update_count == 1);
    }
    {   // test_inversion.cpp:121-133: H_2^{-1} = (1/336) [[240, -12], [-12, 2]]
        const auto table = hb::build_hankel(half, 2, 8);
        const auto f = hb::decompose_serial(table);
        const auto inv = hb::invert_L_partial_serial(f, 2);
        const auto blk = hb::assemble_truncated_inverse(inv, 2);
        CHECK(approx(blk.at(0, 0), 240.0 / 336.0, 1e-15));
        CHECK(approx(blk.at(0, 1), -12.0 / 336.0, 1e-15));
        CHECK(approx(blk.at(1, 1), 2.0 / 336.0, 1e-15));
        CHECK(blk.at(0, 1) == blk.at(1, 0));
        CHECK(blk.M_minus.size() == 1 && blk.M_minus[0] == blk.at(0, 0));
        CHECK(inv.entry(1, 1).to_double() == 1.0 && inv.entry(0, 1).is_zero());
        CHECK(inv.entry(1, 0).to_double() == -6.0);
        CHECK_THROWS_AS(inv.entry(1, 2), std::out_of_range);
        const auto r = hb::smallest_eigs_of_H(blk, 1);
        CHECK(approx(r.lambda[0], 1.39648834586837266, 1e-15));
    }
    {   // test_inversion.cpp:112-116: rows[r] holds min(r, m) entries; argument checks
        const auto table = hb::build_hankel(half, 12, 16);
        const auto f = hb::decompose_serial(table);
        CHECK_THROWS_AS(hb::invert_L_partial_serial(f, 0), std::invalid_argument);
        CHECK_THROWS_AS(hb::invert_L_partial_serial(f, 13), std::invalid_argument);
        const auto inv = hb::invert_L_partial_serial(f, 5);
        CHECK(inv.X().size() == 12 * 5);
        CHECK_THROWS_AS(hb::assemble_truncated_inverse(inv, 6), std::invalid_argument);
    }
    {   // beta = 1 (Laguerre): d_n = (n!)^2, closed form
        const int n = 20;
        const auto table = hb::build_hankel(one, n, 8);
        const auto f = hb::decompose_serial(table);
        long double fact = 1;
        for (int i = 0; i < n; ++i) {
            if (i) fact *= i;
            CHECK(approx(f.D.to_double(size_t(i)), double(fact * fact), 1e-15));
        }
        // ldlt.hpp:92-96: bit-identical for any worker count (emulated split on this GPU)
        for (int w : {2, 3, 4}) {
            const auto g = hb::decompose_parallel(table, hb::assign_columns(n, w));
            CHECK(g.D.l == f.D.l && g.D.e == f.D.e && g.D.s == f.D.s);
            CHECK(g.L_column(3).l == f.L_column(3).l);
            CHECK(g.assignment.workers == w);
        }
        {   // any ColumnAssignment (ldlt.cpp:355-395): contiguous blocks and plain round robin
            hb::ColumnAssignment blk{n, 3, std::vector<int>(size_t(n))}, rr{n, 4, std::vector<int>(size_t(n))};
            for (int c = 0; c < n; ++c) {
                blk.owner[size_t(c)] = c * 3 / n;
                rr.owner[size_t(c)] = c % 4;
            }
            for (const auto& a : {blk, rr}) {
                const auto g = hb::decompose_parallel(table, a);
                CHECK(g.D.l == f.D.l && g.D.e == f.D.e && g.D.s == f.D.s);
                CHECK(g.L_column(7).l == f.L_column(7).l);
            }
            hb::ColumnAssignment bad = rr;
            bad.owner[5] = 9;
            CHECK_THROWS_AS(hb::decompose_parallel(table, bad), std::invalid_argument);
        }
        const auto rows = hb::transpose_redistribute(f);
        hb::WorkerTimings wt;
        const auto inv = hb::invert_L_partial_parallel(rows, 8, &wt);
        CHECK(wt.arith_s > 0);
        CHECK(hb::retranspose(rows).n == n);
    }
    {   // explicit Device: stale handles after the device is reused
        hb::Device dev(8);
        const auto f1 = hb::decompose_serial(dev, hb::build_hankel(one, 10, 8));
        const auto f2 = hb::decompose_serial(dev, hb::build_hankel(one, 12, 8));
        CHECK_THROWS_AS(hb::invert_L_partial_serial(f1, 2), std::logic_error);
        CHECK(hb::invert_L_partial_serial(f2, 2).m == 2);
        CHECK_THROWS_AS(hb::decompose_serial(dev, hb::build_hankel(one, 10, 4)), std::invalid_argument);
    }
    {   // ldlt.cpp:83-87 / test_ldlt.cpp precision exhaustion: non-positive pivot with its column
        hb::Device dev(1);
        bool thrown = false;
        try {
            hb::decompose_serial(dev, hb::build_hankel(one, 16, 1));
        } catch (const hb::precision_error& e) {
            thrown = std::strstr(e.what(), "pivot") != nullptr && dev.bad_column() > 0;
        }
        CHECK(thrown);
    }
    {   // test_pipeline.cpp:41-53: 2x2 pipeline and the quadratic-formula eigenvalue
        hb::ComputeOptions o;
        o.n = 2;
        o.bits = 256;
        o.k = 2;
        const auto r = hb::compute(o);
        CHECK(approx(r.lambda1(), 1.3964883458683727, 1e-15));
        CHECK(r.k == 2 && r.lambda.size() == 2 && r.p_bits % 128 == 0);
        o.n = 1;
        o.k = 8;
        const auto r1 = hb::compute(o); // k clamped to n (pipeline.cpp:36)
        CHECK(r1.k == 1 && approx(r1.lambda1(), 2.0, 1e-15) && std::isnan(r1.trunc_err[0]));
    }
    {   // test_pipeline.cpp:56-77: deterministic across repeats and worker counts
        hb::ComputeOptions o;
        o.n = 20;
        o.bits = 256;
        o.k = 8;
        const auto base = hb::compute(o);
        for (int w : {1, 2, 4}) {
            o.workers = w;
            const auto r = hb::compute(o);
            CHECK(r.lambda == base.lambda && r.trunc_err == base.trunc_err && r.workers == w);
        }
    }
    {   // pipeline.cpp:74-94: auto_precision (start 1024, step 1024) and scan with NaN rows
        hb::ComputeOptions o;
        o.n = 30;
        o.k = 8;
        const auto [bits, rec] = hb::auto_precision(o);
        CHECK(bits == 1024 && rec.required_bits == 1024);
        hb::ScanOptions so;
        so.base = o;
        so.base.bits = 256;
        const auto recs = hb::scan({4, 8}, so);
        CHECK(recs.size() == 2 && recs[1].n == 8 && !std::isnan(recs[1].lambda1()));
    }
}

int main(int argc, char** argv) {
    const bool require_gpu = argc > 1 && std::strcmp(argv[1], "--require-gpu") == 0;
    try {
        host_cases();
        if (device_available()) {
            device_cases();
        } else if (require_gpu) {
            std::fprintf(stderr, "no usable CUDA device\n");
            ++g_fail;
        } else {
            std::printf("device cases skipped (no CUDA device)\n");
        }
    } catch (const std::exception& e) {
        std::fprintf(stderr, "uncaught exception: %s\n", e.what());
        ++g_fail;
    }
    std::printf("test_facade: %d checks passed, %d failed\n", g_pass, g_fail);
    return g_fail == 0 ? 0 : 1;
}
