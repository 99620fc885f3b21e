// hankel_b200.hpp — the reference's C++ entry points over the B200 C ABI.
//
// The reference (hankel-eig, proj/include/hankel/*.hpp) is a C++20 library of
// free functions in `namespace hankel`.  This header keeps those entry points —
// same names, argument meaning and exception types — in `namespace
// hankel::b200`, implemented on top of the C ABI of include/hankel_b200.h (link
// -lhankel_b200).  Header-only C++20; no CUDA or torch types.
//
//   reference (proj/include/hankel)                here
//   WeightSpec, moment, MomentTable, build_hankel  same (moments.hpp:13-58); p = 32*limbs
//                                                  replaces frac_bits
//   assign_columns, ColumnAssignment               same (ldlt.hpp:13-21)
//   LdltFactors, decompose_serial/_parallel        same (ldlt.hpp:76-99); factors stay on the GPU
//   RowDistributedL, transpose_redistribute,       same (inversion.hpp:13-46); the GPU needs no
//   retranspose, PartialInverse,                   row redistribution (the handle is the factors)
//   invert_L_partial_serial/_parallel
//   TruncatedInverse, assemble_truncated_inverse   same (inversion.hpp:50-60) + the MP block
//   JacobiOptions, jacobi_eigenvalues,             same (jacobi.hpp:11-30); binary128 inside, lambda
//   SmallestEigResult, smallest_eigs_of_H          also as hi + lo (~32 digits)
//   ComputeOptions, RunRecord, compute,            same (pipeline.hpp:16-70); `workers` = GPUs,
//   AutoPrecisionOptions, auto_precision, scan,    `bits` = the reference's K, mapped to
//   CSV / JSON writers                             p(K) (precision_bits)
//   precision_error                                same (errors.hpp:7)
//
// Values: the reference's FixScalar (mpz mantissa / 2^K) becomes MpFloat, a
// p-bit binary float (sign, exponent, 32-bit limbs, value = sign*M*2^(e-p)).
// Device state: `Device` owns one hk_ctx (one GPU, or one rank of a sharded
// group).  The free functions with the reference's exact signatures run on a
// per-thread default Device for the table's precision (device 0); the
// overloads taking a Device& are the explicit form.  Factor / inverse handles
// refer to the device state they were computed in; reusing the Device for a
// new factorisation makes old handles stale (std::logic_error on use).
#pragma once

#include "hankel_b200.h"

#include <algorithm>
#include <cstring>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <iomanip>
#include <limits>
#include <map>
#include <memory>
#include <ostream>
#include <sstream>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace hankel::b200 {

// errors.hpp:7 — a non-positive pivot / zero D / precision search exhausted
class precision_error : public std::runtime_error {
public:
    using std::runtime_error::runtime_error;
};

namespace detail {
[[noreturn]] inline void throw_status(int rc, const std::string& msg) {
    if (rc == HK_ERR_PRECISION) throw precision_error(msg);
    if (rc == HK_ERR_INVALID) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
}
inline void check(int rc, const char* what) {
    if (rc != HK_OK) throw_status(rc, what);
}
} // namespace detail

// ------------------------------------------------------------------ values

// One p-bit float: value = sign * M * 2^(exp - p), M = sum limbs[i] 2^(32 i),
// 2^(p-1) <= M < 2^p (sign 0: zero).  The role of FixScalar (fixedpoint.hpp:23).
struct MpFloat {
    int sign = 0;
    int exp = 0;
    std::vector<uint32_t> limbs;

    int bits() const { return 32 * int(limbs.size()); }
    bool is_zero() const { return sign == 0; }
    // nearest binary64 of the value (RNE on the top 64 bits + sticky)
    double to_double() const {
        if (sign == 0 || limbs.empty()) return 0.0;
        const int L = int(limbs.size());
        uint64_t top = (uint64_t(limbs[size_t(L - 1)]) << 32) | (L >= 2 ? limbs[size_t(L - 2)] : 0u);
        bool sticky = false;
        for (int i = 0; i < L - 2; ++i) sticky = sticky || limbs[size_t(i)] != 0;
        // top has its msb set; keep 53 bits, round to nearest even on the 11 below (+ sticky)
        const uint64_t mant = top >> 11, rest = top & 0x7ff;
        uint64_t m53 = mant;
        if (rest > 0x400 || (rest == 0x400 && (sticky || (mant & 1)))) ++m53;
        // value = top * 2^(exp - 64)  (top = M >> (p - 64))
        const double v = std::ldexp(double(m53), exp - 53);
        if (std::isinf(v)) throw std::overflow_error("MpFloat::to_double: out of binary64 range"); // fixedpoint.cpp:115-116
        return sign < 0 ? -v : v;
    }
    bool operator==(const MpFloat& o) const { return sign == o.sign && (sign == 0 || (exp == o.exp && limbs == o.limbs)); }
    bool operator!=(const MpFloat& o) const { return !(*this == o); }

    // exact value of a binary64 at `limbs` limbs (limbs >= 2)
    static MpFloat from_double(double x, int limbs) {
        if (limbs < 2) throw std::invalid_argument("MpFloat::from_double: need >= 2 limbs");
        MpFloat f;
        f.limbs.assign(size_t(limbs), 0u);
        if (x == 0.0) return f;
        if (!std::isfinite(x)) throw std::overflow_error("MpFloat::from_double: not finite");
        int e = 0;
        const double fr = std::frexp(std::fabs(x), &e); // |x| = fr 2^e, fr in [0.5, 1)
        const uint64_t m = uint64_t(std::ldexp(fr, 64)); // exact: 53 significant bits
        f.limbs[size_t(limbs - 1)] = uint32_t(m >> 32);
        f.limbs[size_t(limbs - 2)] = uint32_t(m);
        f.sign = x < 0 ? -1 : 1;
        f.exp = e;
        return f;
    }
};

// Host SoA array of p-bit floats — the C ABI's interchange format.
struct MpVector {
    int limbs = 0;
    std::vector<uint32_t> l;
    std::vector<int32_t> e, s;

    MpVector() = default;
    MpVector(size_t n, int limbs_) : limbs(limbs_), l(n * size_t(limbs_)), e(n), s(n) {}
    size_t size() const { return e.size(); }
    MpFloat at(size_t i) const {
        MpFloat f;
        f.sign = s.at(i);
        f.exp = e[i];
        f.limbs.assign(l.begin() + long(i * size_t(limbs)), l.begin() + long((i + 1) * size_t(limbs)));
        return f;
    }
    void set(size_t i, const MpFloat& f) {
        if (int(f.limbs.size()) != limbs) throw std::invalid_argument("MpVector::set: limb count");
        std::copy(f.limbs.begin(), f.limbs.end(), l.begin() + long(i * size_t(limbs)));
        e.at(i) = f.exp;
        s[i] = f.sign;
    }
    double to_double(size_t i) const { return at(i).to_double(); }
    uint32_t* pl() { return l.data(); }
    int32_t* pe() { return e.data(); }
    int32_t* ps() { return s.data(); }
    const uint32_t* pl() const { return l.data(); }
    const int32_t* pe() const { return e.data(); }
    const int32_t* ps() const { return s.data(); }
};

// ----------------------------------------------------------------- moments

// moments.hpp:13-22.  beta = num/den; 2/beta must be a positive integer
// (make, moments.cpp:72-78).  Odd 2/beta (half-integer Gamma) is not on the
// device path (hk_moments -> std::invalid_argument).
struct WeightSpec {
    unsigned beta_num = 1;
    unsigned beta_den = 2;

    unsigned long doubled_inverse() const { return 2ul * beta_den / beta_num; }
    static WeightSpec make(unsigned num, unsigned den) {
        if (num == 0 || den == 0) throw std::invalid_argument("beta must be positive");
        if ((2ul * den) % num != 0) throw std::invalid_argument("unsupported beta: 2/beta must be a positive integer");
        return WeightSpec{num, den};
    }
    bool operator==(const WeightSpec&) const = default;
};

// The 2n-1 moments mu_0..mu_{2n-2} at p = 32*limbs bits; entry(i,j) = mu_{i+j}
// (moments.hpp:36-55).  exact(): every moment is held without rounding.
class MomentTable {
public:
    MomentTable(WeightSpec spec, int n, int limbs) : spec_(spec), n_(n), limbs_(limbs) {
        if (n < 1) throw std::invalid_argument("build_hankel: order must be >= 1");
        if (limbs < 1) throw std::invalid_argument("build_hankel: need >= 1 limb");
        mu_ = MpVector(size_t(2 * n - 1), limbs);
        int exact = 0;
        detail::check(hk_moments(spec.beta_num, spec.beta_den, 2 * n - 1, limbs, mu_.pl(), mu_.pe(), mu_.ps(), &exact),
                      "build_hankel: unsupported beta (2/beta must be an even integer on this path)");
        exact_ = exact != 0;
    }
    int order() const noexcept { return n_; }
    int limbs() const noexcept { return limbs_; }
    int bits() const noexcept { return 32 * limbs_; }
    bool exact() const noexcept { return exact_; }
    const WeightSpec& weight() const noexcept { return spec_; }
    MpFloat mu(size_t k) const { return mu_.at(k); }
    MpFloat entry(int i, int j) const { return mu_.at(size_t(i) + size_t(j)); }
    const MpVector& moments() const noexcept { return mu_; }

private:
    WeightSpec spec_;
    int n_, limbs_;
    bool exact_ = false;
    MpVector mu_;
};

inline MomentTable build_hankel(const WeightSpec& spec, int n, int limbs) { return MomentTable(spec, n, limbs); }

// moment(spec, k, frac_bits) (moments.hpp:33): mu_k at p = 32*limbs bits
inline MpFloat moment(const WeightSpec& spec, unsigned long k, int limbs) {
    MpVector v(size_t(k) + 1, limbs);
    int exact = 0;
    detail::check(hk_moments(spec.beta_num, spec.beta_den, int(k) + 1, limbs, v.pl(), v.pe(), v.ps(), &exact),
                  "moment: unsupported beta");
    return v.at(size_t(k));
}

// ------------------------------------------------------------- assignment

// ldlt.hpp:13-21; the boustrophedon map of ldlt.cpp:22-35 (hk_assign_columns)
struct ColumnAssignment {
    int n = 0;
    int workers = 1;
    std::vector<int> owner;

    std::vector<int> owned(int worker) const {
        std::vector<int> out;
        for (int c = 0; c < n; ++c)
            if (owner[size_t(c)] == worker) out.push_back(c);
        return out;
    }
};

inline ColumnAssignment assign_columns(int n, int workers) {
    if (n < 1) throw std::invalid_argument("assign_columns: order must be >= 1");
    if (workers < 1) throw std::invalid_argument("assign_columns: worker count must be >= 1");
    ColumnAssignment a;
    a.n = n;
    a.workers = workers;
    a.owner.resize(size_t(n));
    std::vector<int32_t> o(static_cast<size_t>(n));
    detail::check(hk_assign_columns(n, workers, o.data()), "assign_columns");
    std::copy(o.begin(), o.end(), a.owner.begin());
    return a;
}

// ------------------------------------------------------------------ device

// One hk_ctx: a GPU at p = 32*limbs bits, or one rank of a column-sharded
// group (one process per GPU, ncclUniqueId shared by the caller), or — with
// nccl_id128 == nullptr and world > 1 — all `world` ranks emulated on one GPU.
class Device {
public:
    explicit Device(int limbs, int device = 0) { detail::check(hk_create(device, limbs, &h_), "hk_create: no usable CUDA device"); }
    Device(int limbs, int device, int rank, int world, const void* nccl_id128) {
        detail::check(hk_create_sharded(device, limbs, rank, world, nccl_id128, &h_), "hk_create_sharded failed");
    }
    static Device emulated_group(int limbs, int world, int device = 0) { return Device(limbs, device, 0, world, nullptr); }
    ~Device() {
        if (h_) hk_destroy(h_);
    }
    Device(const Device&) = delete;
    Device& operator=(const Device&) = delete;
    Device(Device&& o) noexcept : h_(o.h_), gen_(o.gen_), inv_gen_(o.inv_gen_) { o.h_ = nullptr; }
    Device& operator=(Device&& o) noexcept {
        if (this != &o) {
            if (h_) hk_destroy(h_);
            h_ = o.h_;
            gen_ = o.gen_;
            inv_gen_ = o.inv_gen_;
            o.h_ = nullptr;
        }
        return *this;
    }

    hk_ctx* handle() const noexcept { return h_; }
    int limbs() const { return hk_limbs(h_); }
    // new precision on the same device / communicator (invalidates earlier factor handles)
    void set_limbs(int limbs) {
        if (limbs == this->limbs()) return;
        check(hk_set_limbs(h_, limbs));
        ++gen_;
        ++inv_gen_;
    }
    // kernel_times()[3]: device ms of this rank's pivot-column broadcasts in the last LDLT
    std::vector<double> kernel_times() const {
        std::vector<double> t(6);
        check(hk_kernel_times(h_, t.data()));
        return t;
    }
    int bits() const { return 32 * limbs(); }
    int rank() const {
        int r = 0, w = 1;
        hk_world(h_, &r, &w);
        return r;
    }
    int world() const {
        int r = 0, w = 1;
        hk_world(h_, &r, &w);
        return w;
    }
    // status -> the reference's exception types, message from hk_last_error
    void check(int rc) const {
        if (rc == HK_OK) return;
        std::string msg = hk_last_error(h_);
        detail::throw_status(rc, msg);
    }
    int bad_column() const { return hk_bad_column(h_); }
    // RunRecord stage times of the last calls: wall, ldlt, invL, invH, eigen, h2d, d2h
    std::vector<double> timings() const {
        std::vector<double> t(7);
        hk_timings(h_, t.data());
        return t;
    }
    unsigned long long generation() const noexcept { return gen_; }
    unsigned long long inverse_generation() const noexcept { return inv_gen_; }
    unsigned long long bump() noexcept { return ++gen_; }
    unsigned long long bump_inverse() noexcept { return ++inv_gen_; }

private:
    hk_ctx* h_ = nullptr;
    unsigned long long gen_ = 0, inv_gen_ = 0;
};

namespace detail {
// per-thread default devices: (limbs, emulated world) -> Device on device 0
inline Device& default_device(int limbs, int world = 1) {
    thread_local std::map<std::pair<int, int>, std::unique_ptr<Device>> devs;
    auto& d = devs[{limbs, world}];
    if (!d) d = world == 1 ? std::make_unique<Device>(limbs, 0) : std::make_unique<Device>(Device::emulated_group(limbs, world));
    return *d;
}
} // namespace detail

// ------------------------------------------------------------------- LDLT

struct WorkerTimings { // ldlt.hpp:63-66: here device time of the factorisation
    double arith_s = 0.0;
    double comm_s = 0.0;
};

// ldlt.hpp:76-85.  D on the host; L(row, col) fetched per column on demand.
// On ranks != 0 of a real sharded group the factors live on rank 0 only
// (resident() is false and D is empty).
struct LdltFactors {
    int n = 0;
    int limbs = 0;
    ColumnAssignment assignment;
    MpVector D;
    unsigned long long update_count = 0; // n(n^2-1)/6 (ldlt.cpp:128)

    Device* device = nullptr;
    unsigned long long generation = 0;

    bool resident() const { return device && device->rank() == 0; }
    void require_current() const {
        if (!device || device->generation() != generation)
            throw std::logic_error("LdltFactors: the device was reused for another factorisation (stale handle)");
    }
    // column j of L below the diagonal: rows j+1..n-1 (L[j] of ldlt.hpp:82)
    const MpVector& L_column(int j) const {
        if (j < 0 || j >= n) throw std::out_of_range("LdltFactors: column out of range");
        auto it = cols_.find(j);
        if (it != cols_.end()) return it->second;
        require_current();
        MpVector c(size_t(n - j - 1), limbs);
        device->check(hk_get_L_column(device->handle(), j, c.pl(), c.pe(), c.ps()));
        return cols_.emplace(j, std::move(c)).first->second;
    }
    MpFloat l_entry(int row, int col) const { // ldlt.hpp:84
        if (row <= col || row >= n) throw std::out_of_range("LdltFactors: need col < row < n");
        return L_column(col).at(size_t(row - col - 1));
    }

private:
    mutable std::map<int, MpVector> cols_;
};

inline LdltFactors decompose_parallel(Device& dev, const MomentTable& table, WorkerTimings* host_timings = nullptr) {
    if (dev.limbs() != table.limbs())
        throw std::invalid_argument("decompose: table precision differs from the device's");
    const int n = table.order();
    const MpVector& mu = table.moments();
    dev.check(hk_load_moments(dev.handle(), n, mu.pl(), mu.pe(), mu.ps()));
    const unsigned long long gen = dev.bump();
    dev.check(hk_ldlt(dev.handle()));
    LdltFactors f;
    f.n = n;
    f.limbs = table.limbs();
    f.assignment = assign_columns(n, dev.world());
    f.update_count = (unsigned long long)n * ((unsigned long long)n * n - 1) / 6;
    f.device = &dev;
    f.generation = gen;
    if (f.resident()) {
        f.D = MpVector(size_t(n), f.limbs);
        dev.check(hk_get_D(dev.handle(), f.D.pl(), f.D.pe(), f.D.ps()));
    }
    if (host_timings) { // ldlt.cpp:214-263, 341: comm = waiting on / moving the pivot column
        const double comm = dev.kernel_times()[3] * 1e-3;
        host_timings->comm_s = comm;
        host_timings->arith_s = dev.timings()[1] - comm;
    }
    return f;
}
inline LdltFactors decompose_serial(Device& dev, const MomentTable& table) { return decompose_parallel(dev, table); }

// the reference's signatures (ldlt.hpp:90, 97-99): per-thread default device
// for the table's precision; assignment.workers > 1 emulates that column split
// on one GPU (bit-identical results; one Device per rank with an NCCL id is the
// multi-GPU form).  The broadcast policy only shapes host timing in the
// reference and never values, so it is accepted and ignored.
struct BroadcastPolicy { // ldlt.hpp:23-26
    int chunk_values = 100;
    long min_outstanding_mults = 8000;
};
inline LdltFactors decompose_serial(const MomentTable& table) {
    return decompose_parallel(detail::default_device(table.limbs()), table);
}
inline LdltFactors decompose_parallel(const MomentTable& table, const ColumnAssignment& assignment,
                                      const BroadcastPolicy& = {}, WorkerTimings* host_timings = nullptr) {
    if (assignment.n != table.order() || assignment.workers < 1 || int(assignment.owner.size()) != assignment.n)
        throw std::invalid_argument("decompose_parallel: assignment does not match the table");
    Device& dev = detail::default_device(table.limbs(), assignment.workers);
    if (assignment.workers > 1) { // any map (ldlt.cpp:355-395 takes any assignment); results do not depend on it
        const std::vector<int32_t> o(assignment.owner.begin(), assignment.owner.end());
        dev.check(hk_set_owner_map(dev.handle(), assignment.n, o.data()));
    }
    return decompose_parallel(dev, table, host_timings);
}

// ---------------------------------------------------------------- inverse

// inversion.hpp:13-21.  The device factors are read row-wise in place, so the
// redistribution is the identity on the data; the handle carries the row map.
struct RowDistributedL {
    int n = 0;
    int limbs = 0;
    ColumnAssignment row_owner;
    const LdltFactors* factors = nullptr;
};
inline RowDistributedL transpose_redistribute(const LdltFactors& f) {
    f.require_current();
    return RowDistributedL{f.n, f.limbs, assign_columns(f.n, f.assignment.workers), &f};
}
inline LdltFactors retranspose(const RowDistributedL& rows) {
    if (!rows.factors) throw std::invalid_argument("retranspose: empty handle");
    return *rows.factors;
}

// inversion.hpp:29-38: X = first m columns of L^{-1}; rows[r] = first min(r, m) entries
struct PartialInverse {
    int n = 0;
    int m = 0;
    int limbs = 0;
    MpVector D;
    Device* device = nullptr;
    unsigned long long generation = 0, inverse_generation = 0;

    void require_current() const {
        if (!device || device->generation() != generation || device->inverse_generation() != inverse_generation)
            throw std::logic_error("PartialInverse: the device was reused (stale handle)");
    }
    // row-major n x m, entry (r, c) = L^{-1}(r, c) for c < r (hk_get_Linv)
    const MpVector& X() const {
        if (x_.size() == 0 && n > 0) {
            require_current();
            MpVector x(size_t(n) * size_t(m), limbs);
            device->check(hk_get_Linv(device->handle(), x.pl(), x.pe(), x.ps()));
            x_ = std::move(x);
        }
        return x_;
    }
    MpFloat entry(int row, int col) const { // inversion.cpp:55-60
        if (col >= m) throw std::out_of_range("PartialInverse: column beyond retained block");
        MpFloat z;
        z.limbs.assign(size_t(limbs), 0u);
        if (col > row) return z;
        if (col == row) {
            z.sign = 1;
            z.exp = 1;
            z.limbs[size_t(limbs - 1)] = 0x80000000u;
            return z;
        }
        return X().at(size_t(row) * size_t(m) + size_t(col));
    }

private:
    mutable MpVector x_;
};

inline PartialInverse invert_L_partial_serial(const LdltFactors& f, int m) {
    f.require_current();
    if (m < 1 || m > f.n) throw std::invalid_argument("invert_L_partial: need 1 <= m <= n");
    f.device->check(hk_invert_L_partial(f.device->handle(), m));
    PartialInverse p;
    p.n = f.n;
    p.m = m;
    p.limbs = f.limbs;
    p.D = f.D;
    p.device = f.device;
    p.generation = f.generation;
    p.inverse_generation = f.device->bump_inverse();
    return p;
}
inline PartialInverse invert_L_partial_parallel(const RowDistributedL& rows, int m,
                                                WorkerTimings* host_timings = nullptr) {
    if (!rows.factors) throw std::invalid_argument("invert_L_partial_parallel: empty handle");
    PartialInverse p = invert_L_partial_serial(*rows.factors, m);
    if (host_timings) {
        host_timings->arith_s = p.device->timings()[2];
        host_timings->comm_s = 0.0;
    }
    return p;
}

// inversion.hpp:50-56, plus the block in MP (`Mp`, k x k row-major) — the
// reference casts each entry to binary64 (inversion.cpp:258); here M is that
// cast and Mp keeps the p-bit sums for the ~32-digit eigensolve.
struct TruncatedInverse {
    int k = 0;
    std::vector<double> M;       // k*k, row-major, exactly symmetric
    std::vector<double> M_minus; // (k-1)*(k-1), row-major
    MpVector Mp;                 // k*k p-bit block (empty for a user-built block)
    double at(int i, int j) const { return M[size_t(i) * size_t(k) + size_t(j)]; }
};

inline TruncatedInverse assemble_truncated_inverse(const PartialInverse& inv, int k) {
    if (k < 1 || k > inv.m) throw std::invalid_argument("assemble_truncated_inverse: need 1 <= k <= m");
    inv.require_current();
    inv.device->check(hk_assemble_block(inv.device->handle(), k));
    TruncatedInverse t;
    t.k = k;
    t.Mp = MpVector(size_t(k) * size_t(k), inv.limbs);
    inv.device->check(hk_get_block(inv.device->handle(), t.Mp.pl(), t.Mp.pe(), t.Mp.ps()));
    t.M.resize(size_t(k) * size_t(k));
    for (size_t q = 0; q < t.M.size(); ++q) t.M[q] = t.Mp.to_double(q);
    if (k > 1) {
        t.M_minus.resize(size_t(k - 1) * size_t(k - 1));
        for (int j = 0; j < k - 1; ++j)
            for (int c = 0; c < k - 1; ++c) t.M_minus[size_t(j) * size_t(k - 1) + size_t(c)] = t.at(j, c);
    }
    return t;
}

// ------------------------------------------------------------------ eigen

struct JacobiOptions { // jacobi.hpp:11-14
    double tol_factor = 1e-14;
    int max_sweeps = 100;
};

inline std::vector<double> jacobi_eigenvalues(std::vector<double> m, int k, const JacobiOptions& opts = {}) {
    if (k < 1) throw std::invalid_argument("jacobi_eigenvalues: need k >= 1");
    if (m.size() != size_t(k) * size_t(k)) throw std::invalid_argument("jacobi_eigenvalues: matrix size != k*k");
    std::vector<double> ev(static_cast<size_t>(k));
    const int rc = hk_jacobi_eigenvalues(m.data(), k, opts.tol_factor, opts.max_sweeps, ev.data());
    if (rc == HK_ERR_RUNTIME) throw std::runtime_error("jacobi_eigenvalues: no convergence after max sweeps");
    detail::check(rc, "jacobi_eigenvalues: invalid arguments");
    return ev;
}

struct SmallestEigResult { // jacobi.hpp:23-27 (+ lambda_lo: lambda = lambda + lambda_lo to ~32 digits)
    std::vector<double> lambda;
    std::vector<double> trunc_err;
    int k_used = 0;
    std::vector<double> lambda_lo;
};

// jacobi.hpp:29-30: lambda_i = 1 / mu_{k+1-i} of the block, trunc_err_i vs the
// (k-1) block.  On the MP block when present (binary128 Jacobi of the p-bit
// sums), else on the binary64 block M.
inline SmallestEigResult smallest_eigs_of_H(const TruncatedInverse& block, int s, const JacobiOptions& = {}) {
    const int k = block.k;
    if (s < 1 || s > k) throw std::invalid_argument("smallest_eigs_of_H: need 1 <= s <= k");
    MpVector src = block.Mp;
    if (src.size() != size_t(k) * size_t(k)) {
        if (block.M.size() != size_t(k) * size_t(k)) throw std::invalid_argument("smallest_eigs_of_H: block size");
        src = MpVector(size_t(k) * size_t(k), 4);
        for (size_t q = 0; q < block.M.size(); ++q) src.set(q, MpFloat::from_double(block.M[q], 4));
    }
    SmallestEigResult r;
    r.lambda.resize(size_t(s));
    r.lambda_lo.resize(size_t(s));
    r.trunc_err.resize(size_t(s));
    const int rc = hk_block_eigenvalues(k, src.limbs, src.pl(), src.pe(), src.ps(), s, r.lambda.data(),
                                        r.lambda_lo.data(), r.trunc_err.data());
    if (rc == HK_ERR_RUNTIME)
        throw std::runtime_error("smallest_eigs_of_H: non-positive block eigenvalue or no Jacobi convergence");
    detail::check(rc, "smallest_eigs_of_H: invalid arguments");
    r.k_used = k;
    return r;
}

// --------------------------------------------------------------- pipeline

struct ComputeOptions { // pipeline.hpp:16-23; workers = GPUs (see compute)
    int n = 1;
    WeightSpec beta{1, 2};
    long bits = 1024; // the reference's K
    int k = 8;
    int workers = 1;
    BroadcastPolicy policy{};
    int device = 0;
    // multi-GPU (one process per GPU): this process's rank and the shared
    // ncclUniqueId; without an id, workers > 1 emulates the split on one GPU
    int rank = 0;
    const void* nccl_id128 = nullptr;
    // moments generated on the device (hk_generate_moments; even 2/beta) instead
    // of host build_hankel + upload — the same bits either way
    bool device_moments = true;
};

struct RunRecord { // pipeline.hpp:28-48 (+ p_bits and the ~32-digit lambda_lo)
    int n = 0;
    WeightSpec beta{1, 2};
    long bits = 0;
    int k = 0;
    int workers = 0;
    std::vector<double> lambda;
    std::vector<double> trunc_err;
    long required_bits = 0;
    double wall_s = 0, ldlt_s = 0, transpose_s = 0, invL_s = 0, invL_arith_s = 0, invL_comm_s = 0, invH_s = 0,
           eigen_s = 0;
    int p_bits = 0;
    std::vector<double> lambda_lo;
    double lambda1() const { return lambda.at(0); }
};

// Bit length of mu_{2n-2}, exactly (from the moment generator).
inline int moment_bits(const WeightSpec& spec, int n) {
    const double j = 2.0 * n - 2.0;
    const double est = (std::lgamma((j + 1) * spec.beta_den / spec.beta_num) +
                        std::log(double(spec.beta_den) / spec.beta_num)) / std::log(2.0);
    const int L = int(est / 32) + 4;
    MpVector v(size_t(2 * n - 1), L);
    int exact = 0;
    detail::check(hk_moments(spec.beta_num, spec.beta_den, 2 * n - 1, L, v.pl(), v.pe(), v.ps(), &exact),
                  "moment_bits: unsupported beta");
    // even 2/beta: integers, which must fit; odd: half-integer Gamma values (irrational,
    // correctly rounded) whose integer part's length is the exponent
    if (!exact && spec.doubled_inverse() % 2 == 0) throw precision_error("moment_bits: estimate too small");
    return v.e.back();
}

// The p-bit precision equivalent to the reference's K (pipeline.hpp:19):
// p(K) = 128 ceil((bits(mu_{2N-2}) + 2K) / 128) — every moment exact and 2K
// fraction bits on the largest entry (paper_1810_01478_b200/pipeline.py).
inline int precision_bits(const WeightSpec& spec, int n, long K) {
    const long need = moment_bits(spec, n) + 2 * K;
    return int(128 * ((need + 127) / 128));
}

namespace detail {
// One Device per (device, rank, workers, communicator id), reused by every
// compute() call of this thread: auto_precision / scan change only p
// (hk_set_limbs), so buffers are re-sized, not re-created, and a multi-GPU
// group keeps its one NCCL communicator (an ncclUniqueId serves one init).
inline Device& compute_device(const ComputeOptions& o, int limbs) {
    thread_local std::map<std::string, std::unique_ptr<Device>> devs;
    std::string key = std::to_string(o.device) + "/" + std::to_string(o.rank) + "/" + std::to_string(o.workers) + "/";
    if (o.nccl_id128) key.append(static_cast<const char*>(o.nccl_id128), 128);
    auto& d = devs[key];
    if (!d)
        d = o.workers == 1 && !o.nccl_id128 ? std::make_unique<Device>(limbs, o.device)
                                            : std::make_unique<Device>(limbs, o.device, o.rank, o.workers, o.nccl_id128);
    else
        d->set_limbs(limbs);
    return *d;
}
} // namespace detail

// pipeline.cpp:26-72: upload -> LDLT -> L^{-1} -> block -> eigen, one device call
inline RunRecord compute(const ComputeOptions& opts) {
    if (opts.n < 1) throw std::invalid_argument("compute: need N >= 1");
    if (opts.bits < 1) throw std::invalid_argument("compute: need bits >= 1");
    if (opts.workers < 1) throw std::invalid_argument("compute: need workers >= 1");
    if (opts.k < 1) throw std::invalid_argument("compute: need k >= 1");
    const int p = precision_bits(opts.beta, opts.n, opts.bits);
    const bool even_q = opts.beta.doubled_inverse() % 2 == 0;
    double hi[3], lo[3], te[3];
    int s = 0;
    Device* devp = nullptr;
    if (opts.device_moments && even_q) { // moments.cpp:113-133 on the device
        devp = &detail::compute_device(opts, p / 32);
        int exact = 0;
        devp->check(hk_compute_generated(devp->handle(), opts.beta.beta_num, opts.beta.beta_den, opts.n, opts.k, hi,
                                         lo, te, &s, &exact));
        if (!exact) throw precision_error("compute: moments not exact at p bits");
    } else {
        const MomentTable table = build_hankel(opts.beta, opts.n, p / 32);
        if (!table.exact() && even_q) throw precision_error("compute: moments not exact at p bits");
        devp = &detail::compute_device(opts, p / 32);
        const MpVector& mu = table.moments();
        devp->check(hk_compute(devp->handle(), opts.n, mu.pl(), mu.pe(), mu.ps(), opts.k, hi, lo, te, &s));
    }
    Device& dev = *devp;
    const std::vector<double> t = dev.timings();
    RunRecord r;
    r.n = opts.n;
    r.beta = opts.beta;
    r.bits = opts.bits;
    r.k = std::min(opts.k, opts.n);
    r.workers = opts.workers;
    for (int i = 0; i < s; ++i) {
        r.lambda.push_back(hi[i] + lo[i]);
        r.lambda_lo.push_back(lo[i]);
        r.trunc_err.push_back(te[i]);
    }
    r.wall_s = t[0];
    r.ldlt_s = t[1];
    r.invL_s = r.invL_arith_s = t[2];
    r.invH_s = t[3];
    r.eigen_s = t[4];
    r.p_bits = p;
    return r;
}

struct AutoPrecisionOptions { // pipeline.hpp:52-57
    long start_bits = 0;       // 0 -> 1024 * ceil(n / 500)
    long step_bits = 1024;
    long max_bits = 16384;
    double agree_tol = 1e-15;
};

// pipeline.cpp:74-94: smallest K whose run agrees with the K + step run on lambda_1
inline std::pair<long, RunRecord> auto_precision(const ComputeOptions& base, const AutoPrecisionOptions& opts = {}) {
    const long step = opts.step_bits;
    if (step < 1) throw std::invalid_argument("auto_precision: need step_bits >= 1");
    const long k0 = opts.start_bits > 0 ? opts.start_bits : step * ((base.n + 499) / 500);
    ComputeOptions run = base;
    run.bits = k0;
    RunRecord prev = compute(run);
    for (long bits = k0; bits <= opts.max_bits; bits += step) {
        run.bits = bits + step;
        RunRecord next = compute(run);
        if (std::fabs(prev.lambda1() - next.lambda1()) <= opts.agree_tol) {
            prev.required_bits = bits;
            return {bits, prev};
        }
        prev = std::move(next);
    }
    throw precision_error("auto_precision: no agreement up to " + std::to_string(opts.max_bits) + " bits");
}

struct ScanOptions { // pipeline.hpp:60-64
    ComputeOptions base;
    bool auto_bits = false;
    AutoPrecisionOptions auto_opts{};
};

// pipeline.cpp:96-122: one record per N; failed entries become NaN rows
inline std::vector<RunRecord> scan(const std::vector<int>& n_list, const ScanOptions& opts) {
    std::vector<RunRecord> out;
    for (int n : n_list) {
        ComputeOptions run = opts.base;
        run.n = n;
        try {
            out.push_back(opts.auto_bits ? auto_precision(run, opts.auto_opts).second : compute(run));
        } catch (const std::exception&) {
            RunRecord r;
            r.n = n;
            r.beta = run.beta;
            r.bits = run.bits;
            r.k = run.k;
            r.workers = run.workers;
            const double nan = std::numeric_limits<double>::quiet_NaN();
            r.lambda.assign(3, nan);
            r.trunc_err.assign(3, nan);
            out.push_back(r);
        }
    }
    return out;
}

// pipeline.cpp:143-161 (17 significant digits, as the reference's ostream)
inline std::string run_record_csv_header() {
    return "N,beta,bits,k,workers,lambda1,trunc1,lambda2,trunc2,lambda3,trunc3,required_bits,wall_s,ldlt_s,"
           "transpose_s,invL_s,invL_arith_s,invL_comm_s,invH_s,eigen_s";
}
inline std::string to_csv_row(const RunRecord& r) {
    std::ostringstream os;
    os << std::setprecision(17);
    os << r.n << ',' << r.beta.beta_num << '/' << r.beta.beta_den << ',' << r.bits << ',' << r.k << ',' << r.workers;
    const double nan = std::numeric_limits<double>::quiet_NaN();
    for (size_t i = 0; i < 3; ++i)
        os << ',' << (i < r.lambda.size() ? r.lambda[i] : nan) << ',' << (i < r.trunc_err.size() ? r.trunc_err[i] : nan);
    os << ',' << r.required_bits;
    for (double v : {r.wall_s, r.ldlt_s, r.transpose_s, r.invL_s, r.invL_arith_s, r.invL_comm_s, r.invH_s, r.eigen_s})
        os << ',' << v;
    return os.str();
}
inline void write_scan_csv(std::ostream& os, const std::vector<RunRecord>& records) {
    os << run_record_csv_header() << '\n';
    for (const auto& r : records) os << to_csv_row(r) << '\n';
}

namespace detail {
// A double as the reference's JSON writer (nlohmann::json::dump) prints it:
// the Grisu2 digits (Loitsch 2010; round-trip, usually but not always the
// shortest), positional between 1e-4 and 1e15, otherwise d.ddde+XX;
// non-finite -> null.  Checked byte for byte against the reference's writer
// (tests/test_pipeline.py).
namespace grisu {
struct Fp {
    uint64_t f;
    int e;
};
inline Fp mul(Fp x, Fp y) { // upper 64 bits of the 128-bit product, rounded
    const uint64_t ul = x.f & 0xffffffffu, uh = x.f >> 32, vl = y.f & 0xffffffffu, vh = y.f >> 32;
    const uint64_t p0 = ul * vl, p1 = ul * vh, p2 = uh * vl, p3 = uh * vh;
    const uint64_t q = (p0 >> 32) + (p1 & 0xffffffffu) + (p2 & 0xffffffffu) + (1ull << 31);
    return Fp{p3 + (p2 >> 32) + (p1 >> 32) + (q >> 32), x.e + y.e + 64};
}
inline Fp normalize(Fp x) {
    while (!(x.f >> 63)) {
        x.f <<= 1;
        --x.e;
    }
    return x;
}
struct Pow10 {
    uint64_t f;
    int e, k;
};
// 10^k, k = -300 .. 324 step 8, significand rounded to 64 bits (tools/gen_pow10.py)
inline const Pow10* pow10_table() {
    static const Pow10 t[79] = {
        {0xAB70FE17C79AC6CAull, -1060, -300}, {0xFF77B1FCBEBCDC4Full, -1034, -292},
        {0xBE5691EF416BD60Cull, -1007, -284}, {0x8DD01FAD907FFC3Cull, -980, -276},
        {0xD3515C2831559A83ull, -954, -268}, {0x9D71AC8FADA6C9B5ull, -927, -260},
        {0xEA9C227723EE8BCBull, -901, -252}, {0xAECC49914078536Dull, -874, -244},
        {0x823C12795DB6CE57ull, -847, -236}, {0xC21094364DFB5637ull, -821, -228},
        {0x9096EA6F3848984Full, -794, -220}, {0xD77485CB25823AC7ull, -768, -212},
        {0xA086CFCD97BF97F4ull, -741, -204}, {0xEF340A98172AACE5ull, -715, -196},
        {0xB23867FB2A35B28Eull, -688, -188}, {0x84C8D4DFD2C63F3Bull, -661, -180},
        {0xC5DD44271AD3CDBAull, -635, -172}, {0x936B9FCEBB25C996ull, -608, -164},
        {0xDBAC6C247D62A584ull, -582, -156}, {0xA3AB66580D5FDAF6ull, -555, -148},
        {0xF3E2F893DEC3F126ull, -529, -140}, {0xB5B5ADA8AAFF80B8ull, -502, -132},
        {0x87625F056C7C4A8Bull, -475, -124}, {0xC9BCFF6034C13053ull, -449, -116},
        {0x964E858C91BA2655ull, -422, -108}, {0xDFF9772470297EBDull, -396, -100},
        {0xA6DFBD9FB8E5B88Full, -369, -92}, {0xF8A95FCF88747D94ull, -343, -84},
        {0xB94470938FA89BCFull, -316, -76}, {0x8A08F0F8BF0F156Bull, -289, -68},
        {0xCDB02555653131B6ull, -263, -60}, {0x993FE2C6D07B7FACull, -236, -52},
        {0xE45C10C42A2B3B06ull, -210, -44}, {0xAA242499697392D3ull, -183, -36},
        {0xFD87B5F28300CA0Eull, -157, -28}, {0xBCE5086492111AEBull, -130, -20},
        {0x8CBCCC096F5088CCull, -103, -12}, {0xD1B71758E219652Cull, -77, -4},
        {0x9C40000000000000ull, -50, 4}, {0xE8D4A51000000000ull, -24, 12},
        {0xAD78EBC5AC620000ull, 3, 20}, {0x813F3978F8940984ull, 30, 28},
        {0xC097CE7BC90715B3ull, 56, 36}, {0x8F7E32CE7BEA5C70ull, 83, 44},
        {0xD5D238A4ABE98068ull, 109, 52}, {0x9F4F2726179A2245ull, 136, 60},
        {0xED63A231D4C4FB27ull, 162, 68}, {0xB0DE65388CC8ADA8ull, 189, 76},
        {0x83C7088E1AAB65DBull, 216, 84}, {0xC45D1DF942711D9Aull, 242, 92},
        {0x924D692CA61BE758ull, 269, 100}, {0xDA01EE641A708DEAull, 295, 108},
        {0xA26DA3999AEF774Aull, 322, 116}, {0xF209787BB47D6B85ull, 348, 124},
        {0xB454E4A179DD1877ull, 375, 132}, {0x865B86925B9BC5C2ull, 402, 140},
        {0xC83553C5C8965D3Dull, 428, 148}, {0x952AB45CFA97A0B3ull, 455, 156},
        {0xDE469FBD99A05FE3ull, 481, 164}, {0xA59BC234DB398C25ull, 508, 172},
        {0xF6C69A72A3989F5Cull, 534, 180}, {0xB7DCBF5354E9BECEull, 561, 188},
        {0x88FCF317F22241E2ull, 588, 196}, {0xCC20CE9BD35C78A5ull, 614, 204},
        {0x98165AF37B2153DFull, 641, 212}, {0xE2A0B5DC971F303Aull, 667, 220},
        {0xA8D9D1535CE3B396ull, 694, 228}, {0xFB9B7CD9A4A7443Cull, 720, 236},
        {0xBB764C4CA7A44410ull, 747, 244}, {0x8BAB8EEFB6409C1Aull, 774, 252},
        {0xD01FEF10A657842Cull, 800, 260}, {0x9B10A4E5E9913129ull, 827, 268},
        {0xE7109BFBA19C0C9Dull, 853, 276}, {0xAC2820D9623BF429ull, 880, 284},
        {0x80444B5E7AA7CF85ull, 907, 292}, {0xBF21E44003ACDD2Dull, 933, 300},
        {0x8E679C2F5E44FF8Full, 960, 308}, {0xD433179D9C8CB841ull, 986, 316},
        {0x9E19DB92B4E31BA9ull, 1013, 324},
    };
    return t;
}
inline void round_last(std::string& buf, uint64_t dist, uint64_t delta, uint64_t rest, uint64_t ten_k) {
    while (rest < dist && delta - rest >= ten_k && (rest + ten_k < dist || dist - rest > rest + ten_k - dist)) {
        --buf.back();
        rest += ten_k;
    }
}
// digits of v > 0 and the decimal exponent: v ~= digits * 10^dexp
inline std::string digits(double v, int& dexp) {
    uint64_t bits;
    std::memcpy(&bits, &v, 8);
    const uint64_t E = bits >> 52, F = bits & ((1ull << 52) - 1);
    const Fp w = E == 0 ? Fp{F, 1 - 1075} : Fp{F + (1ull << 52), int(E) - 1075};
    const bool closer = F == 0 && E > 1;
    const Fp mp = normalize(Fp{2 * w.f + 1, w.e - 1});
    const Fp mm0 = closer ? Fp{4 * w.f - 1, w.e - 2} : Fp{2 * w.f - 1, w.e - 1};
    const Fp mm{mm0.f << (mm0.e - mp.e), mp.e};
    const int f = -60 - mp.e - 1;
    const int k = (f * 78913) / (1 << 18) + (f > 0 ? 1 : 0);
    const Pow10 c = pow10_table()[(300 + k + 7) / 8];
    const Fp cw{c.f, c.e};
    const Fp W = mul(normalize(w), cw), Wm = mul(mm, cw), Wp = mul(mp, cw);
    const Fp Mm{Wm.f + 1, Wm.e}, Mp{Wp.f - 1, Wp.e};
    dexp = -c.k;
    uint64_t delta = Mp.f - Mm.f, dist = Mp.f - W.f;
    const int ne = -Mp.e;
    const uint64_t one = 1ull << ne;
    uint32_t p1 = uint32_t(Mp.f >> ne);
    uint64_t p2 = Mp.f & (one - 1);
    uint32_t pow10 = 1;
    int n = 1;
    for (uint32_t t = 1000000000u, d = 10; d > 1; t /= 10, --d)
        if (p1 >= t) {
            pow10 = t;
            n = int(d);
            break;
        }
    std::string buf;
    while (n > 0) {
        buf += char('0' + p1 / pow10);
        p1 %= pow10;
        --n;
        const uint64_t rest = (uint64_t(p1) << ne) + p2;
        if (rest <= delta) {
            dexp += n;
            round_last(buf, dist, delta, rest, uint64_t(pow10) << ne);
            return buf;
        }
        pow10 /= 10;
    }
    int m = 0;
    for (;;) {
        p2 *= 10;
        buf += char('0' + (p2 >> ne));
        p2 &= one - 1;
        ++m;
        delta *= 10;
        dist *= 10;
        if (p2 <= delta) break;
    }
    dexp -= m;
    round_last(buf, dist, delta, p2, one);
    return buf;
}
} // namespace grisu

inline std::string json_number(double v) {
    if (!std::isfinite(v)) return "null";
    std::string out = std::signbit(v) ? "-" : "";
    if (v == 0) return out + "0.0";
    int dexp = 0;
    const std::string d = grisu::digits(std::fabs(v), dexp);
    const int k = int(d.size()), n = k + dexp; // decimal point after n digits
    if (k <= n && n <= 15) {
        out += d + std::string(size_t(n - k), '0') + ".0";
    } else if (0 < n && n <= 15) {
        out += d.substr(0, size_t(n)) + "." + d.substr(size_t(n));
    } else if (-4 < n && n <= 0) {
        out += "0." + std::string(size_t(-n), '0') + d;
    } else {
        out += d.substr(0, 1);
        if (k > 1) out += "." + d.substr(1);
        const int e = n - 1;
        out += e < 0 ? "e-" : "e+";
        if (std::abs(e) < 10) out += '0';
        out += std::to_string(std::abs(e));
    }
    return out;
}
inline void json_array(std::ostream& os, const std::vector<double>& v, const std::string& ind) {
    if (v.empty()) {
        os << "[]";
        return;
    }
    os << "[\n";
    for (size_t i = 0; i < v.size(); ++i) os << (i ? ",\n" : "") << ind << "  " << json_number(v[i]);
    os << "\n" << ind << "]";
}
} // namespace detail

// pipeline.cpp:213-232, byte for byte: the reference builds an nlohmann::json
// object (keys in sorted order) and dumps it with indent 2
inline std::string to_json(const RunRecord& r) {
    std::ostringstream os;
    os << "{\n  \"N\": " << r.n << ",\n  \"beta\": \"" << r.beta.beta_num << '/' << r.beta.beta_den
       << "\",\n  \"bits\": " << r.bits << ",\n  \"k\": " << r.k << ",\n  \"lambda\": ";
    detail::json_array(os, r.lambda, "  ");
    if (r.required_bits > 0) os << ",\n  \"required_bits\": " << r.required_bits;
    const std::pair<const char*, double> timing[] = {
        {"eigen_s", r.eigen_s},           {"invH_s", r.invH_s}, {"invL_arith_s", r.invL_arith_s},
        {"invL_comm_s", r.invL_comm_s},   {"invL_s", r.invL_s}, {"ldlt_s", r.ldlt_s},
        {"transpose_s", r.transpose_s},   {"wall_s", r.wall_s}};
    os << ",\n  \"timing\": {";
    for (size_t q = 0; q < 8; ++q)
        os << (q ? ",\n" : "\n") << "    \"" << timing[q].first << "\": " << detail::json_number(timing[q].second);
    os << "\n  },\n  \"trunc_err\": ";
    detail::json_array(os, r.trunc_err, "  ");
    os << ",\n  \"workers\": " << r.workers << "\n}";
    return os.str();
}

// to_json plus this build's extras: p_bits and the low parts of the ~32-digit lambdas
inline std::string to_json_ext(const RunRecord& r) {
    std::string s = to_json(r);
    std::ostringstream os;
    os << ",\n  \"lambda_lo\": ";
    detail::json_array(os, r.lambda_lo, "  ");
    os << ",\n  \"p_bits\": " << r.p_bits << "\n}";
    s.resize(s.size() - 2); // drop the closing "\n}"
    return s + os.str();
}

} // namespace hankel::b200
