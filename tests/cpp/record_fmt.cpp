// tests/cpp/record_fmt.cpp — the product's RunRecord writers (include/hankel_b200.hpp:
// to_csv_row, to_json) on records read from stdin, in the format of
// `oracle/_ref/ref_driver record`, so tests/test_pipeline.py can compare the
// bytes with the reference's own writers (pipeline.cpp:150-160, 213-232).
#include "hankel_b200.hpp"

#include <cstdlib>
#include <iostream>
#include <sstream>
#include <string>

namespace hb = hankel::b200;

int main() {
    std::string line;
    while (std::getline(std::cin, line)) {
        if (line.empty()) continue;
        std::istringstream is(line);
        auto dbl = [&]() {
            std::string t;
            is >> t;
            return std::strtod(t.c_str(), nullptr);
        };
        hb::RunRecord r;
        unsigned bn = 1, bd = 2;
        is >> r.n >> bn >> bd >> r.bits >> r.k >> r.workers >> r.required_bits;
        r.beta = hb::WeightSpec{bn, bd};
        size_t nl = 0, nt = 0;
        is >> nl;
        for (size_t i = 0; i < nl; ++i) r.lambda.push_back(dbl());
        is >> nt;
        for (size_t i = 0; i < nt; ++i) r.trunc_err.push_back(dbl());
        for (double* f : {&r.wall_s, &r.ldlt_s, &r.transpose_s, &r.invL_s, &r.invL_arith_s, &r.invL_comm_s, &r.invH_s,
                          &r.eigen_s})
            *f = dbl();
        std::cout << hb::to_csv_row(r) << "\n" << hb::to_json(r) << "\n@@" << std::endl;
    }
    return 0;
}
