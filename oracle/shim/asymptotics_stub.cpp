// oracle/shim/asymptotics_stub.cpp — TEST INFRASTRUCTURE ONLY.
//
// proj/src/asymptotics.cpp needs Boost.Math (absent from the image, SURVEY.md
// §0.4) and is OUT OF SCOPE for the hot path.  pipeline.cpp's
// report() still references fit_leading_exponent, so the oracle build links
// these throwing stand-ins instead of the Boost-based originals
// (proj/include/hankel/asymptotics.hpp:23,50,56).
#include "hankel/asymptotics.hpp"

#include <stdexcept>

namespace hankel {

Prediction predict(int) {
    throw std::runtime_error("asymptotics not built in the oracle (Boost.Math absent; out of scope)");
}

FitResult fit_leading_exponent(const std::vector<FitPoint>&) {
    throw std::runtime_error("asymptotics not built in the oracle (Boost.Math absent; out of scope)");
}

namespace detail {
WlsFit weighted_linear_fit(const std::vector<double>&, const std::vector<double>&, const std::vector<double>&) {
    throw std::runtime_error("asymptotics not built in the oracle (Boost.Math absent; out of scope)");
}
} // namespace detail

} // namespace hankel
