// ssbh/geat.hpp — declarations of the reference's entropy-accumulation bounds
// (proj/include/ssbh/geat.hpp). Host-side security analysis, not part of the B200 data path:
// libssbh.so does not implement these; they are the reference's own proj/src/geat.cpp,
// compiled unmodified against these headers (tests/refsuite/Makefile).
#pragma once

#include <cstdint>

namespace ssbh {

/// Affine min-tradeoff function summary (rate h, Max, Min_Sigma, Var bound).
struct MinTradeoff {
    double h = 0;
    double max_f = 0;
    double min_f = 0;
    double var_f = 0;

    /// f -> s f: h, Max and Min scale by s, Var by s^2.
    MinTradeoff scaled(double s) const { return {h * s, max_f * s, min_f * s, var_f * s * s}; }
};

/// Inputs shared by the full and the simplified bound (alpha: full form only).
struct GeatInput {
    double n_rounds = 0;
    int d_x = 2;
    double eps_smooth = 0;
    double p_omega = 1.0;
    double alpha = 1.0;
};

double g_eps(double eps);
double v_of(const MinTradeoff& tradeoff, int d_x);
double geat_full_bound(const GeatInput& input, const MinTradeoff& tradeoff);

struct SimplifiedBound {
    double v0 = 0;
    double v1 = 0;
    double bound = 0;
};
SimplifiedBound geat_simplified_bound(const GeatInput& input, const MinTradeoff& tradeoff);

namespace geat_detail {
double xi();
double log2_kprime(double alpha, double nu);
double ln_pow2_plus_e2(double nu);
}  // namespace geat_detail

}  // namespace ssbh
