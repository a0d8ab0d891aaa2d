// Device evaluation of the jump density nu, the trapezoid kernel nu(j h) w_j and the quartic
// window (fractional.py:65-86, :108-127, :285-296); shared by the symbol generator (build.cu)
// and the matrix-free evaluators (apply.cu).
#pragma once

#include "core.h"

namespace lh {

struct MeasureDev {
    int kind;
    double c, expo;           // power: c * |y|^expo, expo = -1 - 2s
    double C, G, M, Yexpo;    // CGMY: C e^{-rate|y|} |y|^Yexpo, Yexpo = -1 - Y
    const double *table;      // tabulated nu(j h), j = -Mw..Mw
    i64 Mw;
};

__device__ __forceinline__ double nu_eval(const MeasureDev &nu, i64 j, double y) {
    if (nu.kind == 0) return nu.c * pow(fabs(y), nu.expo);
    if (nu.kind == 1) {
        double rate = y < 0.0 ? nu.G : nu.M;
        double ay = fabs(y);
        return nu.C * exp(-rate * ay) * pow(ay, nu.Yexpo);
    }
    return nu.table[j + nu.Mw];
}

// kern_j = nu(j h) * w_j, w = h (h/2 at |j| = M), kern_0 = 0  (fractional.py:285-296)
__device__ __forceinline__ double kern_eval(const MeasureDev &nu, i64 j, double h, i64 M) {
    if (j == 0) return 0.0;
    double y = (double)j * h;
    double w = (j == M || j == -M) ? h / 2.0 : h;
    return nu_eval(nu, j, y) * w;
}

__device__ __forceinline__ double window_eval(double y, double r) {
    double t = fabs(y) / r;
    if (!(t < 1.0)) return 0.0;
    double p = pow(fmin(t, 1.0), 4.0);
    double q = 1.0 - p;
    return q * q;
}

inline MeasureDev measure_to_dev(const lh_measure &m, i64 Mw) {
    LH_REQUIRE(m.kind >= 0 && m.kind <= 2, LH_EINVAL, "unknown measure kind");
    LH_REQUIRE(m.kind != 2 || m.table_dev, LH_EINVAL, "tabulated measure needs a table");
    MeasureDev nu{};
    nu.kind = m.kind;
    nu.c = m.c;
    nu.expo = -1 - 2 * m.s;
    nu.C = m.C;
    nu.G = m.G;
    nu.M = m.M;
    nu.Yexpo = -1.0 - m.Y;
    nu.table = m.table_dev;
    nu.Mw = Mw;
    return nu;
}

}  // namespace lh
