// fsai.cpp -- NEXT-1: the paper's own preconditioner P = Z~ Z~^t, the banded FSAI of
// T = band(A, 1) (Eq. 19; reading R25), built on the host in the
// factored AINV form (unit-diagonal Zhat in owned columns, pivots D) so that the device path of
// AINV applies it unchanged.  Written from the paper, independently of oracle/fsai.c.
#include <cmath>

#include "internal.h"

namespace pcg {

// A's entry between consecutive unknowns a < b (grid indices), i.e. T's superdiagonal: the E face
// (same row, next column), the periodic W face of column 0 when the next unknown of the row is
// column ni-1, or the N face (next row, same column); 0 otherwise.  A_pq = -c (reading R1).
static double band_coupling(int32_t ni, int32_t periodic, const double* cE, const double* cN, int64_t a, int64_t b) {
    const int32_t ia = (int32_t)(a % ni), ja = (int32_t)(a / ni), ib = (int32_t)(b % ni), jbb = (int32_t)(b / ni);
    if (ja == jbb) {
        if (ib == ia + 1) return -cE[a];
        if (periodic && ia == 0 && ib == ni - 1) return -cE[b];
        return 0.0;
    }
    if (jbb == ja + 1 && ib == ia) return -cN[a];
    return 0.0;
}

void fsai_block(int32_t ni, int32_t nj, int32_t periodic, const double* cE, const double* cN, const uint8_t* mask,
                int32_t q, const std::function<double(int64_t)>& diag_of, AinvBlock& blk) {
    std::vector<int64_t> g;                           // unknowns in natural order (grid index)
    for (int64_t k = 0; k < (int64_t)ni * nj; ++k)
        if (mask[k]) g.push_back(k);
    const int64_t n = (int64_t)g.size();
    blk.row_lo = 0; blk.row_own = 0; blk.row_hi = nj;
    blk.fail_grid = -1;
    std::vector<double> u((size_t)n), rho((size_t)(n > 0 ? n : 1), 0.0);
    // T = U^t U: u_00 = sqrt(t_00), u_{k,k+1} = t_{k,k+1} / u_kk, u_{k+1,k+1} = sqrt(t_{k+1} - u_{k,k+1}^2)
    for (int64_t k = 0; k < n; ++k) {
        double rad = diag_of(g[(size_t)k]);
        double o = 0.0;
        if (k > 0) {
            o = band_coupling(ni, periodic, cE, cN, g[(size_t)k - 1], g[(size_t)k]);
            const double v = o / u[(size_t)k - 1];
            rad = rad - v * v;
        }
        if (!(rad > 0.0) || !std::isfinite(rad)) {
            blk.fail_grid = g[(size_t)k];
            return;
        }
        u[(size_t)k] = std::sqrt(rad);
        if (k > 0) rho[(size_t)k - 1] = -((o / u[(size_t)k - 1]) / u[(size_t)k - 1]);
    }
    // Eq. 19, unit form: zhat_{k-i,k} = zhat_{k-i+1,k} * rho_{k-i} for i = 1..q, until the chain breaks
    blk.colptr.assign(1, 0);
    blk.row_g.clear(); blk.zhat.clear(); blk.piv.clear(); blk.col_g.clear();
    std::vector<double> col((size_t)q + 1);
    for (int64_t k = 0; k < n; ++k) {
        int32_t m = 0;
        double prod = 1.0;
        for (int32_t i = 1; i <= q && k - i >= 0; ++i) {
            prod = prod * rho[(size_t)(k - i)];
            if (prod == 0.0) break;
            col[(size_t)m++] = prod;
        }
        for (int32_t e = m - 1; e >= 0; --e) {       // rows ascending
            blk.row_g.push_back(g[(size_t)(k - (e + 1))]);
            blk.zhat.push_back(col[(size_t)e]);
        }
        blk.row_g.push_back(g[(size_t)k]);
        blk.zhat.push_back(1.0);
        blk.colptr.push_back((int64_t)blk.row_g.size());
        blk.piv.push_back(u[(size_t)k] * u[(size_t)k]);
        blk.col_g.push_back(g[(size_t)k]);
    }
}

}  // namespace pcg
