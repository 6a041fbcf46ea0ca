// ainv.cpp -- host AINV(A, tau) of libpcg, one row block at a time.
//
// The paper's "P_B1" ("A-orthogonalization method ... posing a (fixed) drop
// tolerance and by ignoring the elements below the fixed tolerance"), AINV cited at
// PAPER.md:26 and 224.  The exact variant -- Jacobi pre-scaling, left-looking
// A-orthogonalisation of e_1..e_n in natural order, drop-as-you-go on touched entries with a
// strict |z| < tau test, pivot threshold 1e-12 -- is DESIGN.md §3.2 (readings R11-R13).
// Compiled with -ffp-contract=off: every product and sum below is one IEEE operation, in
// the order written, so the result is reproducible bit for bit by any implementation that
// follows DESIGN.md §3.2 (the oracle's is independent code and is compared in tests).
//
// Block mode (reading R15): the index set is the ocean points of grid rows
// [row_lo, row_hi); the principal submatrix of A on that set is orthogonalised and only
// the columns of rows >= row_own are returned ("AINV computed per partition").
#include <cmath>
#include <cstring>
#include <algorithm>
#include <functional>
#include <queue>
#include <vector>

#include "internal.h"

namespace pcg {

namespace {

struct BlockMatrix {
    int32_t n = 0;
    std::vector<int32_t> rp, ci;      // CSR of the scaled matrix A^, columns ascending
    std::vector<double> a;
    std::vector<int64_t> grid;        // local unknown -> grid index
    std::vector<double> diag;         // A_pp
};

// Faces of (i,j): E, W, N, S with existence and coupling.
inline void faces(int32_t ni, int32_t nj, int32_t periodic, const double* cE, const double* cN,
                  int32_t i, int32_t j, bool ex[4], int64_t nb[4], double c[4]) {
    const int64_t row = (int64_t)j * ni;
    ex[0] = (i + 1 < ni) || periodic;  nb[0] = row + (i + 1) % ni;      c[0] = ex[0] ? cE[row + i] : 0.0;
    ex[1] = (i >= 1) || periodic;      nb[1] = row + (i - 1 + ni) % ni; c[1] = ex[1] ? cE[row + (i - 1 + ni) % ni] : 0.0;
    ex[2] = (j + 1 < nj);              nb[2] = row + ni + i;            c[2] = ex[2] ? cN[row + i] : 0.0;
    ex[3] = (j >= 1);                  nb[3] = row - ni + i;            c[3] = ex[3] ? cN[row - ni + i] : 0.0;
}

}  // namespace

void ainv_block(int32_t ni, int32_t nj, int32_t periodic, const double* cE, const double* cN,
                const double* sigma, const uint8_t* mask, double tau, int32_t fill, AinvBlock& blk) {
    const int32_t r0 = blk.row_lo, r1 = blk.row_hi;
    BlockMatrix M;
    // local numbering of the ocean points of rows [r0, r1), natural order
    std::vector<int32_t> loc((size_t)(r1 - r0) * ni, -1);
    for (int32_t j = r0; j < r1; ++j)
        for (int32_t i = 0; i < ni; ++i) {
            int64_t g = (int64_t)j * ni + i;
            if (mask[g]) { loc[(size_t)(j - r0) * ni + i] = M.n++; M.grid.push_back(g); }
        }
    const int32_t n = M.n;
    M.rp.assign(n + 1, 0);
    M.diag.resize(n);
    std::vector<double> sc(n);
    // diagonal A_pp = ((c_E + c_W) + c_N) + c_S (+ sigma) over all faces, then s = 1/sqrt(A_pp)
    for (int32_t p = 0; p < n; ++p) {
        int64_t g = M.grid[p];
        int32_t i = (int32_t)(g % ni), j = (int32_t)(g / ni);
        bool ex[4]; int64_t nb[4]; double c[4];
        faces(ni, nj, periodic, cE, cN, i, j, ex, nb, c);
        double d = ((c[0] + c[1]) + c[2]) + c[3];
        if (sigma) d = d + sigma[g];
        M.diag[p] = d;
        sc[p] = 1.0 / std::sqrt(d);
    }
    // CSR of A^ restricted to the block: a^_pq = A_pq * (s_p * s_q)
    M.ci.reserve((size_t)5 * n);
    M.a.reserve((size_t)5 * n);
    for (int32_t p = 0; p < n; ++p) {
        int64_t g = M.grid[p];
        int32_t i = (int32_t)(g % ni), j = (int32_t)(g / ni);
        bool ex[4]; int64_t nb[4]; double c[4];
        faces(ni, nj, periodic, cE, cN, i, j, ex, nb, c);
        int32_t cols[5]; double vals[5]; int m = 0;
        cols[m] = p; vals[m] = M.diag[p] * (sc[p] * sc[p]); ++m;
        for (int f = 0; f < 4; ++f) {
            if (!ex[f] || !(c[f] > 0.0) || !mask[nb[f]]) continue;
            int32_t jn = (int32_t)(nb[f] / ni);
            if (jn < r0 || jn >= r1) continue;          // outside the block's index set
            int32_t q = loc[(size_t)(jn - r0) * ni + (int32_t)(nb[f] % ni)];
            cols[m] = q; vals[m] = (-c[f]) * (sc[p] * sc[q]); ++m;
        }
        for (int x = 1; x < m; ++x)
            for (int y = x; y > 0 && cols[y - 1] > cols[y]; --y) { std::swap(cols[y], cols[y - 1]); std::swap(vals[y], vals[y - 1]); }
        for (int x = 0; x < m; ++x) { M.ci.push_back(cols[x]); M.a.push_back(vals[x]); }
        M.rp[p + 1] = (int32_t)M.ci.size();
    }

    // Zhat columns (CSC), pivots
    std::vector<int64_t> zp(1, 0);
    zp.reserve(n + 1);
    std::vector<int32_t> zr;
    std::vector<double> zv;
    zr.reserve((size_t)6 * n); zv.reserve((size_t)6 * n);
    std::vector<double> piv(n);

    std::vector<double> w(n, 0.0);
    std::vector<uint8_t> live(n, 0);        // entry present in the current column
    std::vector<int32_t> listed(n, -1);     // stamp: k recorded in `members` for column j
    std::vector<int32_t> queued(n, -1);     // stamp: k queued as a candidate for column j
    std::vector<int32_t> members, touched;
    std::priority_queue<int32_t, std::vector<int32_t>, std::greater<int32_t>> cand;

    int64_t fail = -1;
    for (int32_t j = 0; j < n; ++j) {
        members.clear();
        members.push_back(j); listed[j] = j; live[j] = 1; w[j] = 1.0;
        for (int32_t e = M.rp[j]; e < M.rp[j + 1]; ++e) {
            int32_t i = M.ci[e];
            if (i < j && queued[i] != j) { queued[i] = j; cand.push(i); }
        }
        while (!cand.empty()) {
            const int32_t i = cand.top(); cand.pop();
            // pi = a^_i . z over row i of A^ (ascending columns, present entries)
            double pi = 0.0;
            for (int32_t e = M.rp[i]; e < M.rp[i + 1]; ++e) {
                int32_t k = M.ci[e];
                if (live[k]) pi = pi + M.a[e] * w[k];
            }
            if (pi == 0.0) continue;
            const double coef = pi / piv[i];
            touched.clear();
            for (int64_t e = zp[i]; e < zp[i + 1]; ++e) {
                const int32_t k = zr[e];
                if (!live[k]) {
                    live[k] = 1; w[k] = 0.0;
                    if (listed[k] != j) { listed[k] = j; members.push_back(k); }
                    for (int32_t e2 = M.rp[k]; e2 < M.rp[k + 1]; ++e2) {
                        int32_t i2 = M.ci[e2];
                        if (i2 > i && i2 < j && queued[i2] != j) { queued[i2] = j; cand.push(i2); }
                    }
                }
                w[k] = w[k] - coef * zv[e];
                touched.push_back(k);
            }
            for (int32_t k : touched)
                if (k != j && std::fabs(w[k]) < tau) { live[k] = 0; w[k] = 0.0; }
            if (fill > 0) {
                // P_B2 (reading R26): keep the diagonal and the fill-1 largest |z|, ties to the
                // smaller index
                touched.clear();
                for (int32_t k : members)
                    if (k != j && live[k]) touched.push_back(k);
                if ((int64_t)touched.size() > (int64_t)fill - 1) {
                    std::sort(touched.begin(), touched.end(), [&](int32_t a, int32_t b) {
                        const double fa = std::fabs(w[a]), fb = std::fabs(w[b]);
                        return fa > fb || (fa == fb && a < b);
                    });
                    for (size_t t = (size_t)fill - 1; t < touched.size(); ++t) { live[touched[t]] = 0; w[touched[t]] = 0.0; }
                }
            }
        }
        double pj = 0.0;
        for (int32_t e = M.rp[j]; e < M.rp[j + 1]; ++e) {
            int32_t k = M.ci[e];
            if (live[k]) pj = pj + M.a[e] * w[k];
        }
        piv[j] = pj;
        if (!(pj > kPivotMin) || !std::isfinite(pj)) { fail = j; }
        std::sort(members.begin(), members.end());
        for (int32_t k : members) {
            if (live[k]) { zr.push_back(k); zv.push_back(w[k]); }
            live[k] = 0; w[k] = 0.0;
        }
        zp.push_back((int64_t)zr.size());
        if (fail >= 0) break;
    }
    blk.fail_grid = fail >= 0 ? M.grid[fail] : -1;
    if (fail >= 0) return;

    // owned columns: local unknowns whose grid row >= row_own
    int32_t first_owned = n;
    for (int32_t p = 0; p < n; ++p)
        if (M.grid[p] / ni >= blk.row_own) { first_owned = p; break; }
    blk.colptr.assign(1, 0);
    blk.row_g.clear(); blk.zhat.clear(); blk.piv.clear(); blk.col_g.clear();
    for (int32_t j = first_owned; j < n; ++j) {
        for (int64_t e = zp[j]; e < zp[j + 1]; ++e) { blk.row_g.push_back(M.grid[zr[e]]); blk.zhat.push_back(zv[e]); }
        blk.colptr.push_back((int64_t)blk.row_g.size());
        blk.piv.push_back(piv[j]);
        blk.col_g.push_back(M.grid[j]);
    }
}

}  // namespace pcg
