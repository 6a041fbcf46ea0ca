// plan.cpp -- host half of pcg_setup: validation, row partition, anchor check, device-layout
// coefficient arrays, AINV per block, SELL-32 packing of Z and Z^T.
#include <algorithm>
#include <cstdlib>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <thread>

#include "internal.h"

namespace pcg {

Status partition_rows(int32_t ni, int32_t nj, const uint8_t* mask, int32_t parts, int32_t* rb) {
    if (ni < 1 || nj < 1 || parts < 1 || parts > nj || !mask || !rb)
        return Status::err(PCG_ERR_ARG, "pcg_partition: need 1 <= parts <= nj and non-NULL mask/row_begin");
    std::vector<int64_t> cum(nj + 1, 0);
    for (int32_t j = 0; j < nj; ++j) {
        int64_t c = 0;
        for (int32_t i = 0; i < ni; ++i) c += mask[(int64_t)j * ni + i] ? 1 : 0;
        cum[j + 1] = cum[j] + c;
    }
    const int64_t N = cum[nj];
    rb[0] = 0;
    for (int32_t p = 1; p < parts; ++p) {
        // smallest j with cum[j] * parts >= p * N (cum is non-decreasing)
        int32_t j = (int32_t)(std::lower_bound(cum.begin(), cum.end(), 0, [&](int64_t v, int) {
                        return v * parts < (int64_t)p * N; }) - cum.begin());
        j = std::max(j, rb[p - 1] + 1);
        j = std::min(j, nj - (parts - p));
        rb[p] = j;
    }
    rb[parts] = nj;
    return Status::ok();
}

namespace {

// Anchor check (reading R22): every 4-connected ocean component (faces with c > 0,
// E-W wrap included) must own a positive face to a land cell or a point with sigma > 0.
Status anchor_check(int32_t ni, int32_t nj, int32_t periodic, const double* cE, const double* cN,
                    const double* sigma, const uint8_t* mask) {
    const int64_t ng = (int64_t)ni * nj;
    std::vector<int32_t> comp(ng, -1);
    std::vector<int64_t> stack;
    int64_t unknown = 0;                    // natural-order index of the component root
    std::vector<int64_t> unk_of(ng, -1);
    for (int64_t g = 0; g < ng; ++g) if (mask[g]) unk_of[g] = unknown++;
    for (int64_t root = 0; root < ng; ++root) {
        if (!mask[root] || comp[root] >= 0) continue;
        bool anchored = false;
        stack.clear(); stack.push_back(root); comp[root] = 1;
        while (!stack.empty()) {
            int64_t g = stack.back(); stack.pop_back();
            int32_t i = (int32_t)(g % ni), j = (int32_t)(g / ni);
            if (sigma && sigma[g] > 0.0) anchored = true;
            const int64_t row = (int64_t)j * ni;
            struct { bool ex; int64_t nb; double c; } f[4] = {
                {(i + 1 < ni) || periodic != 0, row + (i + 1) % ni, cE[row + i]},
                {(i >= 1) || periodic != 0, row + (i - 1 + ni) % ni, cE[row + (i - 1 + ni) % ni]},
                {j + 1 < nj, row + ni + i, j + 1 < nj ? cN[row + i] : 0.0},
                {j >= 1, row - ni + i, j >= 1 ? cN[row - ni + i] : 0.0}};
            for (auto& x : f) {
                if (!x.ex || !(x.c > 0.0)) continue;
                if (!mask[x.nb]) { anchored = true; continue; }
                if (comp[x.nb] < 0) { comp[x.nb] = 1; stack.push_back(x.nb); }
            }
        }
        if (!anchored) {
            char buf[256];
            snprintf(buf, sizeof buf,
                     "A is singular: the ocean basin containing grid point (i=%d, j=%d) has no positive "
                     "face to land and sigma = 0 (anchor check, DESIGN.md R22)",
                     (int)(root % ni), (int)(root / ni));
            return Status::err(PCG_ERR_NOT_SPD, buf, unk_of[root]);
        }
    }
    return Status::ok();
}

int64_t global_unknown(const uint8_t* mask, int32_t ni, int64_t g) {
    (void)ni;
    int64_t c = 0;
    for (int64_t k = 0; k < g; ++k) c += mask[k] ? 1 : 0;
    return c;
}

// parallel for over [0, n) in T contiguous ranges (independent iterations only)
void pfor(int T, int64_t n, const std::function<void(int64_t, int64_t)>& f, int64_t serial_below = 100000) {
    if (n < serial_below) T = 1;
    T = std::max(1, T);
    std::vector<std::thread> pool;
    for (int t = 1; t < T; ++t) pool.emplace_back(f, n * t / T, n * (t + 1) / T);
    f(0, n / T);
    for (auto& th : pool) th.join();
}

// exclusive prefix sum out[0..n] of cnt(i), i in [0, n), in T contiguous ranges (two passes)
template <class V, class F>
void pscan(int T, int64_t n, V& out, F cnt) {
    out.resize((size_t)n + 1);                           // every slot is written below
    if (n < 100000) T = 1;
    T = std::max(1, T);
    std::vector<int64_t> part((size_t)T + 1, 0);
    auto run = [&](auto&& body) {                        // body(t, [a, b)) on T threads
        std::vector<std::thread> pool;
        for (int t = 1; t < T; ++t) pool.emplace_back([&, t] { body(t, n * t / T, n * (t + 1) / T); });
        body(0, 0, n / T);
        for (auto& th : pool) th.join();
    };
    run([&](int t, int64_t a, int64_t b) {
        int64_t sum = 0;
        for (int64_t i = a; i < b; ++i) sum += cnt(i);
        part[(size_t)t + 1] = sum;
    });
    for (int t = 0; t < T; ++t) part[(size_t)t + 1] += part[(size_t)t];
    run([&](int t, int64_t a, int64_t b) {
        int64_t acc = part[(size_t)t];
        for (int64_t i = a; i < b; ++i) { out[(size_t)i] = acc; acc += cnt(i); }
    });
    out[(size_t)n] = part[(size_t)T];
}

// Ocean components each need an anchor (a positive face to land, or sigma > 0; R22):
// the parallel check -- a lock-free union-find over the ocean-ocean faces with positive
// coupling, linking the larger root to the smaller, so each root is its component's smallest
// grid index (the component the sequential walk below would report first) -- then every cell
// with an anchor marks its root.  true = every component anchored.
bool anchors_ok_parallel(int T, int32_t ni, int32_t nj, int32_t periodic, const double* cE, const double* cN,
                         const double* sigma, const uint8_t* mask) {
    const int64_t ng = (int64_t)ni * nj;
    std::unique_ptr<std::atomic<int64_t>[]> par(new std::atomic<int64_t>[(size_t)ng]);
    pfor(T, ng, [&](int64_t a, int64_t b) { for (int64_t g = a; g < b; ++g) par[g].store(g, std::memory_order_relaxed); });
    auto find = [&](int64_t x) {
        for (;;) {
            int64_t p = par[x].load(std::memory_order_relaxed);
            if (p == x) return x;
            const int64_t gp = par[p].load(std::memory_order_relaxed);
            if (gp != p) par[x].compare_exchange_weak(p, gp, std::memory_order_relaxed);   // path halving
            x = gp;
        }
    };
    auto unite = [&](int64_t a, int64_t b) {
        for (;;) {
            a = find(a); b = find(b);
            if (a == b) return;
            if (a < b) std::swap(a, b);                  // link the larger root under the smaller
            int64_t expect = a;
            if (par[a].compare_exchange_strong(expect, b, std::memory_order_acq_rel)) return;
        }
    };
    pfor(T, ng, [&](int64_t a, int64_t b) {
        for (int64_t g = a; g < b; ++g) {
            if (!mask[g]) continue;
            const int32_t i = (int32_t)(g % ni), j = (int32_t)(g / ni);
            const int64_t row = (int64_t)j * ni;
            if (((i + 1 < ni) || periodic) && cE[row + i] > 0.0 && mask[row + (i + 1) % ni]) unite(g, row + (i + 1) % ni);
            if (j + 1 < nj && cN[row + i] > 0.0 && mask[row + ni + i]) unite(g, row + ni + i);
        }
    });
    std::unique_ptr<std::atomic<uint8_t>[]> anch(new std::atomic<uint8_t>[(size_t)ng]);
    pfor(T, ng, [&](int64_t a, int64_t b) { for (int64_t g = a; g < b; ++g) anch[g].store(0, std::memory_order_relaxed); });
    pfor(T, ng, [&](int64_t a, int64_t b) {
        for (int64_t g = a; g < b; ++g) {
            if (!mask[g]) continue;
            const int32_t i = (int32_t)(g % ni), j = (int32_t)(g / ni);
            const int64_t row = (int64_t)j * ni;
            bool an = sigma && sigma[g] > 0.0;
            const bool ex[4] = {(i + 1 < ni) || periodic != 0, (i >= 1) || periodic != 0, j + 1 < nj, j >= 1};
            const int64_t nb[4] = {row + (i + 1) % ni, row + (i - 1 + ni) % ni, row + ni + i, row - ni + i};
            const double cf[4] = {cE[row + i], cE[row + (i - 1 + ni) % ni], j + 1 < nj ? cN[row + i] : 0.0,
                                  j >= 1 ? cN[row - ni + i] : 0.0};
            for (int f = 0; f < 4 && !an; ++f) an = ex[f] && cf[f] > 0.0 && !mask[nb[f]];
            if (an) anch[find(g)].store(1, std::memory_order_relaxed);
        }
    });
    std::atomic<bool> ok(true);
    pfor(T, ng, [&](int64_t a, int64_t b) {
        for (int64_t g = a; g < b && ok.load(std::memory_order_relaxed); ++g)
            if (mask[g] && par[g].load(std::memory_order_relaxed) == g && !anch[g].load(std::memory_order_relaxed)) ok = false;
    });
    return ok.load();
}

// ELL(kEll) + SELL-32 overflow (internal.h Ell) over nel owned elements, filled in place: the
// first kEll entries of every row in its fixed slots, the rest of the slice's rows as SELL-32 (L =
// the slice's longest overflow).  ell_shape sizes the arrays from the row lengths and writes the
// padding everywhere (value 0 at the row's own array index; also the pages' first touch, in
// parallel); ell_slot then gives the slot of a row's k-th entry, so the rows are written straight
// from the AINV's columns (Z^T) or from the transposition (Z), with no intermediate copy.
template <class F>
void ell_shape(Ell& E, int64_t nel, int64_t hoff, int T, F len) {
    E.n = nel;
    E.val.resize((size_t)kEll * nel);
    E.col.resize((size_t)kEll * nel);
    E.col16.resize((size_t)kEll * nel);
    const int64_t nsl = nel / kSlice;
    pscan(T, nsl, E.ovf.off, [&](int64_t s) {
        int64_t L = 0;
        for (int l = 0; l < kSlice; ++l) L = std::max(L, len(s * kSlice + l) - kEll);
        return L * kSlice;
    });
    E.ovf.val.resize(E.ovf.off[nsl]);
    E.ovf.col.resize(E.ovf.off[nsl]);
    pfor(T, nsl, [&](int64_t s0, int64_t s1) {
        for (int64_t s = s0; s < s1; ++s) {
            for (int64_t e = s * kSlice; e < (s + 1) * kSlice; ++e)
                for (int m = 0; m < kEll; ++m) {
                    E.col[(size_t)e * kEll + m] = (int32_t)(e + hoff);
                    E.val[(size_t)e * kEll + m] = 0.0;
                    E.col16[(size_t)e * kEll + m] = 0;
                }
            for (int64_t o = E.ovf.off[s]; o < E.ovf.off[s + 1]; ++o) {
                E.ovf.col[(size_t)o] = (int32_t)(s * kSlice + (o - E.ovf.off[s]) % kSlice + hoff);
                E.ovf.val[(size_t)o] = 0.0;
            }
        }
    });
}
// (col16: the ELL slot's column as an int16 offset from the element's own array index -- the
// device form; when one does not fit, c16_fits is cleared and the int32 columns are used)
inline void ell_put(Ell& E, int64_t e, int64_t k, int32_t col, double val, int64_t hoff, std::atomic<bool>& c16_fits) {
    if (k < kEll) {
        E.col[(size_t)(e * kEll + k)] = col;
        E.val[(size_t)(e * kEll + k)] = val;
        const int64_t off = (int64_t)col - (e + hoff);
        if (off < -32768 || off > 32767) c16_fits.store(false, std::memory_order_relaxed);
        else E.col16[(size_t)(e * kEll + k)] = (int16_t)off;
    } else {
        const int64_t s = e / kSlice, o = E.ovf.off[(size_t)s] + (k - kEll) * kSlice + (e - s * kSlice);
        E.ovf.col[(size_t)o] = col;
        E.ovf.val[(size_t)o] = val;
    }
}

}  // namespace

Status build_plan(const pcg_coeffs* c, const pcg_grid* g, const pcg_opts* o, Plan& P) {
    auto t0 = std::chrono::steady_clock::now();
    const bool verbose = getenv("PCG_VERBOSE") != nullptr;
    auto tprev = t0;
    auto stage = [&](const char* what) {
        if (!verbose) return;
        const auto now = std::chrono::steady_clock::now();
        fprintf(stderr, "libpcg: setup %-28s %.3f s\n", what, std::chrono::duration<double>(now - tprev).count());
        tprev = now;
    };
    if (!c || !g || !o) return Status::err(PCG_ERR_ARG, "pcg_setup: NULL coeffs/grid/opts");
    if (!c->cE || !c->cN || !c->mask) return Status::err(PCG_ERR_ARG, "pcg_setup: coeffs.cE, cN and mask are required");
    if (g->ni < 3 || g->nj < 3) return Status::err(PCG_ERR_ARG, "pcg_setup: need ni >= 3 and nj >= 3");
    if (g->nranks < 1 || g->rank < 0 || g->rank >= g->nranks)
        return Status::err(PCG_ERR_ARG, "pcg_setup: need 0 <= rank < nranks");
    if (g->j_begin < 0 || g->j_end > g->nj || g->j_begin >= g->j_end)
        return Status::err(PCG_ERR_ARG, "pcg_setup: need 0 <= j_begin < j_end <= nj");
    if (g->nranks == 1 && (g->j_begin != 0 || g->j_end != g->nj))
        return Status::err(PCG_ERR_ARG, "pcg_setup: a single rank must own rows [0, nj)");
    if (o->precond < PCG_PRECOND_AINV || o->precond > PCG_PRECOND_FSAI)
        return Status::err(PCG_ERR_ARG, "pcg_setup: unknown preconditioner");
    if (o->ainv_fill < 0) return Status::err(PCG_ERR_ARG, "pcg_setup: ainv_fill < 0");
    if (o->precond == PCG_PRECOND_FSAI && (o->fsai_q < 0 || g->nranks > 1 || o->ainv_parts > 1))
        return Status::err(PCG_ERR_ARG, "pcg_setup: FSAI needs fsai_q >= 0 and one rank (no ainv_parts)");
    if (o->precond == PCG_PRECOND_AINV && !(o->drop_tol >= 0.0))
        return Status::err(PCG_ERR_ARG, "pcg_setup: drop_tol must be >= 0 (inf allowed, NaN not)");
    if (o->ainv_parts < 0 || o->ainv_halo < 0) return Status::err(PCG_ERR_ARG, "pcg_setup: ainv_parts/ainv_halo < 0");
    if (o->ainv_parts > 1 && g->nranks > 1)
        return Status::err(PCG_ERR_ARG, "pcg_setup: ainv_parts emulates ranks on one GPU; use nranks instead");
    const int32_t ni = g->ni, nj = g->nj;
    const int64_t ng = (int64_t)ni * nj;
    const int nthr = std::min(64, o->setup_threads > 0 ? o->setup_threads : (int)std::max(1u, std::thread::hardware_concurrency()));
    std::atomic<bool> bad_input(false);
    pfor(nthr, ng, [&](int64_t a, int64_t b) {
        for (int64_t k = a; k < b; ++k)
            if (!(c->cE[k] >= 0.0) || !std::isfinite(c->cE[k]) || !(c->cN[k] >= 0.0) || !std::isfinite(c->cN[k]) ||
                (c->sigma && (!(c->sigma[k] >= 0.0) || !std::isfinite(c->sigma[k]))) || c->mask[k] > 1) {
                bad_input = true;
                return;
            }
    });
    for (int64_t k = 0; k < (bad_input ? ng : 0); ++k) {     // the first offending point, in order
        if (!(c->cE[k] >= 0.0) || !std::isfinite(c->cE[k]) || !(c->cN[k] >= 0.0) || !std::isfinite(c->cN[k])) {
            char buf[160];
            snprintf(buf, sizeof buf, "pcg_setup: coefficient at (i=%d, j=%d) is negative or not finite",
                     (int)(k % ni), (int)(k / ni));
            return Status::err(PCG_ERR_ARG, buf);
        }
        if (c->sigma && (!(c->sigma[k] >= 0.0) || !std::isfinite(c->sigma[k])))
            return Status::err(PCG_ERR_ARG, "pcg_setup: sigma must be finite and >= 0");
        if (c->mask[k] > 1) return Status::err(PCG_ERR_ARG, "pcg_setup: mask values must be 0 or 1");
    }
    P.ni = ni; P.nj = nj; P.periodic = g->periodic_ew ? 1 : 0;
    P.jb = g->j_begin; P.je = g->j_end; P.rank = g->rank; P.nranks = g->nranks;
    P.nloc = P.je - P.jb;
    P.pitch = (ni + kSlice - 1) / kSlice * kSlice;
    P.halo = 1;
    if (const char* e = getenv("PCG_HALO_ROWS")) P.halo = std::max(1, atoi(e));   // layout test hook
    P.precond = o->precond;
    P.fsai_q = o->fsai_q;
    P.ainv_fill = o->ainv_fill;
    P.tau = o->drop_tol;
    P.flags = o->flags;
    P.has_sigma = c->sigma != nullptr;
    const int32_t pitch = P.pitch, nloc = P.nloc;

    // diagonal of every ocean point must be positive, then the structural anchor check
    auto diag_of = [&](int64_t gi) {
        int32_t i = (int32_t)(gi % ni), j = (int32_t)(gi / ni);
        const int64_t row = (int64_t)j * ni;
        double e = ((i + 1 < ni) || P.periodic) ? c->cE[row + i] : 0.0;
        double w = ((i >= 1) || P.periodic) ? c->cE[row + (i - 1 + ni) % ni] : 0.0;
        double n = (j + 1 < nj) ? c->cN[row + i] : 0.0;
        double s = (j >= 1) ? c->cN[row - ni + i] : 0.0;
        double d = ((e + w) + n) + s;
        if (c->sigma) d = d + c->sigma[gi];
        return d;
    };
    std::atomic<bool> bad_diag(false);
    pfor(nthr, ng, [&](int64_t a, int64_t b) {
        for (int64_t k = a; k < b; ++k)
            if (c->mask[k] && !(diag_of(k) > 0.0)) { bad_diag = true; return; }
    });
    for (int64_t k = 0; k < (bad_diag ? ng : 0); ++k)
        if (c->mask[k] && !(diag_of(k) > 0.0)) {
            char buf[160];
            snprintf(buf, sizeof buf, "pcg_setup: ocean point (i=%d, j=%d) has A_pp <= 0 (isolated, all faces 0)",
                     (int)(k % ni), (int)(k / ni));
            return Status::err(PCG_ERR_NOT_SPD, buf, global_unknown(c->mask, ni, k));
        }
    stage("validation + diagonal");
    // the parallel union-find decides; the sequential walk names the first unanchored basin
    if (!anchors_ok_parallel(nthr, ni, nj, P.periodic, c->cE, c->cN, c->sigma, c->mask))
        if (Status s = anchor_check(ni, nj, P.periodic, c->cE, c->cN, c->sigma, c->mask); !s) return s;
    stage("anchor check");
    if (ni > 65534) return Status::err(PCG_ERR_ARG, "pcg_setup: ni > 65534 not supported (int16 column offsets)");

    // device-layout coefficient arrays: absent faces -> 0, land flagged by the
    // sign bit of cN (cN >= 0 always, so -0.0 / -c mark a land cell).
    auto build_coeff_arrays = [&]() {
    const int64_t nel = P.elements();
    P.cE.resize(nel); P.cN.resize(nel); P.diag.resize(nel); P.piv.resize(nel);
    if (P.has_sigma) P.sigma.resize(nel);
    pfor(nthr, nel, [&](int64_t a, int64_t b) {              // defaults, first touch in parallel
        for (int64_t e = a; e < b; ++e) {
            P.cE[e] = 0.0; P.cN[e] = 0.0; P.diag[e] = 1.0; P.piv[e] = 1.0;
            if (P.has_sigma) P.sigma[e] = 0.0;
        }
    });
    const int32_t H = P.halo;
    pfor(nthr, (int64_t)(nloc + 2 * H), [&](int64_t r0, int64_t r1) {
    for (int32_t lr = (int32_t)r0; lr < (int32_t)r1; ++lr) {
        const int32_t j = P.jb + lr - H;
        if (j < 0 || j >= nj) continue;
        const int64_t row = (int64_t)j * ni;
        for (int32_t i = 0; i < ni; ++i) {
            const int64_t a = (int64_t)lr * pitch + i;
            const bool owned = lr >= H && lr < H + nloc;
            double ce = ((i + 1 < ni) || P.periodic) ? c->cE[row + i] : 0.0;
            double cn = (j + 1 < nj) ? c->cN[row + i] : 0.0;
            if (owned) {
                P.cE[a] = ce;
                P.cN[a] = c->mask[row + i] ? cn : -cn;
                if (std::fabs(cn) == 0.0 && !c->mask[row + i]) P.cN[a] = -0.0;
                if (P.has_sigma) P.sigma[a] = c->mask[row + i] ? c->sigma[row + i] : 0.0;
                if (c->mask[row + i]) P.diag[a] = diag_of(row + i);
            } else if (lr == H - 1) {
                P.cN[a] = cn;                   // southern halo: S face of row j_begin
            }
        }
    }
    }, 64);
    };

    // owned ocean unknowns, first global index
    {
        std::atomic<int64_t> fg(0), no(0);
        pfor(nthr, (int64_t)P.je * ni, [&](int64_t a, int64_t b) {
            int64_t f = 0, o2 = 0;
            for (int64_t k = a; k < b; ++k)
                if (c->mask[k]) (k < (int64_t)P.jb * ni ? f : o2) += 1;
            fg += f; no += o2;
        });
        P.first_global = fg.load();
        P.n_owned = no.load();
    }

    if (!P.factored()) {
        build_coeff_arrays();
        P.setup_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        P.zcolptr.assign(P.n_owned + 1, 0);
        return Status::ok();
    }

    // ---- AINV per block (reading R15)
    std::vector<AinvBlock> blocks;
    // halo-AINV across ranks (w > 0): this rank's block covers its owned rows plus w
    // southern halo rows (its columns' entries there are applied through K2's gathers of the
    // received q / r halo rows), and the columns of the northern neighbour whose entries fall in
    // this rank's top rows are recomputed here -- the neighbour's block starts w rows below its
    // first row and AINV is left-looking, so its first kNorthRows rows of columns depend on rows
    // [je - w, je + kNorthRows) only -- and appended to this rank's Z rows (K3 then gathers t on
    // the northern halo rows it receives from the neighbour).
    constexpr int32_t kNorthRows = 16;
    const bool halo_x = P.nranks > 1 && o->ainv_halo > 0;
    const int32_t w = std::min(o->ainv_halo, nj);     // >= nj: the global Z (every block from row 0)
    if (halo_x && P.rank < P.nranks - 1 && P.nloc < kNorthRows)
        return Status::err(PCG_ERR_ARG, "pcg_setup: halo-AINV across ranks needs >= 16 rows per rank");
    bool have_north = false;
    if (P.nranks > 1) {
        AinvBlock b; b.row_lo = std::max(0, P.jb - w); b.row_own = P.jb; b.row_hi = P.je;
        blocks.push_back(b);
        if (halo_x && P.rank < P.nranks - 1) {
            have_north = true;
            AinvBlock nb; nb.row_lo = std::max(0, P.je - w); nb.row_own = P.je; nb.row_hi = std::min(nj, P.je + kNorthRows);
            blocks.push_back(nb);                        // blocks[1]: the neighbour's first columns
        }
    } else {
        int32_t parts = std::max(1, o->ainv_parts);
        if (parts > nj) return Status::err(PCG_ERR_ARG, "pcg_setup: ainv_parts > nj");
        std::vector<int32_t> rb(parts + 1);
        if (Status s = partition_rows(ni, nj, c->mask, parts, rb.data()); !s) return s;
        for (int32_t p = 0; p < parts; ++p) {
            AinvBlock b;
            b.row_own = rb[p]; b.row_hi = rb[p + 1];
            b.row_lo = parts == 1 ? 0 : std::max(0, rb[p] - o->ainv_halo);
            blocks.push_back(b);
        }
    }
    if (P.precond == PCG_PRECOND_FSAI) {            // one block: the banded FSAI of T (NEXT-1)
        blocks.assign(1, AinvBlock());
        fsai_block(ni, nj, P.periodic, c->cE, c->cN, c->mask, P.fsai_q, diag_of, blocks[0]);
    } else {
        int nthreads = o->setup_threads > 0 ? o->setup_threads : (int)std::max(1u, std::thread::hardware_concurrency());
        nthreads = std::min(nthreads, 64);
        // threads across blocks first, the rest inside each block (ainv.cpp's column wavefront)
        const int inner = std::max(1, nthreads / (int)blocks.size());
        nthreads = std::min<int>(nthreads, (int)blocks.size());
        std::vector<std::thread> pool;
        std::atomic_size_t next{0};
        auto work = [&]() {
            for (size_t k; (k = next.fetch_add(1)) < blocks.size();)
                ainv_block(ni, nj, P.periodic, c->cE, c->cN, c->sigma, c->mask, P.tau, P.ainv_fill, blocks[k], inner);
        };
        const auto ta = std::chrono::steady_clock::now();
        for (int t = 1; t < nthreads; ++t) pool.emplace_back(work);
        work();
        for (auto& t : pool) t.join();
        if (getenv("PCG_VERBOSE"))
            fprintf(stderr, "libpcg: AINV %zu block(s) x %d thread(s): %.3f s\n", blocks.size(), inner,
                    std::chrono::duration<double>(std::chrono::steady_clock::now() - ta).count());
    }
    for (auto& b : blocks)
        if (b.fail_grid >= 0) {
            char buf[200];
            snprintf(buf, sizeof buf, "pcg_setup: AINV pivot <= 1e-12 or not finite at grid point (i=%d, j=%d): "
                     "A is not SPD to working precision", (int)(b.fail_grid % ni), (int)(b.fail_grid / ni));
            return Status::err(PCG_ERR_NOT_SPD, buf, global_unknown(c->mask, ni, b.fail_grid));
        }

    stage("AINV");
    AinvBlock north;
    int32_t reach = 0;                                   // t rows needed north of je
    if (have_north) {
        north = std::move(blocks[1]);
        blocks.pop_back();
        for (size_t q = 0; q < north.col_g.size(); ++q) {
            const int32_t jc = (int32_t)(north.col_g[q] / ni);
            for (int64_t e = north.colptr[q]; e < north.colptr[q + 1]; ++e)
                if (north.row_g[e] < (int64_t)P.je * ni) {
                    if (jc >= P.je + kNorthRows - 1)
                        return Status::err(PCG_ERR_ARG, "pcg_setup: Z reaches more than 15 rows (halo-AINV across ranks)");
                    reach = std::max(reach, jc - P.je + 1);
                }
        }
    }
    // rows of this rank's t the southern neighbour gathers: the reach of this rank's own columns
    // into its southern halo rows (the neighbour computed the same columns as its north block)
    int32_t reach_s = 0;
    if (halo_x && P.rank > 0)
        for (size_t q = 0; q < blocks[0].col_g.size(); ++q) {
            const int32_t jc = (int32_t)(blocks[0].col_g[q] / ni);
            for (int64_t e = blocks[0].colptr[q]; e < blocks[0].colptr[q + 1]; ++e)
                if (blocks[0].row_g[e] < (int64_t)P.jb * ni) reach_s = std::max(reach_s, jc - P.jb + 1);
        }
    // rows of q / r the solve exchanges: the actual southern extent of this rank's columns (<= w;
    // with w >= jb every block starts at row 0 and the owned columns are the GLOBAL Z's -- the
    // left-looking column j only involves rows and columns < j -- NEXT-3's P-invariant
    // preconditioner, whose extent is still Z's pattern reach, 2-3 rows at tau = 0.1)
    int32_t w_eff = 0;
    if (halo_x)
        for (size_t q = 0; q < blocks[0].col_g.size(); ++q)
            for (int64_t e = blocks[0].colptr[q]; e < blocks[0].colptr[q + 1]; ++e)
                if (blocks[0].row_g[e] < (int64_t)P.jb * ni)
                    w_eff = std::max(w_eff, P.jb - (int32_t)(blocks[0].row_g[e] / ni));
    // rows of q / r this rank SENDS north: the southern extent of the northern neighbour's first
    // columns, which this rank recomputed bitwise in `north` (same index set as the neighbour's
    // block), so sender and receiver agree on the message size without communicating
    int32_t w_send = 0;
    if (have_north)
        for (size_t q = 0; q < north.col_g.size(); ++q)
            for (int64_t e = north.colptr[q]; e < north.colptr[q + 1]; ++e)
                if (north.row_g[e] < (int64_t)P.je * ni) w_send = std::max(w_send, P.je - (int32_t)(north.row_g[e] / ni));
    if (halo_x) P.halo = std::max({P.halo, w_eff, reach});
    P.halo_w = halo_x ? std::max(1, w_eff) : 0;
    P.halo_w_send = halo_x ? std::max(1, w_send) : 0;
    P.halo_t = reach;
    P.halo_t_send = reach_s;
    build_coeff_arrays();
    stage("coefficient arrays");

    // ---- owned columns in natural order: export + Z values z_kj = fl(s_k * zhat_kj)
    auto arr_of = [&](int64_t gi) -> int64_t {        // grid index -> array index (owned / halo rows)
        int32_t i = (int32_t)(gi % ni), j = (int32_t)(gi / ni);
        return (int64_t)(j - P.jb + P.halo) * pitch + i;
    };
    P.zcolptr.assign(1, 0);
    bigvec<int64_t> colarr;                      // array index of each owned column
    bigvec<int32_t> ent_row_arr;                 // per entry: array index of its row
    bigvec<double> ent_z;                        // per entry: z value
    std::vector<int64_t> gunk_cache;
    // global unknown numbering of grid rows [min row_lo, je)
    int32_t rlo = P.je;
    for (auto& b : blocks) rlo = std::min(rlo, b.row_lo);
    const bool exp = P.keep_export;
    std::vector<int64_t> unk(exp ? (size_t)(P.je - rlo) * ni : 0, -1);
    if (exp) {
        std::atomic<int64_t> below(0);
        pfor(nthr, (int64_t)rlo * ni, [&](int64_t a, int64_t b) {
            int64_t u = 0;
            for (int64_t k = a; k < b; ++k) u += c->mask[k] ? 1 : 0;
            below += u;
        });
        std::vector<int64_t> rowstart;                   // ocean points before each row of [rlo, je)
        pscan(nthr, (int64_t)(P.je - rlo), rowstart, [&](int64_t r) {
            int64_t u = 0;
            const uint8_t* m = c->mask + (int64_t)(rlo + r) * ni;
            for (int32_t i = 0; i < ni; ++i) u += m[i] ? 1 : 0;
            return u;
        });
        pfor(nthr, (int64_t)(P.je - rlo), [&](int64_t r0, int64_t r1) {
            for (int64_t r = r0; r < r1; ++r) {
                int64_t u = below.load() + rowstart[(size_t)r];
                for (int32_t i = 0; i < ni; ++i)
                    if (c->mask[(rlo + r) * ni + i]) unk[(size_t)(r * ni + i)] = u++;
            }
        }, 64);
    }
    // Jacobi scale s_g = 1/sqrt(A_gg) once per grid point of the rows the entries touch (the same
    // IEEE operations as per entry; FSAI: no scale)
    const int32_t rhi = std::min(nj, P.je + kNorthRows);
    bigvec<double> sgrid((size_t)(rhi - rlo) * ni);
    pfor(nthr, (int64_t)(rhi - rlo) * ni, [&](int64_t a, int64_t b) {
        for (int64_t g2 = (int64_t)rlo * ni + a; g2 < (int64_t)rlo * ni + b; ++g2)
            sgrid[(size_t)(g2 - (int64_t)rlo * ni)] =
                (P.precond != PCG_PRECOND_FSAI && c->mask[g2]) ? 1.0 / std::sqrt(diag_of(g2)) : 1.0;
    });
    auto scale_of = [&](int64_t gr) { return sgrid[(size_t)(gr - (int64_t)rlo * ni)]; };
    stage("  numbering + scales");
    int64_t ntot = 0, ncols = 0;
    for (auto& b : blocks) { ntot += b.colptr.back(); ncols += (int64_t)b.col_g.size(); }
    // flat column index over the blocks, entry offsets by prefix sum, then a parallel fill
    struct ColSrc { int32_t first, second; };                        // trivial: no serial init
    bigvec<ColSrc> colsrc((size_t)ncols);                            // (block, column in block)
    {
        int64_t k0 = 0;
        for (size_t bi = 0; bi < blocks.size(); ++bi) {
            const int64_t nb = (int64_t)blocks[bi].col_g.size();
            pfor(nthr, nb, [&](int64_t a, int64_t b) {
                for (int64_t q = a; q < b; ++q) colsrc[(size_t)(k0 + q)] = {(int32_t)bi, (int32_t)q};
            });
            k0 += nb;
        }
    }
    pscan(nthr, ncols, P.zcolptr, [&](int64_t k) {
        const AinvBlock& b = blocks[(size_t)colsrc[(size_t)k].first];
        const int32_t q = colsrc[(size_t)k].second;
        return b.colptr[q + 1] - b.colptr[q];
    });
    stage("  column offsets");
    if (exp) { P.zrow.resize((size_t)ntot); P.zhat.resize((size_t)ntot); }
    ent_z.resize((size_t)ntot); ent_row_arr.resize((size_t)ntot);
    P.pivots.resize((size_t)ncols); P.scale.resize((size_t)ncols); colarr.resize((size_t)ncols);
    pfor(nthr, ncols, [&](int64_t k0, int64_t k1) {
        for (int64_t k = k0; k < k1; ++k) {
            const AinvBlock& b = blocks[(size_t)colsrc[(size_t)k].first];
            const int32_t q = colsrc[(size_t)k].second;
            int64_t dst = P.zcolptr[(size_t)k];
            for (int64_t e = b.colptr[q]; e < b.colptr[q + 1]; ++e, ++dst) {
                const int64_t gr = b.row_g[e];
                if (exp) {
                    P.zrow[(size_t)dst] = unk[gr - (int64_t)rlo * ni];
                    P.zhat[(size_t)dst] = b.zhat[e];
                }
                ent_z[(size_t)dst] = scale_of(gr) * b.zhat[e];
                ent_row_arr[(size_t)dst] = (int32_t)arr_of(gr);
            }
            P.pivots[(size_t)k] = b.piv[q];
            P.scale[(size_t)k] = scale_of(b.col_g[q]);
            colarr[(size_t)k] = arr_of(b.col_g[q]);
            P.piv[colarr[(size_t)k]] = b.piv[q];
        }
    });
    P.nnz_off = ntot - ncols;
    if ((int64_t)colarr.size() != P.n_owned) return Status::err(PCG_ERR_ARG, "internal: owned column count mismatch");
    const int64_t hoff = (int64_t)P.halo * pitch;        // array index of owned element 0
    {
        std::atomic<bool> outside(false);        // entries in the southern halo rows only with halo-AINV across ranks
        pfor(nthr, (int64_t)ent_row_arr.size(), [&](int64_t a, int64_t b) {
            for (int64_t e = a; e < b; ++e)
                if (ent_row_arr[(size_t)e] < hoff - (int64_t)P.halo_w * pitch) outside = true;
        });
        if (outside) return Status::err(PCG_ERR_ARG, "internal: Z entry outside the owned rows");
    }

    stage("export + Z values");
    // ---- SELL of Z^T rows: row (column j of Z) = entries k ascending
    const int64_t nown = P.owned_elements();
    std::atomic<bool> fits_zt(true), fits_z(true);
    {
        bigvec<int64_t> colq((size_t)nown);                 // element -> owned column (-1: none)
        pfor(nthr, nown, [&](int64_t a, int64_t b) { for (int64_t e = a; e < b; ++e) colq[(size_t)e] = -1; });
        pfor(nthr, (int64_t)colarr.size(), [&](int64_t a, int64_t b) {
            for (int64_t q = a; q < b; ++q) colq[(size_t)(colarr[(size_t)q] - hoff)] = q;
        });
        auto len = [&](int64_t e) {
            const int64_t q = colq[(size_t)e];
            return q < 0 ? (int64_t)0 : P.zcolptr[(size_t)q + 1] - P.zcolptr[(size_t)q];
        };
        ell_shape(P.ZT, nown, hoff, nthr, len);
        pfor(nthr, (int64_t)colarr.size(), [&](int64_t q0, int64_t q1) {
            for (int64_t q = q0; q < q1; ++q) {
                const int64_t e = colarr[(size_t)q] - hoff, z0 = P.zcolptr[(size_t)q];
                for (int64_t k = 0; k < P.zcolptr[(size_t)q + 1] - z0; ++k)
                    ell_put(P.ZT, e, k, ent_row_arr[(size_t)(z0 + k)], ent_z[(size_t)(z0 + k)], hoff, fits_zt);
            }
        });
    }
    stage("pack Z^T");
    // ---- SELL of Z rows: row i = entries z_ij over columns j ascending (owned rows only; with
    // halo-AINV across ranks the northern neighbour's columns follow this rank's, ascending)
    {
        std::vector<int64_t> ncol_arr, nrow_arr;           // north entries in owned rows
        std::vector<double> nz;
        for (size_t q = 0; q < north.col_g.size(); ++q)
            for (int64_t e = north.colptr[q]; e < north.colptr[q + 1]; ++e)
                if (north.row_g[e] < (int64_t)P.je * ni) {
                    const int64_t gr = north.row_g[e];
                    ncol_arr.push_back(arr_of(north.col_g[q]));
                    nrow_arr.push_back(arr_of(gr));
                    nz.push_back(scale_of(gr) * north.zhat[e]);
                }
        for (int64_t r : nrow_arr)
            if (r < hoff) return Status::err(PCG_ERR_ARG, "internal: northern Z entry below the owned rows");
        // transpose with the ascending column order per row kept: thread t owns the rows
        // [R_t, R_t+1) and visits, in ascending order, the columns that can hold entries of them
        // (a column's entries are at rows <= the column, so columns from the first row >= R_t on,
        // until past Z's reach); one such walk counts the rows' entries, the second places them
        const int64_t nc = (int64_t)colarr.size();
        std::atomic<int64_t> reach_a(0);                   // largest column - row distance of an entry
        pfor(nthr, nc, [&](int64_t a, int64_t b) {
            int64_t r = 0;
            for (int64_t q = a; q < b; ++q)
                for (int64_t e = P.zcolptr[q]; e < P.zcolptr[q + 1]; ++e) r = std::max(r, colarr[q] - ent_row_arr[e]);
            int64_t cur = reach_a.load();
            while (r > cur && !reach_a.compare_exchange_weak(cur, r)) {
            }
        });
        const int64_t reach = reach_a.load();
        const int T = (nc < 100000) ? 1 : nthr;
        auto walk = [&](auto&& visit) {                    // visit(row, column q, entry e) in order
            std::vector<std::thread> pool;
            auto part = [&](int t) {
                const int64_t R0 = nown * t / T, R1 = nown * (t + 1) / T;
                const int64_t q0 = std::lower_bound(colarr.begin(), colarr.end(), R0 + hoff) - colarr.begin();
                for (int64_t q = q0; q < nc; ++q) {
                    bool below = false;                    // some entry of this column lies below R1
                    for (int64_t e = P.zcolptr[q]; e < P.zcolptr[q + 1]; ++e) {
                        if (ent_row_arr[e] < hoff) continue;   // a southern halo row: rank-1's Z row
                        const int64_t r = ent_row_arr[e] - hoff;
                        if (r < R1) below = true;
                        if (r < R0 || r >= R1) continue;
                        visit(r, q, e);
                    }
                    if (!below && colarr[q] - hoff >= R1 + reach) break;   // past Z's reach
                }
            };
            for (int t = 1; t < T; ++t) pool.emplace_back(part, t);
            part(0);
            for (auto& th : pool) th.join();
        };
        bigvec<int64_t> cnt((size_t)nown);                      // entries per row, then placed so far
        pfor(nthr, nown, [&](int64_t a, int64_t b) { for (int64_t e = a; e < b; ++e) cnt[(size_t)e] = 0; });
        walk([&](int64_t r, int64_t, int64_t) { cnt[(size_t)r]++; });
        for (int64_t r : nrow_arr) cnt[(size_t)(r - hoff)]++;
        ell_shape(P.Z, nown, hoff, nthr, [&](int64_t e) { return cnt[(size_t)e]; });
        bigvec<int64_t>& fill = cnt;
        pfor(nthr, nown, [&](int64_t a, int64_t b) { for (int64_t e = a; e < b; ++e) fill[(size_t)e] = 0; });
        walk([&](int64_t r, int64_t q, int64_t e) {
            ell_put(P.Z, r, fill[(size_t)r]++, (int32_t)colarr[q], ent_z[e], hoff, fits_z);
        });
        for (size_t m = 0; m < nrow_arr.size(); ++m) {     // north columns, ascending
            const int64_t r = nrow_arr[m] - hoff;
            ell_put(P.Z, r, fill[(size_t)r]++, (int32_t)ncol_arr[m], nz[m], hoff, fits_z);
        }
    }
    for (auto [E, f] : {std::pair<Ell*, bool>{&P.ZT, fits_zt.load()}, {&P.Z, fits_z.load()}})
        if (!f) { E->col16.clear(); E->col16.shrink_to_fit(); }
    stage("pack Z");
    // ---- FSAI DIA form: each owned column's entries at consecutive columns of the
    // same grid row i-1, i-2, ... (no land, wrap or N-S link inside the chain) -> diagonals
    if (P.precond == PCG_PRECOND_FSAI && P.fsai_q > 0) {
        const int32_t q = P.fsai_q;
        bool plain = true;
        std::vector<double> dia((size_t)q * nown, 0.0);
        for (size_t c0 = 0; c0 < colarr.size() && plain; ++c0) {
            const int64_t ec = colarr[c0] - hoff;                        // owned element of column
            const int64_t ne = P.zcolptr[c0 + 1] - P.zcolptr[c0] - 1;  // entries above the diagonal
            for (int64_t m = 1; m <= ne; ++m) {
                const int64_t e = P.zcolptr[c0 + 1] - 1 - m;             // entry at row k - m
                if (ent_row_arr[e] != colarr[c0] - m || (colarr[c0] % pitch) < m) { plain = false; break; }
                dia[(size_t)(m - 1) * nown + ec] = ent_z[e];
            }
        }
        if (plain) {
            P.dia_q = q;
            P.dia = std::move(dia);
        }
    }
    P.setup_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return Status::ok();
}

}  // namespace pcg
