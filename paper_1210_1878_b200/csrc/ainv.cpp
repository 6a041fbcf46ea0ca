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
#include <sys/mman.h>

#include <atomic>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <memory>
#include <mutex>
#include <thread>
#include <cstdlib>
#include <cstring>
#include <new>
#include <algorithm>
#include <functional>
#include <queue>
#include <vector>

#include "internal.h"

namespace pcg {

namespace {

struct BlockMatrix {
    int32_t n = 0;
    // the scaled matrix A^ as 5 fixed slots per row (value and column side by side, columns
    // ascending): row p = e5[5p .. 5p + m5[p])
    struct Ent { double a; int32_t c; int32_t pad; };
    bigvec<Ent> e5;
    bigvec<uint8_t> m5;
    bigvec<int64_t> grid;             // local unknown -> grid index
    bigvec<double> diag;              // A_pp
};

// zero-initialised array from an anonymous mapping advised as transparent huge pages: the pages a
// thread never touches are never written (the per-thread n-sized work arrays of the column
// workers touch only their columns' neighbourhood), and the ones it touches fault in 2 MB at a
// time (4 KB faults of 16 threads serialise in the kernel)
template <class T>
struct ZeroArr {
    T* p = nullptr;
    size_t bytes = 0;
    explicit ZeroArr(size_t n) : bytes((std::max<size_t>(n, 1) * sizeof(T) + (size_t(2) << 20) - 1) & ~((size_t(2) << 20) - 1)) {
        void* m = mmap(nullptr, bytes, PROT_READ | PROT_WRITE, MAP_PRIVATE | MAP_ANONYMOUS, -1, 0);
        if (m == MAP_FAILED) throw std::bad_alloc();
        madvise(m, bytes, MADV_HUGEPAGE);
        p = static_cast<T*>(m);
    }
    ~ZeroArr() { munmap(p, bytes); }
    ZeroArr(const ZeroArr&) = delete;
    ZeroArr& operator=(const ZeroArr&) = delete;
    T& operator[](size_t i) { return p[i]; }
};

// Faces of (i,j): E, W, N, S with existence and coupling.
inline void faces(int32_t ni, int32_t nj, int32_t periodic, const double* cE, const double* cN,
                  int32_t i, int32_t j, bool ex[4], int32_t in[4], int32_t jn[4], double c[4]) {
    const int64_t row = (int64_t)j * ni;
    const int32_t ie = i + 1 == ni ? 0 : i + 1, iw = i == 0 ? ni - 1 : i - 1;     // E-W wrap
    ex[0] = (i + 1 < ni) || periodic;  in[0] = ie; jn[0] = j;     c[0] = ex[0] ? cE[row + i] : 0.0;
    ex[1] = (i >= 1) || periodic;      in[1] = iw; jn[1] = j;     c[1] = ex[1] ? cE[row + iw] : 0.0;
    ex[2] = (j + 1 < nj);              in[2] = i;  jn[2] = j + 1; c[2] = ex[2] ? cN[row + i] : 0.0;
    ex[3] = (j >= 1);                  in[3] = i;  jn[3] = j - 1; c[3] = ex[3] ? cN[row - ni + i] : 0.0;
}

}  // namespace

void ainv_block(int32_t ni, int32_t nj, int32_t periodic, const double* cE, const double* cN,
                const double* sigma, const uint8_t* mask, double tau, int32_t fill, AinvBlock& blk, int threads) {

    const int32_t r0 = blk.row_lo, r1 = blk.row_hi;
    const int T0 = std::max(1, threads);
    // parallel for over [0, n) in T0 contiguous ranges (element-wise independent work only)
    auto pfor = [&](int64_t n_, const std::function<void(int64_t, int64_t)>& f) {
        const int T = n_ < 50000 ? 1 : T0;
        std::vector<std::thread> pool;
        for (int t = 1; t < T; ++t) pool.emplace_back(f, n_ * t / T, n_ * (t + 1) / T);
        f(0, n_ / T);
        for (auto& th : pool) th.join();
    };
    const bool verbose = getenv("PCG_VERBOSE") != nullptr;
    auto tprev = std::chrono::steady_clock::now();
    auto stage = [&](const char* what) {
        if (!verbose) return;
        const auto now = std::chrono::steady_clock::now();
        fprintf(stderr, "libpcg:   ainv %-24s %.3f s\n", what, std::chrono::duration<double>(now - tprev).count());
        tprev = now;
    };
    // exclusive prefix sum out[0..n] of cnt(i) in T0 contiguous ranges (two passes)
    auto prefix = [&](int64_t n_, auto&& cnt, auto* out) {
        const int T = n_ < 50000 ? 1 : T0;
        std::vector<int64_t> part((size_t)T + 1, 0);
        auto run = [&](auto&& body) {
            std::vector<std::thread> pool;
            for (int t = 1; t < T; ++t) pool.emplace_back([&, t] { body(t, n_ * t / T, n_ * (t + 1) / T); });
            body(0, 0, n_ / T);
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
            for (int64_t i = a; i < b; ++i) { out[i] = acc; acc += cnt(i); }
        });
        out[n_] = part[(size_t)T];
    };
    BlockMatrix M;
    // local numbering of the ocean points of rows [r0, r1), natural order: ocean points per row,
    // prefix over the rows, then every row numbered in parallel
    const int32_t nr = r1 - r0;
    std::vector<int32_t> rowstart((size_t)nr + 1, 0);
    {
        std::vector<int32_t> cnt((size_t)nr, 0);
        pfor((int64_t)nr * 256, [&](int64_t a0, int64_t a1) {      // (x256: rows are few, each ni wide)
            for (int64_t r = (a0 + 255) / 256; r < (a1 + 255) / 256; ++r) {
                int32_t u = 0;
                for (int32_t i = 0; i < ni; ++i) u += mask[(int64_t)(r0 + r) * ni + i] ? 1 : 0;
                cnt[(size_t)r] = u;
            }
        });
        for (int32_t r = 0; r < nr; ++r) rowstart[(size_t)r + 1] = rowstart[(size_t)r] + cnt[(size_t)r];
    }
    M.n = rowstart[(size_t)nr];
    const int32_t n = M.n;
    bigvec<int32_t> loc((size_t)nr * ni);
    M.grid.resize((size_t)n);
    pfor((int64_t)nr * 256, [&](int64_t a0, int64_t a1) {
        for (int64_t r = (a0 + 255) / 256; r < (a1 + 255) / 256; ++r) {
            int32_t u = rowstart[(size_t)r];
            for (int32_t i = 0; i < ni; ++i) {
                const int64_t g = (int64_t)(r0 + r) * ni + i;
                if (mask[g]) { loc[(size_t)r * ni + i] = u; M.grid[(size_t)u] = g; ++u; }
                else loc[(size_t)r * ni + i] = -1;
            }
        }
    });
    stage("numbering");
    M.diag.resize(n);
    bigvec<double> sc(n);
    bigvec<int32_t> gi(n), gj(n);                   // grid column / row of each unknown
    pfor((int64_t)nr * 256, [&](int64_t a0, int64_t a1) {
        for (int64_t r = (a0 + 255) / 256; r < (a1 + 255) / 256; ++r)
            for (int32_t i = 0; i < ni; ++i) {
                const int32_t p = loc[(size_t)r * ni + i];
                if (p >= 0) { gi[(size_t)p] = i; gj[(size_t)p] = r0 + (int32_t)r; }
            }
    });
    // diagonal A_pp = ((c_E + c_W) + c_N) + c_S (+ sigma) over all faces, then s = 1/sqrt(A_pp)
    pfor(n, [&](int64_t lo, int64_t hi) {
        for (int64_t p = lo; p < hi; ++p) {
            const int64_t g = M.grid[p];
            const int32_t i = gi[(size_t)p], j = gj[(size_t)p];
            bool ex[4]; int32_t in[4], jn[4]; double c[4];
            faces(ni, nj, periodic, cE, cN, i, j, ex, in, jn, c);
            double d = ((c[0] + c[1]) + c[2]) + c[3];
            if (sigma) d = d + sigma[g];
            M.diag[p] = d;
            sc[p] = 1.0 / std::sqrt(d);
        }
    });
    // A^ restricted to the block: a^_pq = A_pq * (s_p * s_q), every row in its 5 slots (sorted by
    // column)
    M.e5.resize((size_t)5 * n);
    M.m5.resize((size_t)n);
    auto row_of = [&](int64_t p, BlockMatrix::Ent* r) {
        const int32_t i = gi[(size_t)p], j = gj[(size_t)p];
        bool ex[4]; int32_t in[4], jn[4]; double c[4];
        faces(ni, nj, periodic, cE, cN, i, j, ex, in, jn, c);
        int m = 0;
        r[m].c = (int32_t)p; r[m].a = M.diag[p] * (sc[p] * sc[p]); r[m].pad = 0;
        ++m;
        for (int f = 0; f < 4; ++f) {
            if (!ex[f] || !(c[f] > 0.0) || !mask[(int64_t)jn[f] * ni + in[f]]) continue;
            if (jn[f] < r0 || jn[f] >= r1) continue;    // outside the block's index set
            const int32_t q = loc[(size_t)(jn[f] - r0) * ni + in[f]];
            r[m].c = q; r[m].a = (-c[f]) * (sc[p] * sc[q]); r[m].pad = 0;
            ++m;
        }
        for (int x = 1; x < m; ++x)
            for (int y = x; y > 0 && r[y - 1].c > r[y].c; --y) std::swap(r[y], r[y - 1]);
        return m;
    };
    pfor(n, [&](int64_t lo, int64_t hi) {
        for (int64_t p = lo; p < hi; ++p) M.m5[(size_t)p] = (uint8_t)row_of(p, &M.e5[(size_t)5 * p]);
    });
    stage("scaled matrix");
    // Zhat columns and pivots.  Column j needs the finished columns i < j it meets as
    // candidates (pivot p_i, entries of zhat_i), nothing else, so the columns can be built by
    // several threads at once with bitwise the sequential result (every column runs the same
    // operations in the same order; only the time it waits differs).  Thread t owns the grid
    // columns [cb[t], cb[t+1]) of every row and builds its columns in increasing order -- a
    // wavefront: the first column of its chunk in row r waits for the west neighbour, the last one
    // of thread t-1's chunk in row r, so thread t runs about one row behind thread t-1.  A column
    // whose candidate is not finished yet spins on its `done` flag (release / acquire).
    // Progress: a thread only waits for smaller columns, and the smallest unfinished column's
    // dependencies are all finished.  On an AINV failure (pivot <= 1e-12) columns beyond the
    // smallest failing one are abandoned, so the reported column is the sequential one.
    struct ColRef {                              // trivial: bigvec leaves it uninitialised
        const int32_t* r;
        const double* v;
        int32_t len;
    };
    bigvec<ColRef> cref(n);                      // written before done[j], read after it
    bigvec<double> piv(n);
    std::unique_ptr<std::atomic<uint8_t>[]> done(new std::atomic<uint8_t>[std::max(n, 1)]);
    pfor(n, [&](int64_t lo, int64_t hi) { for (int64_t p = lo; p < hi; ++p) done[p].store(0, std::memory_order_relaxed); });
    std::atomic<int32_t> limit(n);
    int T = std::max(1, threads);
    if (n < 20000) T = 1;
    T = std::min(T, std::max(1, ni / 64));
    // thread t: grid columns [cb[t], cb[t+1]) of every row (i -> min(T-1, i T / ni)), its
    // unknowns in increasing order, listed by the threads themselves from the local numbering
    std::vector<int32_t> cb((size_t)T + 1, ni);
    for (int32_t i = ni - 1; i >= 0; --i) cb[(size_t)std::min<int64_t>(T - 1, (int64_t)i * T / ni)] = i;
    for (int t = T - 1; t >= 0; --t) cb[(size_t)t] = std::min(cb[(size_t)t], cb[(size_t)t + 1]);
    std::vector<std::vector<int32_t>> mine((size_t)T);
    {
        std::vector<std::thread> pool;
        auto list = [&](int t) {
            std::vector<int32_t>& v = mine[(size_t)t];
            v.reserve((size_t)n / T + (size_t)nr + 16);
            for (int32_t r = 0; r < nr; ++r)
                for (int32_t i = cb[(size_t)t]; i < cb[(size_t)t + 1]; ++i) {
                    const int32_t p = loc[(size_t)r * ni + i];
                    if (p >= 0) v.push_back(p);
                }
        };
        std::atomic<bool> oom(false);
        auto run = [&](int t) {
            try { list(t); } catch (const std::bad_alloc&) { oom = true; }
        };
        for (int t = 1; t < T; ++t) pool.emplace_back(run, t);
        run(0);
        for (auto& th : pool) th.join();
        if (oom) throw std::bad_alloc();
    }
    std::vector<std::vector<std::unique_ptr<int32_t[]>>> seg_r((size_t)T);
    std::vector<std::vector<std::unique_ptr<double[]>>> seg_v((size_t)T);
    auto worker = [&](int t) {
        // per unknown k, one 16-byte slot: the working value w, the stamp of the last column that
        // listed k (bit 31: k is live -- present -- in the current column; a live k is always
        // listed by it), the stamp of the last column that queued k as a candidate
        struct Slot { double w; uint32_t lst; int32_t queued; };
        ZeroArr<Slot> sl((size_t)n);
        constexpr uint32_t kLive = 0x80000000u;
        std::vector<int32_t> members, touched;
        std::priority_queue<int32_t, std::vector<int32_t>, std::greater<int32_t>> cand;
        // column storage in fixed segments (a column's entries never move once published; the
        // segments outlive every thread, which may read them until the last one finishes)
        std::vector<std::unique_ptr<int32_t[]>>& segr = seg_r[(size_t)t];
        std::vector<std::unique_ptr<double[]>>& segv = seg_v[(size_t)t];
        size_t seg_cap = 0, seg_used = 0;
        auto wait_for = [&](int32_t i, int32_t j) -> bool {
            for (unsigned spin = 0; !done[i].load(std::memory_order_acquire); ++spin) {
                if (j >= limit.load(std::memory_order_relaxed)) return false;
                if (spin > 64) std::this_thread::yield();
            }
            return true;
        };
        for (int32_t j : mine[(size_t)t]) {
            if (j >= limit.load(std::memory_order_relaxed)) return;
            members.clear();
            const int32_t stamp = j + 1;
            members.push_back(j); sl[j].lst = (uint32_t)stamp | kLive; sl[j].w = 1.0;
            for (const BlockMatrix::Ent* e = &M.e5[(size_t)5 * j], *ee = e + M.m5[(size_t)j]; e < ee; ++e) {
                const int32_t i = e->c;
                if (i < j && sl[i].queued != stamp) { sl[i].queued = stamp; cand.push(i); }
            }
            bool ok = true;
            while (!cand.empty()) {
                const int32_t i = cand.top(); cand.pop();
                // pi = a^_i . z over row i of A^ (ascending columns, present entries)
                double pi = 0.0;
                for (const BlockMatrix::Ent* e = &M.e5[(size_t)5 * i], *ee = e + M.m5[(size_t)i]; e < ee; ++e) {
                    const int32_t k = e->c;
                    if (sl[k].lst == ((uint32_t)stamp | kLive)) pi = pi + e->a * sl[k].w;
                }
                if (pi == 0.0) continue;
                if (!wait_for(i, j)) { ok = false; break; }
                const double coef = pi / piv[i];
                touched.clear();
                const ColRef zi = cref[i];
                for (int32_t q = 0; q < zi.len; ++q) {
                    const int32_t k = zi.r[q];
                    if (sl[k].lst != ((uint32_t)stamp | kLive)) {
                        if (sl[k].lst != (uint32_t)stamp) members.push_back(k);
                        sl[k].lst = (uint32_t)stamp | kLive; sl[k].w = 0.0;
                        for (const BlockMatrix::Ent* e2 = &M.e5[(size_t)5 * k], *ee2 = e2 + M.m5[(size_t)k]; e2 < ee2; ++e2) {
                            const int32_t i2 = e2->c;
                            if (i2 > i && i2 < j && sl[i2].queued != stamp) { sl[i2].queued = stamp; cand.push(i2); }
                        }
                    }
                    sl[k].w = sl[k].w - coef * zi.v[q];
                    touched.push_back(k);
                }
                for (int32_t k : touched)
                    if (k != j && std::fabs(sl[k].w) < tau) { sl[k].lst = (uint32_t)stamp; sl[k].w = 0.0; }
                if (fill > 0) {
                    // P_B2 (reading R26): keep the diagonal and the fill-1 largest |z|, ties to the
                    // smaller index
                    touched.clear();
                    for (int32_t k : members)
                        if (k != j && sl[k].lst == ((uint32_t)stamp | kLive)) touched.push_back(k);
                    if ((int64_t)touched.size() > (int64_t)fill - 1) {
                        std::sort(touched.begin(), touched.end(), [&](int32_t a, int32_t b) {
                            const double fa = std::fabs(sl[a].w), fb = std::fabs(sl[b].w);
                            return fa > fb || (fa == fb && a < b);
                        });
                        for (size_t x = (size_t)fill - 1; x < touched.size(); ++x) { sl[touched[x]].lst = (uint32_t)stamp; sl[touched[x]].w = 0.0; }
                    }
                }
            }
            if (!ok) {                                    // abandoned: a smaller column failed
                while (!cand.empty()) cand.pop();
                for (int32_t k : members) { sl[k].lst = (uint32_t)stamp; sl[k].w = 0.0; }
                return;
            }
            double pj = 0.0;
            for (const BlockMatrix::Ent* e = &M.e5[(size_t)5 * j], *ee = e + M.m5[(size_t)j]; e < ee; ++e) {
                const int32_t k = e->c;
                if (sl[k].lst == ((uint32_t)stamp | kLive)) pj = pj + e->a * sl[k].w;
            }
            std::sort(members.begin(), members.end());
            int32_t len = 0;
            for (int32_t k : members) len += sl[k].lst == ((uint32_t)stamp | kLive);
            if (seg_used + (size_t)len > seg_cap) {
                seg_cap = std::max<size_t>((size_t)len, 1 << 16);
                segr.emplace_back(new int32_t[seg_cap]);
                segv.emplace_back(new double[seg_cap]);
                seg_used = 0;
            }
            int32_t* rr = segr.back().get() + seg_used;
            double* vv = segv.back().get() + seg_used;
            int32_t q = 0;
            for (int32_t k : members) {
                if (sl[k].lst == ((uint32_t)stamp | kLive)) { rr[q] = k; vv[q] = sl[k].w; ++q; }
                sl[k].lst = (uint32_t)stamp; sl[k].w = 0.0;
            }
            seg_used += (size_t)len;
            cref[j] = ColRef{rr, vv, len};
            piv[j] = pj;
            if (!(pj > kPivotMin) || !std::isfinite(pj)) {
                int32_t cur = limit.load();
                while (j < cur && !limit.compare_exchange_weak(cur, j)) {
                }
                done[j].store(1, std::memory_order_release);
                return;
            }
            done[j].store(1, std::memory_order_release);
        }
    };
    stage("column lists");
    {
        // an allocation failure in a worker abandons every column (limit 0) and is rethrown here,
        // in the calling thread (pcg_setup reports PCG_ERR_NOMEM), never out of a std::thread
        std::atomic<bool> oom(false);
        auto run = [&](int t) {
            try {
                worker(t);
            } catch (const std::bad_alloc&) {
                oom = true;
                limit.store(0);
            }
        };
        std::vector<std::thread> pool;
        for (int t = 1; t < T; ++t) pool.emplace_back(run, t);
        run(0);
        for (auto& th : pool) th.join();
        if (oom) throw std::bad_alloc();
    }
    stage("column wavefront");
    const int64_t fail = limit.load() < n ? (int64_t)limit.load() : -1;
    blk.fail_grid = fail >= 0 ? M.grid[fail] : -1;
    if (fail >= 0) return;

    // owned columns (local unknowns whose grid row >= row_own), straight from the column
    // segments into the block's arrays (offsets by prefix sum, copies in parallel)
    int32_t first_owned = n;
    for (int32_t p = 0; p < n; ++p)
        if (M.grid[p] / ni >= blk.row_own) { first_owned = p; break; }
    const int32_t nown = n - first_owned;
    blk.colptr.resize((size_t)nown + 1);
    prefix(nown, [&](int64_t q) { return (int64_t)cref[first_owned + q].len; }, blk.colptr.data());
    blk.row_g.resize((size_t)blk.colptr[nown]);
    blk.zhat.resize((size_t)blk.colptr[nown]);
    blk.piv.resize(nown);
    blk.col_g.resize(nown);
    pfor(nown, [&](int64_t lo, int64_t hi) {
        for (int64_t q = lo; q < hi; ++q) {
            const int32_t j = first_owned + (int32_t)q;
            const ColRef& z = cref[j];
            for (int32_t x = 0; x < z.len; ++x) {
                blk.row_g[(size_t)blk.colptr[q] + x] = M.grid[z.r[x]];
                blk.zhat[(size_t)blk.colptr[q] + x] = z.v[x];
            }
            blk.piv[q] = piv[j];
            blk.col_g[q] = M.grid[j];
        }
    });
    stage("owned columns");
}

}  // namespace pcg
