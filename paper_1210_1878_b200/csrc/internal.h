// internal.h -- private structures of libpcg (host setup + device state).
//
// Device layout: every per-point array of a rank holds nloc+2 grid rows of
// `pitch` doubles (pitch = ni rounded up to a multiple of 32): row 0 is the southern halo,
// rows 1..nloc the owned rows j_begin..j_end-1, row nloc+1 the northern halo.  An owned
// element e = (j - j_begin)*pitch + i lives at array index a = e + pitch.  Entries with
// i >= ni, land points and (on one GPU) the halo rows hold 0 in every vector.
#pragma once

#include <sys/mman.h>

#include <cstdint>
#include <cstdlib>
#include <new>
#include <string>
#include <functional>
#include <utility>
#include <vector>

#include "../../include/libpcg.h"

namespace pcg {

constexpr int kBlock = 256;        // threads per block of every streaming kernel
constexpr int kSlice = 32;         // SELL slice height (one warp)
constexpr double kPivotMin = 1e-12;

struct Status {
    pcg_status code = PCG_OK;
    std::string msg;
    int64_t index = -1;
    static Status ok() { return {}; }
    static Status err(pcg_status c, std::string m, int64_t idx = -1) { return {c, std::move(m), idx}; }
    explicit operator bool() const { return code == PCG_OK; }
};

// std::vector whose elements are left uninitialised by resize: the large setup arrays (hundreds
// of MB at ORCA12 size) are written -- and their pages first touched -- by the parallel loops
// that compute them, instead of being zero-filled by one thread first.
template <class T>
struct NoInitAlloc : std::allocator<T> {
    NoInitAlloc() noexcept = default;
    template <class U> NoInitAlloc(const NoInitAlloc<U>&) noexcept {}
    template <class U> struct rebind { using other = NoInitAlloc<U>; };
    // arrays of 2 MB and more: 2 MB-aligned and advised as transparent huge pages, so the
    // parallel first touch takes one fault per 2 MB instead of one per 4 KB page (page faults
    // of one process serialise in the kernel)
    static constexpr size_t kHuge = size_t(2) << 20;
    T* allocate(size_t n) {
        const size_t bytes = n * sizeof(T);
#ifndef PCG_NO_THP
        if (bytes < kHuge) return std::allocator<T>::allocate(n);
#else
        if (true) return std::allocator<T>::allocate(n);
#endif
        const size_t r = (bytes + kHuge - 1) / kHuge * kHuge;
        void* p = std::aligned_alloc(kHuge, r);
        if (!p) throw std::bad_alloc();
        madvise(p, r, MADV_HUGEPAGE);
        return static_cast<T*>(p);
    }
    void deallocate(T* p, size_t n) noexcept {
#ifndef PCG_NO_THP
        if (n * sizeof(T) < kHuge) std::allocator<T>::deallocate(p, n);
#else
        if (true) std::allocator<T>::deallocate(p, n);
#endif
        else std::free(p);
    }
    template <class U> void construct(U* p) noexcept { ::new ((void*)p) U; }
    template <class U, class... A> void construct(U* p, A&&... a) { ::new ((void*)p) U(std::forward<A>(a)...); }
};
template <class T>
using bigvec = std::vector<T, NoInitAlloc<T>>;

// SELL-32 matrix over the owned elements: slice s covers owned elements [32 s, 32 s + 32)
// of one grid row; entry m of lane l is at off[s] + 32 m + l.  A column is stored as the
// packed grid offset (dj << 16) | (di & 0xffff) from the row's own point, di wrapped into
// (-ni/2, ni/2] on a periodic grid.  Padding entries: value 0, offset (0, 0).
struct Sell {
    std::vector<int64_t> off;      // nslices + 1
    bigvec<double> val;
    bigvec<int32_t> col;           // array indices (padding: the row's own index)
    int64_t entries() const { return (int64_t)val.size(); }
};

// ELL(K) + SELL overflow: the first kEll entries of every owned element's row
// at fixed slots val[e*kEll + m], col[e*kEll + m] (one 256-bit and one 128-bit load per element,
// no offset load: a pure stream), the remaining
// entries (rows longer than kEll) in a SELL-32 `ovf` whose slices are empty for most rows.
// Columns are ARRAY indices (owned element + pitch; halo rows allowed); padding = value 0 at the
// row's own index.
constexpr int kEll = 4;
struct Ell {
    int64_t n = 0;                 // owned elements
    bigvec<double> val;            // n * kEll (element-major)
    bigvec<int32_t> col;           // n * kEll
    bigvec<int16_t> col16;         // n * kEll: col - (own array index), when every slot fits (else empty)
    Sell ovf;
    int64_t entries() const { return (int64_t)val.size() + ovf.entries(); }
};


// Host product of setup: everything the device needs, in device layout.
struct Plan {
    int32_t ni = 0, nj = 0, periodic = 1, jb = 0, je = 0, rank = 0, nranks = 1;
    int32_t nloc = 0, pitch = 0;
    int32_t halo = 1;              // halo grid rows on each side of the owned rows
    int32_t halo_w = 0;            // halo-AINV across ranks: q / r rows received from the south
    int32_t halo_w_send = 0;       // ... q / r rows sent to the northern neighbour (= its halo_w)
    int32_t halo_t = 0;            // halo-AINV across ranks: t rows received from the north
    int32_t halo_t_send = 0;       // ... t rows the southern neighbour needs from this rank
    pcg_precond precond = PCG_PRECOND_AINV;
    int32_t fsai_q = 4;
    int32_t ainv_fill = 0;        // P_B2: entries kept per column of Zhat (0 = drop tolerance only)
    // AINV and FSAI share the factored form s = Z D^-1 Z^T r and every device path
    bool factored() const { return precond == PCG_PRECOND_AINV || precond == PCG_PRECOND_FSAI; }
    double tau = 0.1;
    int32_t flags = 0;
    bool has_sigma = false;
    int64_t n_owned = 0, first_global = 0, nnz_off = 0;
    // per-element arrays, (nloc + 2) * pitch
    bigvec<double> cE, cN, sigma, diag, piv;
    Ell Z, ZT;                     // rows of Z (for s = Z t) and of Z^T (for t = Z^T r)
    // FSAI (NEXT-1) DIA form when every chain link is an E-W neighbour pair: dia[m-1][e] =
    // zhat between owned element e - m and e (the column k = e's entry at row k - m), m = 1..dia_q;
    // 0 where the chain is shorter.  dia_q = 0: no DIA form (the ELL path applies the factor).
    int32_t dia_q = 0;
    std::vector<double> dia;
    // export (owned columns of Zhat, global unknown numbering); zrow / zhat are filled only with
    // keep_export (pcg_plan_build), not for pcg_setup, which never reads them
    bool keep_export = true;
    bigvec<int64_t> zcolptr;
    bigvec<int64_t> zrow;
    bigvec<double> zhat;
    bigvec<double> pivots, scale;
    double setup_s = 0.0;
    int64_t elements() const { return (int64_t)(nloc + 2 * halo) * pitch; }
    int64_t hoff() const { return (int64_t)halo * pitch; }   // array index of owned element 0
    int64_t owned_elements() const { return (int64_t)nloc * pitch; }
};

Status build_plan(const pcg_coeffs* c, const pcg_grid* g, const pcg_opts* o, Plan& plan);
Status partition_rows(int32_t ni, int32_t nj, const uint8_t* mask, int32_t parts, int32_t* rb);

// Library AINV on one row block (written independently of the oracle).
struct AinvBlock {
    // input: grid rows [row_lo, row_hi) form the index set; columns of rows >= row_own are kept
    int32_t row_lo = 0, row_own = 0, row_hi = 0;
    // output: owned columns, local unknown numbering of the block converted to GLOBAL grid
    // indices (j*ni + i) for rows, values zhat, pivots; failure column (global grid index)
    bigvec<int64_t> colptr;        // owned columns + 1
    bigvec<int64_t> row_g;         // grid index of each entry's row
    bigvec<double> zhat;
    bigvec<double> piv;            // per owned column
    bigvec<int64_t> col_g;         // grid index of each owned column
    int64_t fail_grid = -1;
};
void ainv_block(int32_t ni, int32_t nj, int32_t periodic, const double* cE, const double* cN,
                const double* sigma, const uint8_t* mask, double tau, int32_t fill, AinvBlock& blk, int threads = 1);
// NEXT-1 banded FSAI of T = band(A, 1) over the whole grid, as one factored block (fsai.cpp)
void fsai_block(int32_t ni, int32_t nj, int32_t periodic, const double* cE, const double* cN, const uint8_t* mask,
                int32_t q, const std::function<double(int64_t)>& diag_of, AinvBlock& blk);

}  // namespace pcg
