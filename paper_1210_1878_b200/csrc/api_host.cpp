// api_host.cpp -- C ABI of the host-only calls: row partition, setup plan (no GPU needed).
#include <cstring>
#include <string>

#include "internal.h"

namespace pcg {
void set_thread_error(const std::string& m);
}

struct pcg_plan {
    pcg::Plan p;
};

extern "C" {

pcg_status pcg_partition(int32_t ni, int32_t nj, const uint8_t* mask, int32_t parts, int32_t* row_begin) {
    pcg::Status s = pcg::partition_rows(ni, nj, mask, parts, row_begin);
    if (!s) pcg::set_thread_error(s.msg);
    return s.code;
}

pcg_status pcg_plan_build(const pcg_coeffs* coeffs, const pcg_grid* grid, const pcg_opts* opts, pcg_plan** out) {
    if (!out) return PCG_ERR_ARG;
    *out = nullptr;
    pcg_plan* pl = new (std::nothrow) pcg_plan();
    if (!pl) return PCG_ERR_NOMEM;
    pcg::Status s;
    try {
        s = pcg::build_plan(coeffs, grid, opts, pl->p);
    } catch (const std::bad_alloc&) {
        s = pcg::Status::err(PCG_ERR_NOMEM, "pcg_plan_build: out of host memory");
    }
    if (!s) {
        pcg::set_thread_error(s.msg);
        delete pl;
        return s.code;
    }
    *out = pl;
    return PCG_OK;
}

void pcg_plan_free(pcg_plan* plan) { delete plan; }

pcg_status pcg_plan_counts(const pcg_plan* plan, int64_t* c) {
    if (!plan || !c) return PCG_ERR_ARG;
    const pcg::Plan& P = plan->p;
    c[0] = P.n_owned;
    c[1] = (int64_t)P.zrow.size();
    c[2] = P.pitch;
    c[3] = P.Z.entries();      // ELL slots + overflow SELL entries
    c[4] = P.ZT.entries();
    c[5] = P.first_global;
    return PCG_OK;
}

pcg_status pcg_plan_export_zhat(const pcg_plan* plan, int64_t* colptr, int64_t* row, double* zhat,
                                double* pivots, double* scale) {
    if (!plan) return PCG_ERR_ARG;
    const pcg::Plan& P = plan->p;
    if (colptr && !P.zcolptr.empty()) std::memcpy(colptr, P.zcolptr.data(), P.zcolptr.size() * sizeof(int64_t));
    if (row && !P.zrow.empty()) std::memcpy(row, P.zrow.data(), P.zrow.size() * sizeof(int64_t));
    if (zhat && !P.zhat.empty()) std::memcpy(zhat, P.zhat.data(), P.zhat.size() * sizeof(double));
    if (pivots && !P.pivots.empty()) std::memcpy(pivots, P.pivots.data(), P.pivots.size() * sizeof(double));
    if (scale && !P.scale.empty()) std::memcpy(scale, P.scale.data(), P.scale.size() * sizeof(double));
    return PCG_OK;
}

}  // extern "C"
