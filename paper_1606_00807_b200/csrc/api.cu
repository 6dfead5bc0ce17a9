// Device side of the C-ABI (include/enkf_mc.h): map upload, workspace, stage launchers and
// the host-buffer entry point that assimilate_parallel binds (driver.py:159-253).

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "kernels.cuh"
#include "plan.h"

#define CK(expr)                                                                          \
    do {                                                                                  \
        cudaError_t _e = (expr);                                                          \
        if (_e != cudaSuccess) {                                                          \
            enkfmc_set_error(std::string("CUDA error: ") + cudaGetErrorString(_e) + " at " #expr); \
            return ENKFMC_E_CUDA;                                                         \
        }                                                                                 \
    } while (0)

struct DeviceState {
    int device = -1, sm_count = 0;
    size_t smem_limit = 0;
    // maps
    int64_t *tile_ptr = nullptr, *row_ptr = nullptr, *csc_ptr = nullptr, *csc_src = nullptr;
    int32_t *col_idx = nullptr, *csc_row = nullptr, *phys = nullptr, *iphys = nullptr, *bw = nullptr,
            *state_row = nullptr, *pred_state = nullptr, *work_order = nullptr, *tile_order = nullptr,
            *regress_order = nullptr, *alias_row = nullptr, *alias_rep = nullptr;
    int64_t *rq_ptr = nullptr, *band_ptr = nullptr;
    int32_t *row_tile = nullptr;
    int64_t band_stride = 0, band_fields = 0;
    double *band = nullptr;
    int64_t rq_stride = 0;
    double *Rq = nullptr;
    int64_t rq_alloc = 0;           // doubles the QR scratch holds
    uint8_t *is_interior = nullptr, *tile_mono = nullptr;
    int32_t *obs_slot = nullptr, *tile_nobs = nullptr;
    bool obs_current = false, orders_current = false;
    std::vector<cudaEvent_t> prof;   // 4 events per profiled analysis_device call
    size_t prof_used = 0;
    // workspace
    int64_t ws_nens = 0;
    // T / D / flags / band cover the owned tiles only: first owned local row, CSR position and band offset, and the field strides
    int64_t ws_row0 = 0, ws_nnz0 = 0, ws_rows = 0, ws_nnz = 0, ws_tb = -1, ws_te = -1;
    int64_t band_off0 = 0, band_own = 0, band_tb = -1, band_te = -1;
    double *U = nullptr, *T = nullptr, *D = nullptr, *scratch = nullptr;
    int32_t *flags = nullptr, *status = nullptr;
    unsigned int *counters = nullptr;
    unsigned int *worklist = nullptr;
    int64_t worklist_alloc = 0;
    SolveParams solve_layout{};
    int solve_grid = 0;
    // host-path staging
    double *dX = nullptr, *dXa = nullptr, *dR = nullptr, *dYs = nullptr;
    int64_t stage_nens = 0, stage_nobs = -1;
    cudaEvent_t ev[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
    cudaStream_t stream = nullptr, copy_stream = nullptr, down_stream = nullptr;   // kernels, uploads, downloads
    std::vector<cudaEvent_t> hev;    // events of the pipelined host path
};

void enkfmc_device_release(enkfmc_plan *p);

namespace {

template <class T>
int upload(T *&dst, const std::vector<T> &src) {
    if (dst) { cudaFree(dst); dst = nullptr; }
    const size_t bytes = std::max<size_t>(src.size(), 1) * sizeof(T);
    CK(cudaMalloc(&dst, bytes));
    if (!src.empty()) CK(cudaMemcpy(dst, src.data(), src.size() * sizeof(T), cudaMemcpyHostToDevice));
    return ENKFMC_OK;
}

template <class T>
void release(T *&p) { if (p) { cudaFree(p); p = nullptr; } }

int init_device(enkfmc_plan *p) {
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0) {
        enkfmc_set_error(std::string("no CUDA device available (") + cudaGetErrorString(e) +
                         "); libenkfmc has no CPU fallback");
        return ENKFMC_E_CUDA;
    }
    auto *d = new DeviceState();
    CK(cudaGetDevice(&d->device));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, d->device));
    if (prop.major < 10) {
        enkfmc_set_error("libenkfmc is built for sm_100a only; found sm_" + std::to_string(prop.major) +
                         std::to_string(prop.minor));
        delete d;
        return ENKFMC_E_CUDA;
    }
    d->sm_count = prop.multiProcessorCount;
    d->smem_limit = prop.sharedMemPerBlockOptin;
    p->dev = d;       // (ensure_device releases it again if anything below fails)
    int rc;
    if ((rc = upload(d->tile_ptr, p->tile_ptr))) return rc;
    if ((rc = upload(d->row_ptr, p->row_ptr))) return rc;
    if ((rc = upload(d->csc_ptr, p->csc_ptr))) return rc;
    if ((rc = upload(d->csc_src, p->csc_src))) return rc;
    if ((rc = upload(d->col_idx, p->col_idx))) return rc;
    if ((rc = upload(d->csc_row, p->csc_row))) return rc;
    if ((rc = upload(d->phys, p->phys))) return rc;
    if ((rc = upload(d->iphys, p->iphys))) return rc;
    if ((rc = upload(d->bw, p->bw))) return rc;
    if ((rc = upload(d->state_row, p->state_row))) return rc;
    if ((rc = upload(d->pred_state, p->pred_state))) return rc;
    if ((rc = upload(d->is_interior, p->is_interior))) return rc;
    if ((rc = upload(d->tile_mono, p->tile_mono))) return rc;
    if ((rc = upload(d->row_tile, p->row_tile))) return rc;
    {   // row-form band of every tile: [8 ceil(n/8)][8 (Wb + 1)], Wb = floor((b + 7) / 8)
        std::vector<int64_t> bp(p->ntiles + 1, 0);
        for (int64_t t = 0; t < p->ntiles; ++t)
            bp[t + 1] = bp[t] + ((p->tile_ptr[t + 1] - p->tile_ptr[t] + 7) / 8 * 8) * (int64_t)(8 * ((p->bw[t] + 7) / 8 + 1));
        d->band_stride = bp.back();
        if ((rc = upload(d->band_ptr, bp))) return rc;
    }
    CK(cudaMalloc(&d->counters, 16 * sizeof(unsigned int)));
    CK(cudaMemset(d->counters, 0, 16 * sizeof(unsigned int)));
    for (auto &ev : d->ev) CK(cudaEventCreate(&ev));
    CK(cudaStreamCreateWithFlags(&d->stream, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&d->copy_stream, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&d->down_stream, cudaStreamNonBlocking));
    return ENKFMC_OK;
}

// Device mirror of the plan, created on first use.  A failure part-way (out of memory) leaves no half-initialised state
// behind: the next call starts from scratch instead of launching with null buffers.
int ensure_device(enkfmc_plan *p) {
    if (p->dev) return ENKFMC_OK;
    const int rc = init_device(p);
    if (rc != ENKFMC_OK && p->dev) enkfmc_device_release(p);
    return rc;
}

int ensure_orders(enkfmc_plan *p) {
    DeviceState *d = p->dev;
    if (d->orders_current) return ENKFMC_OK;
    int rc;
    if ((rc = upload(d->work_order, p->work_order))) return rc;
    if ((rc = upload(d->tile_order, p->tile_order))) return rc;
    if ((rc = upload(d->regress_order, p->regress_order))) return rc;
    if ((rc = upload(d->alias_row, p->alias_row))) return rc;
    if ((rc = upload(d->alias_rep, p->alias_rep))) return rc;
    if ((rc = upload(d->rq_ptr, p->rq_ptr))) return rc;
    d->rq_stride = p->rq_ptr.empty() ? 0 : p->rq_ptr.back();
    d->orders_current = true;
    return ENKFMC_OK;
}

int ensure_obs(enkfmc_plan *p) {
    DeviceState *d = p->dev;
    if (d->obs_current) return ENKFMC_OK;
    if (!p->have_obs) { enkfmc_set_error("observations not set on this plan"); return ENKFMC_E_VALUE; }
    int rc;
    if ((rc = upload(d->obs_slot, p->obs_slot))) return rc;
    if ((rc = upload(d->tile_nobs, p->tile_nobs))) return rc;
    d->obs_current = true;
    return ENKFMC_OK;
}

int check_nens(int64_t nens) {
    if (nens < 2) {
        enkfmc_set_error("ensemble size must be at least 2, got " + std::to_string(nens));
        return ENKFMC_E_CONFIG;
    }
    if (nens > ENKFMC_MAX_NENS) {
        enkfmc_set_error("ensemble size " + std::to_string(nens) + " exceeds the kernel cap " +
                         std::to_string(ENKFMC_MAX_NENS));
        return ENKFMC_E_CAPACITY;
    }
    return ENKFMC_OK;
}

// Solve-stage layout (scratch, window placement) for a given ensemble size.
int ensure_solve_layout(enkfmc_plan *p, int64_t nens) {
    DeviceState *d = p->dev;
    if (d->scratch && d->solve_layout.N == (int)nens) return ENKFMC_OK;
    release(d->scratch);
    SolveParams &L = d->solve_layout;
    L = SolveParams{};
    L.N = (int)nens;
    L.bmax = (int)p->max_bw;
    L.nfields = (int)p->nfields;
    L.ntiles = (int)p->ntiles;
    L.ntiles_owned = (int)p->ntiles;
    const int64_t stride = solve_plan_scratch(L, std::max<int64_t>(p->max_nlocal, 1), d->smem_limit);
    d->solve_grid = solve_grid_size(d->sm_count, L, d->smem_limit);
    CK(cudaMalloc(&d->scratch, (size_t)stride * d->solve_grid * sizeof(double)));
    return ENKFMC_OK;
}

// Band / Cholesky-factor buffer: as many fields per launch pair as fit in the budget (16 GiB).
int ensure_band(enkfmc_plan *p) {
    DeviceState *d = p->dev;
    const int64_t budget = (int64_t)16 << 30;
    if (d->band_tb != p->tile_begin || d->band_te != p->tile_end) {   // the owned tiles' share of the band
        std::vector<int64_t> bp((size_t)p->ntiles + 1);
        CK(cudaMemcpy(bp.data(), d->band_ptr, bp.size() * sizeof(int64_t), cudaMemcpyDeviceToHost));
        d->band_off0 = bp[(size_t)p->tile_begin];
        d->band_own = bp[(size_t)p->tile_end] - bp[(size_t)p->tile_begin];
        d->band_tb = p->tile_begin;
        d->band_te = p->tile_end;
        d->band_fields = 0;
    }
    const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(p->nfields, budget / std::max<int64_t>(8 * d->band_own, 1)));
    if (d->band && d->band_fields >= chunk) return ENKFMC_OK;
    release(d->band);
    CK(cudaMalloc(&d->band, std::max<size_t>((size_t)chunk * d->band_own, 1) * sizeof(double)));
    d->band_fields = chunk;
    return ENKFMC_OK;
}

int ensure_workspace(enkfmc_plan *p, int64_t nens) {
    DeviceState *d = p->dev;
    if (d->ws_nens == nens && d->U && d->ws_tb == p->tile_begin && d->ws_te == p->tile_end) return ENKFMC_OK;
    release(d->U); release(d->T); release(d->D); release(d->flags); release(d->status);
    const int64_t nstate = p->nstate2d * p->nfields;
    // factors of the owned tiles only (one rank's share): contiguous local rows, contiguous CSR positions
    d->ws_row0 = p->tile_ptr[(size_t)p->tile_begin];
    d->ws_rows = p->tile_ptr[(size_t)p->tile_end] - d->ws_row0;
    d->ws_nnz0 = p->row_ptr[(size_t)d->ws_row0];
    d->ws_nnz = p->row_ptr[(size_t)(d->ws_row0 + d->ws_rows)] - d->ws_nnz0;
    CK(cudaMalloc(&d->U, std::max<size_t>(1, (size_t)nstate * nens) * sizeof(double)));
    CK(cudaMalloc(&d->T, std::max<size_t>(1, (size_t)d->ws_nnz * p->nfields) * sizeof(double)));
    CK(cudaMalloc(&d->D, std::max<size_t>(1, (size_t)d->ws_rows * p->nfields) * sizeof(double)));
    CK(cudaMalloc(&d->flags, std::max<size_t>(1, (size_t)d->ws_rows * p->nfields) * sizeof(int32_t)));
    CK(cudaMalloc(&d->status, std::max<size_t>(1, (size_t)p->ntiles * p->nfields) * sizeof(int32_t)));
    d->ws_nens = nens;
    d->ws_tb = p->tile_begin;
    d->ws_te = p->tile_end;
    return ENKFMC_OK;
}

// fields [fbeg, fend) (fend < 0: all)
// d_T / d_D / d_flags are indexed by the plan's global CSR position / local row with field strides tstride / dstride:
// caller-owned full-size buffers (tstride = nnz, dstride = sum_nlocal) or the plan's workspace, biased by the first owned
// position (own = true).
int do_regress(enkfmc_plan *p, const double *d_U, int64_t nens, double rank_tol, double floor_, double *d_T,
               double *d_D, int32_t *d_flags, cudaStream_t s, cudaEvent_t mid = nullptr, int64_t fbeg = 0,
               int64_t fend = -1, bool own = false) {
    if (fend < 0) fend = p->nfields;
    const int64_t tstride = own ? p->dev->ws_nnz : p->nnz(), dstride = own ? p->dev->ws_rows : p->sum_nlocal();
    if (own) {
        d_T -= p->dev->ws_nnz0;
        d_D -= p->dev->ws_row0;
        if (d_flags) d_flags -= p->dev->ws_row0;
    }
    DeviceState *d = p->dev;
    int rc0 = ensure_orders(p);
    if (rc0) return rc0;
    RegressParams R{};
    R.U = d_U; R.N = (int)nens; R.ld = (int)nens | 1; R.pmax = (int)std::max<int64_t>(p->max_pred, 1);
    R.nfields = (int)p->nfields; R.nloc = p->sum_nlocal(); R.nnz = p->nnz(); R.nstate2d = p->nstate2d;
    R.nwork = (int64_t)p->regress_order.size() * p->nfields;
    R.row_ptr = d->row_ptr; R.pred_state = d->pred_state; R.state_row = d->state_row; R.work_order = d->regress_order;
    R.rank_tol = rank_tol; R.variance_floor = floor_; R.fast_ratio = 1e-6;
    R.T = d_T; R.D = d_D; R.flags = d_flags; R.tstride = tstride; R.dstride = dstride; R.counter = d->counters; R.lcounter = d->counters + 8;
    R.rq_ptr = d->rq_ptr; R.rq_stride = d->rq_stride;
    // QR scratch: as many fields per launch pair as fit in the budget (default 16 GiB)
    const int64_t budget = (int64_t)16 << 30;
    int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(p->nfields, budget / std::max<int64_t>(8 * d->rq_stride, 1)));
    if (!d->Rq || d->rq_alloc < chunk * d->rq_stride) {
        release(d->Rq);
        CK(cudaMalloc(&d->Rq, std::max<size_t>((size_t)chunk * d->rq_stride, 1) * sizeof(double)));
        d->rq_alloc = chunk * d->rq_stride;
    }
    R.Rq = d->Rq;
    const int64_t list_need = (int64_t)p->regress_order.size() * chunk;
    if (!d->worklist || d->worklist_alloc < list_need) {
        release(d->worklist);
        CK(cudaMalloc(&d->worklist, std::max<size_t>((size_t)list_need, 1) * 2 * sizeof(unsigned int)));
        d->worklist_alloc = list_need;
    }
    R.worklist = d->worklist;
    R.worklist2 = d->worklist + std::max<int64_t>(list_need, 1);
    for (int64_t f0 = fbeg; f0 < fend; f0 += chunk) {
        R.f0 = (int)f0;
        R.f1 = (int)std::min<int64_t>(fend, f0 + chunk);
        R.nwork = (int64_t)p->regress_order.size() * (R.f1 - R.f0);
        if (R.nwork > 0xfffffff0LL) { enkfmc_set_error("too many regressions for one launch"); return ENKFMC_E_CAPACITY; }
        cudaError_t e = launch_regress(R, d->sm_count, d->smem_limit, s, mid);
        if (e == cudaErrorInvalidConfiguration) {
            enkfmc_set_error("regression workspace (nens=" + std::to_string(nens) + ", predecessors=" +
                             std::to_string(p->max_pred) + ") exceeds shared memory or the 128-predecessor cap");
            return ENKFMC_E_CAPACITY;
        }
        CK(e);
        if (R.nwork > 0) p->counters[0] += 4;
    }
    if (!p->alias_row.empty()) {   // copy each distinct regression to the other tiles holding the same row
        CK(launch_replicate_rows(d->alias_row, d->alias_rep, (int64_t)p->alias_row.size(), d->row_ptr, fend - fbeg,
                                 tstride, dstride, d_T + fbeg * tstride, d_D + fbeg * dstride,
                                 d_flags ? d_flags + fbeg * dstride : nullptr, s));
        p->counters[0] += 1;
    }
    return ENKFMC_OK;
}

int do_solve(enkfmc_plan *p, const double *d_X, const double *d_T, const double *d_D, const double *d_r,
             const double *d_Ys, int64_t nens, double *d_Xa, int32_t *d_status, cudaStream_t s, int64_t fbeg = 0,
             int64_t fend = -1, bool own = false) {
    if (fend < 0) fend = p->nfields;
    if (own) { d_T -= p->dev->ws_nnz0; d_D -= p->dev->ws_row0; }
    DeviceState *d = p->dev;
    int rc = ensure_obs(p);
    if (rc) return rc;
    if ((rc = ensure_solve_layout(p, nens))) return rc;
    if ((rc = ensure_orders(p))) return rc;
    SolveParams S = d->solve_layout;
    S.ntiles_owned = (int)p->tile_order.size();
    S.X = d_X; S.T = d_T; S.D = d_D; S.rdiag = d_r; S.Ys = d_Ys; S.Xa = d_Xa;
    S.nloc = p->sum_nlocal(); S.nnz = p->nnz(); S.nstate2d = p->nstate2d;
    S.tstride = own ? d->ws_nnz : p->nnz(); S.dstride = own ? d->ws_rows : p->sum_nlocal();
    S.tile_ptr = d->tile_ptr; S.row_ptr = d->row_ptr; S.csc_ptr = d->csc_ptr; S.csc_src = d->csc_src;
    S.col_idx = d->col_idx; S.csc_row = d->csc_row; S.phys = d->phys; S.iphys = d->iphys; S.bw = d->bw;
    S.state_row = d->state_row; S.obs_slot = d->obs_slot; S.tile_nobs = d->tile_nobs; S.tile_order = d->tile_order;
    S.is_interior = d->is_interior; S.tile_mono = d->tile_mono; S.scratch = d->scratch; S.status = d_status; S.counter = d->counters + 2;
    S.band_ptr = d->band_ptr; S.row_tile = d->row_tile; S.work_order = d->work_order;
    S.nrows_owned = (int64_t)p->work_order.size();
    S.asm_nmax = (int)p->max_nlocal;
    S.asm_nnzmax = 0;
    for (int64_t t = 0; t < p->ntiles; ++t)
        S.asm_nnzmax = std::max<int>(S.asm_nnzmax, (int)(p->row_ptr[p->tile_ptr[t + 1]] - p->row_ptr[p->tile_ptr[t]]));
    S.all_mono = 1;
    for (uint8_t m : p->tile_mono) if (!m) S.all_mono = 0;
    int rc2 = ensure_band(p);
    if (rc2) return rc2;
    S.band = d->band - d->band_off0;          // band_ptr[t] counts from tile 0: biased by the first owned tile's offset
    S.band_stride = d->band_own;
    if (fbeg == 0) CK(cudaMemsetAsync(d->counters + 3, 0, sizeof(unsigned int), s));   // clamped-pivot counter
    for (int64_t f0 = fbeg; f0 < fend; f0 += d->band_fields) {
        S.f0 = (int)f0;
        S.f1 = (int)std::min<int64_t>(fend, f0 + d->band_fields);
        cudaError_t e = launch_assemble_band(S, d->sm_count, d->smem_limit, s);
        if (e == cudaSuccess) e = launch_local_solve(S, d->solve_grid, d->smem_limit, s);
        if (e == cudaErrorInvalidConfiguration) {
            enkfmc_set_error("local-solve window (half-bandwidth " + std::to_string(p->max_bw) + ") exceeds shared memory");
            return ENKFMC_E_CAPACITY;
        }
        CK(e);
        p->counters[0] += 2;
    }
    return ENKFMC_OK;
}

// Reads the per-tile status words of the last analysis (0 ok, 1 not positive definite, 2 non-finite) and the clamped-pivot
// count; a failed tile becomes ENKFMC_E_NUMERIC naming the sub-domain (kernels.py:194-195).  Synchronises.
int scan_status(enkfmc_plan *p) {
    DeviceState *d = p->dev;
    CK(cudaDeviceSynchronize());
    unsigned int clamped = 0;
    CK(cudaMemcpy(&clamped, d->counters + 3, sizeof(unsigned int), cudaMemcpyDeviceToHost));
    p->counters[5] = clamped;
    std::vector<int32_t> st((size_t)(p->ntiles * p->nfields));
    if (!st.empty()) CK(cudaMemcpy(st.data(), d->status, st.size() * sizeof(int32_t), cudaMemcpyDeviceToHost));
    p->counters[4] = -1;
    for (size_t it = 0; it < st.size(); ++it) {
        if (st[it] != 0) {
            const int64_t f = (int64_t)it / p->ntiles, t = (int64_t)it % p->ntiles;
            p->counters[4] = (int64_t)it;
            enkfmc_set_error("primal analysis solve failed in subdomain " + std::to_string(t) + " (field " +
                             std::to_string(f) + "): " +
                             (st[it] == 1 ? "matrix not positive definite" : st[it] == 2 ? "non-finite pivot" : "non-finite solution"));
            return ENKFMC_E_NUMERIC;
        }
    }
    return ENKFMC_OK;
}

}  // namespace

void enkfmc_device_invalidate_obs(enkfmc_plan *p) { if (p->dev) p->dev->obs_current = false; }
void enkfmc_device_invalidate_orders(enkfmc_plan *p) { if (p->dev) p->dev->orders_current = false; }

void enkfmc_device_release(enkfmc_plan *p) {
    DeviceState *d = p->dev;
    if (!d) return;
    release(d->tile_ptr); release(d->row_ptr); release(d->csc_ptr); release(d->csc_src); release(d->col_idx);
    release(d->csc_row); release(d->phys); release(d->iphys); release(d->bw); release(d->state_row);
    release(d->pred_state); release(d->regress_order); release(d->alias_row); release(d->alias_rep); release(d->work_order); release(d->tile_order); release(d->is_interior); release(d->tile_mono);
    release(d->obs_slot); release(d->tile_nobs); release(d->U); release(d->T); release(d->D); release(d->scratch);
    release(d->flags); release(d->status); release(d->counters); release(d->rq_ptr); release(d->Rq); release(d->worklist); release(d->band_ptr); release(d->band); release(d->row_tile); release(d->dX); release(d->dXa); release(d->dR);
    release(d->dYs);
    for (auto &ev : d->ev) if (ev) cudaEventDestroy(ev);
    for (auto &ev : d->hev) cudaEventDestroy(ev);
    if (d->copy_stream) cudaStreamDestroy(d->copy_stream);
    if (d->down_stream) cudaStreamDestroy(d->down_stream);
    for (auto &ev : d->prof) cudaEventDestroy(ev);
    if (d->stream) cudaStreamDestroy(d->stream);
    delete d;
    p->dev = nullptr;
}

extern "C" int enkfmc_center_rows(const double *d_X, double *d_U, int64_t nrows, int64_t nens, void *stream) {
    int rc = check_nens(nens);
    if (rc) return rc;
    CK(launch_center_rows(d_X, d_U, nrows, (int)nens, (cudaStream_t)stream));
    return ENKFMC_OK;
}

extern "C" int enkfmc_regress(enkfmc_plan *p, const double *d_U, int64_t nens, double rank_tol, double floor_,
                              double *d_T, double *d_D, int32_t *d_flags, void *stream) {
    int rc = check_nens(nens);
    if (rc) return rc;
    if ((rc = ensure_device(p))) return rc;
    return do_regress(p, d_U, nens, rank_tol, floor_, d_T, d_D, d_flags, (cudaStream_t)stream);
}

extern "C" int enkfmc_local_solve(enkfmc_plan *p, const double *d_X, const double *d_T, const double *d_D,
                                  const double *d_r, const double *d_Ys, int64_t nens, double *d_Xa,
                                  int32_t *d_status, void *stream) {
    int rc = check_nens(nens);
    if (rc) return rc;
    if ((rc = ensure_device(p))) return rc;
    return do_solve(p, d_X, d_T, d_D, d_r, d_Ys, nens, d_Xa, d_status, (cudaStream_t)stream);
}

extern "C" int enkfmc_analysis_device(enkfmc_plan *p, const double *d_X, const double *d_r, const double *d_Ys,
                                      int64_t nens, double rank_tol, double floor_, double *d_Xa, void *stream) {
    int rc = check_nens(nens);
    if (rc) return rc;
    if ((rc = ensure_device(p))) return rc;
    if ((rc = ensure_workspace(p, nens))) return rc;
    DeviceState *d = p->dev;
    cudaStream_t s = (cudaStream_t)stream;
    cudaEvent_t *ev = nullptr;
    if (p->profile) {
        while (d->prof.size() < d->prof_used + 5) {
            cudaEvent_t e;
            CK(cudaEventCreate(&e));
            d->prof.push_back(e);
        }
        ev = d->prof.data() + d->prof_used;
        d->prof_used += 5;
        CK(cudaEventRecord(ev[0], s));
    }
    CK(cudaMemsetAsync(d->status, 0, std::max<size_t>(1, (size_t)p->ntiles * p->nfields) * sizeof(int32_t), s));
    CK(launch_center_rows(d_X, d->U, p->nstate2d * p->nfields, (int)nens, s));
    p->counters[0] += 1;
    if (ev) CK(cudaEventRecord(ev[1], s));
    if ((rc = do_regress(p, d->U, nens, rank_tol, floor_, d->T, d->D, d->flags, s, ev ? ev[2] : nullptr, 0, -1, true))) return rc;
    if (ev) CK(cudaEventRecord(ev[3], s));
    rc = do_solve(p, d_X, d->T, d->D, d_r, d_Ys, nens, d_Xa, d->status, s, 0, -1, true);
    if (ev) CK(cudaEventRecord(ev[4], s));
    return rc;
}

extern "C" int enkfmc_plan_check_status(enkfmc_plan *p) {
    if (!p->dev || !p->dev->status) return ENKFMC_OK;
    return scan_status(p);
}

extern "C" int enkfmc_plan_profile(enkfmc_plan *p, int enable) {
    p->profile = enable != 0;
    if (p->dev) p->dev->prof_used = 0;
    return ENKFMC_OK;
}

extern "C" int enkfmc_plan_stage_times(enkfmc_plan *p, int64_t *ncalls, double *ms3) {
    ms3[0] = ms3[1] = ms3[2] = ms3[3] = 0.0;
    *ncalls = 0;
    if (!p->dev) return ENKFMC_OK;
    DeviceState *d = p->dev;
    CK(cudaDeviceSynchronize());
    for (size_t k = 0; k + 5 <= d->prof_used; k += 5) {
        for (int st = 0; st < 4; ++st) {
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, d->prof[k + st], d->prof[k + st + 1]));
            ms3[st] += ms;
        }
        ++*ncalls;
    }
    return ENKFMC_OK;
}

extern "C" int enkfmc_fp64_peak(double *tflops, void *stream) {
    int dev = 0;
    CK(cudaGetDevice(&dev));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, dev));
    cudaStream_t s = (cudaStream_t)stream;
    double *out = nullptr;
    CK(cudaMalloc(&out, sizeof(double)));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    const int iters = 4096;
    double best = 0.0;
    for (int rep = 0; rep < 6; ++rep) {
        CK(cudaEventRecord(a, s));
        CK(launch_fp64_peak(out, iters, prop.multiProcessorCount, s));
        CK(cudaEventRecord(b, s));
        CK(cudaEventSynchronize(b));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, a, b));
        const double flops = 2.0 * 64.0 * iters * 256.0 * prop.multiProcessorCount * 8.0;
        if (rep > 0) best = std::max(best, flops / (ms * 1e-3) * 1e-12);
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(out);
    *tflops = best;
    return ENKFMC_OK;
}

extern "C" int enkfmc_fp64_mma_peak(double *tflops, void *stream) {
    int dev = 0;
    CK(cudaGetDevice(&dev));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, dev));
    cudaStream_t s = (cudaStream_t)stream;
    double *out = nullptr;
    CK(cudaMalloc(&out, sizeof(double)));
    cudaEvent_t a, b;
    CK(cudaEventCreate(&a));
    CK(cudaEventCreate(&b));
    const int iters = 2048;
    double best = 0.0;
    for (int rep = 0; rep < 6; ++rep) {
        CK(cudaEventRecord(a, s));
        CK(launch_dmma_peak(out, iters, prop.multiProcessorCount, s));
        CK(cudaEventRecord(b, s));
        CK(cudaEventSynchronize(b));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, a, b));
        // 8 tiles x (8*8*4 FMA) per warp per iteration, 8 warps per block, 8 blocks per SM
        const double flops = 2.0 * 8.0 * 256.0 * iters * 8.0 * prop.multiProcessorCount * 8.0;
        if (rep > 0) best = std::max(best, flops / (ms * 1e-3) * 1e-12);
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    cudaFree(out);
    *tflops = best;
    return ENKFMC_OK;
}

extern "C" int enkfmc_analysis_host(enkfmc_plan *p, const double *X, const double *r_diag, const double *Ys,
                                    int64_t nens, double rank_tol, double floor_, double *Xa, double *timings_ms) {
    int rc = check_nens(nens);
    if (rc) return rc;
    if ((rc = ensure_device(p))) return rc;
    if ((rc = ensure_workspace(p, nens))) return rc;
    DeviceState *d = p->dev;
    const int64_t nstate = p->nstate2d * p->nfields;
    const size_t xbytes = (size_t)nstate * nens * sizeof(double);
    if (d->stage_nens != nens || !d->dX) {
        release(d->dX); release(d->dXa);
        CK(cudaMalloc(&d->dX, std::max<size_t>(xbytes, 8)));
        CK(cudaMalloc(&d->dXa, std::max<size_t>(xbytes, 8)));
        d->stage_nens = nens;
        d->stage_nobs = -1;
    }
    if (d->stage_nobs != p->nobs) {
        release(d->dR); release(d->dYs);
        CK(cudaMalloc(&d->dR, std::max<size_t>((size_t)p->nobs, 1) * sizeof(double)));
        CK(cudaMalloc(&d->dYs, std::max<size_t>((size_t)p->nobs * nens, 1) * sizeof(double)));
        d->stage_nobs = p->nobs;
    }
    // Pipelined over groups of fields: the copy stream uploads group g + 1 and downloads the analysis of group
    // g - 1 while the compute stream works on group g (fields are independent: PAPER.md:201).
    cudaStream_t s = d->stream, cs = d->copy_stream, ds = d->down_stream;
    // tiles outside the owned range are never written: start every analysis from a clean status array
    CK(cudaMemsetAsync(d->status, 0, std::max<size_t>(1, (size_t)p->ntiles * p->nfields) * sizeof(int32_t), s));
    // Five groups for a dozen fields or more, the first and the last small (the kernels start after a short upload and
    // only a short download is exposed; smaller groups than this cost more in kernel tails than they hide).
    std::vector<int64_t> cuts;
    {
        const int64_t nf = p->nfields;
        // ordinary (pageable) host arrays: a staged copy blocks the host, smaller groups start the device earlier and keep the
        // staging of the next group under its kernels (measured on cfg3: 75 ms with 5 groups, 66 ms with 12; page-locked: 61 / 64)
        bool pinned = false;
        {
            cudaPointerAttributes attr;
            if (cudaPointerGetAttributes(&attr, X) == cudaSuccess) pinned = attr.type == cudaMemoryTypeHost;
            else cudaGetLastError();
        }
        int64_t ng = nf >= 12 ? (pinned ? 5 : 12) : std::min<int64_t>(nf, 4);
        if (const char *genv = getenv("ENKFMC_HOST_GROUPS")) ng = std::max<int64_t>(1, std::min<int64_t>(nf, atoi(genv)));
        const int64_t edge = ng >= 3 ? std::max<int64_t>(1, nf / (4 * ng)) : 0;   // fields in the edge groups
        for (int64_t g = 0; g <= ng; ++g) {
            if (ng < 3) cuts.push_back(nf * g / ng);
            else if (g == 0) cuts.push_back(0);
            else if (g == ng) cuts.push_back(nf);
            else cuts.push_back(edge + (nf - 2 * edge) * (g - 1) / (ng - 2));
        }
    }
    const int ngroups = (int)cuts.size() - 1;
    // observations are sorted by state index, hence by field: the rows of Ys / r_diag each group needs are contiguous
    std::vector<int64_t> ocut((size_t)ngroups + 1, 0);
    for (int g = 0; g <= ngroups; ++g)
        ocut[(size_t)g] = std::lower_bound(p->obs_indices.begin(), p->obs_indices.end(), cuts[(size_t)g] * p->nstate2d) -
                          p->obs_indices.begin();
    const size_t need_ev = 2 + 8 * (size_t)ngroups;
    while (d->hev.size() < need_ev) { cudaEvent_t e; CK(cudaEventCreate(&e)); d->hev.push_back(e); }
    cudaEvent_t evY0 = d->hev[0], evY1 = d->hev[1];
    auto EV = [&](int g, int k) { return d->hev[2 + 8 * (size_t)g + k]; };   // 0,1 X up; 7 Ys up; 2,3,4 compute; 5,6 down
    const size_t rowbytes = (size_t)nens * sizeof(double);
    auto fcut = [&](int g) { return cuts[(size_t)g]; };
    // Issue order: upload g + 1 and download g - 1 are queued right after the kernels of group g.  With page-locked host
    // arrays every call returns at once and the order is immaterial; with ordinary (pageable) arrays a copy blocks the host
    // while it is staged, and this order lets the staging of the neighbouring groups run while the device computes group g.
    auto upload_group = [&](int g) -> int {
        const size_t r0 = (size_t)fcut(g) * p->nstate2d, r1 = (size_t)fcut(g + 1) * p->nstate2d;
        CK(cudaEventRecord(EV(g, 0), cs));
        CK(cudaMemcpyAsync(d->dX + r0 * nens, X + r0 * nens, (r1 - r0) * rowbytes, cudaMemcpyHostToDevice, cs));
        CK(cudaEventRecord(EV(g, 1), cs));
        if (g == 0) {   // r_diag is small and usually in pageable memory (a staged, host-blocking copy): once, up front
            CK(cudaEventRecord(evY0, cs));
            if (p->nobs) CK(cudaMemcpyAsync(d->dR, r_diag, (size_t)p->nobs * sizeof(double), cudaMemcpyHostToDevice, cs));
        }
        const int64_t o0 = ocut[(size_t)g], o1 = ocut[(size_t)g + 1];
        if (o1 > o0)
            CK(cudaMemcpyAsync(d->dYs + o0 * nens, Ys + o0 * nens, (size_t)(o1 - o0) * rowbytes, cudaMemcpyHostToDevice, cs));
        CK(cudaEventRecord(EV(g, 7), cs));
        if (g == ngroups - 1) CK(cudaEventRecord(evY1, cs));
        return ENKFMC_OK;
    };
    auto download_group = [&](int g) -> int {
        const size_t r0 = (size_t)fcut(g) * p->nstate2d, r1 = (size_t)fcut(g + 1) * p->nstate2d;
        CK(cudaStreamWaitEvent(ds, EV(g, 4), 0));
        CK(cudaEventRecord(EV(g, 5), ds));
        CK(cudaMemcpyAsync(Xa + r0 * nens, d->dXa + r0 * nens, (r1 - r0) * rowbytes, cudaMemcpyDeviceToHost, ds));
        CK(cudaEventRecord(EV(g, 6), ds));
        return ENKFMC_OK;
    };
    auto drain = [&]() { cudaStreamSynchronize(cs); cudaStreamSynchronize(ds); cudaStreamSynchronize(s); };
    if ((rc = upload_group(0))) { drain(); return rc; }
    for (int g = 0; g < ngroups; ++g) {
        const int64_t f0 = fcut(g), f1 = fcut(g + 1);
        const size_t r0 = (size_t)f0 * p->nstate2d, r1 = (size_t)f1 * p->nstate2d;
        CK(cudaStreamWaitEvent(s, EV(g, 1), 0));
        CK(cudaEventRecord(EV(g, 2), s));
        CK(launch_center_rows(d->dX + r0 * nens, d->U + r0 * nens, (int64_t)(r1 - r0), (int)nens, s));
        p->counters[0] += 1;
        if ((rc = do_regress(p, d->U, nens, rank_tol, floor_, d->T, d->D, d->flags, s, nullptr, f0, f1, true))) { drain(); return rc; }
        CK(cudaEventRecord(EV(g, 3), s));
        CK(cudaStreamWaitEvent(s, EV(g, 7), 0));
        if (p->tile_begin != 0 || p->tile_end != p->ntiles)   // a rank's share: rows it does not own come back as the background
            CK(cudaMemcpyAsync(d->dXa + r0 * nens, d->dX + r0 * nens, (r1 - r0) * rowbytes, cudaMemcpyDeviceToDevice, s));
        if ((rc = do_solve(p, d->dX, d->T, d->D, d->dR, d->dYs, nens, d->dXa, d->status, s, f0, f1, true))) { drain(); return rc; }
        CK(cudaEventRecord(EV(g, 4), s));
        if (g + 1 < ngroups && (rc = upload_group(g + 1))) { drain(); return rc; }
        if (g >= 1 && (rc = download_group(g - 1))) { drain(); return rc; }
    }
    if ((rc = download_group(ngroups - 1))) { drain(); return rc; }
    CK(cudaStreamSynchronize(ds));
    CK(cudaStreamSynchronize(cs));
    CK(cudaStreamSynchronize(s));
    if (timings_ms) {   // busy time of each stage, summed over the groups (the stages overlap in wall-clock time)
        auto span = [&](cudaEvent_t a, cudaEvent_t b, double &acc) {
            float ms = 0.f;
            cudaError_t e = cudaEventElapsedTime(&ms, a, b);
            if (e == cudaSuccess) acc += ms;
            return e;
        };
        timings_ms[0] = timings_ms[1] = timings_ms[2] = timings_ms[3] = 0.0;
        (void)evY0; (void)evY1;
        for (int g = 0; g < ngroups; ++g) {
            CK(span(EV(g, 0), EV(g, 7), timings_ms[0]));
            CK(span(EV(g, 2), EV(g, 3), timings_ms[1]));
            CK(span(EV(g, 3), EV(g, 4), timings_ms[2]));
            CK(span(EV(g, 5), EV(g, 6), timings_ms[3]));
        }
    }
    if ((rc = scan_status(p))) return rc;
    return ENKFMC_OK;
}

extern "C" int64_t enkfmc_plan_counter(const enkfmc_plan *p, int what) {
    if (what < 0 || what >= 8) return -1;
    return p->counters[what];
}

extern "C" void *enkfmc_plan_device_buffer(const enkfmc_plan *p, int what) {
    if (!p->dev) return nullptr;
    switch (what) {
        case 0: return p->dev->U;
        case 1: return p->dev->T;
        case 2: return p->dev->D;
        case 3: return p->dev->flags;
        case 4: return p->dev->status;
        default: return nullptr;
    }
}

extern "C" int enkfmc_scatter_rows(double *d_dst, const int64_t *d_dst_rows, const double *d_src,
                                   const int64_t *d_src_rows, int64_t nrows, int64_t nens, void *stream) {
    if (nens < 1) { enkfmc_set_error("nens must be positive"); return ENKFMC_E_VALUE; }
    CK(launch_scatter_rows(d_dst, d_dst_rows, d_src, d_src_rows, nrows, (int)nens, (cudaStream_t)stream));
    return ENKFMC_OK;
}

extern "C" int enkfmc_assemble_band(enkfmc_plan *p, const double *d_T, const double *d_D, int64_t tile,
                                    double *d_band, void *stream) {
    if (p->ntiles != 1 || p->nfields != 1 || tile != 0) {
        enkfmc_set_error("assemble_band needs a single-tile, single-field plan");
        return ENKFMC_E_VALUE;
    }
    int rc = ensure_device(p);
    if (rc) return rc;
    if ((rc = ensure_orders(p))) return rc;
    DeviceState *d = p->dev;
    SolveParams S{};
    S.T = d_T; S.D = d_D; S.nfields = 1; S.ntiles = 1; S.ntiles_owned = 1; S.bmax = (int)p->max_bw;
    S.nloc = p->sum_nlocal(); S.nnz = p->nnz(); S.nstate2d = p->nstate2d;
    S.tstride = p->nnz(); S.dstride = p->sum_nlocal();
    S.tile_ptr = d->tile_ptr; S.row_ptr = d->row_ptr; S.csc_ptr = d->csc_ptr; S.csc_src = d->csc_src;
    S.col_idx = d->col_idx; S.csc_row = d->csc_row; S.phys = d->phys; S.bw = d->bw;
    S.band_ptr = d->band_ptr; S.band_stride = d->band_stride; S.row_tile = d->row_tile; S.work_order = d->work_order;
    S.nrows_owned = (int64_t)p->work_order.size();
    S.assemble_only = 1; S.f0 = 0; S.f1 = 1; S.band = d_band;
    S.tile_order = d->tile_order; S.tile_mono = d->tile_mono; S.asm_nmax = (int)p->max_nlocal; S.asm_nnzmax = (int)std::min<int64_t>(p->nnz(), 1 << 30);
    S.all_mono = 1;
    for (uint8_t m : p->tile_mono) if (!m) S.all_mono = 0;
    {
        cudaError_t e = launch_assemble_band(S, d->sm_count, d->smem_limit, (cudaStream_t)stream);
        if (e == cudaErrorInvalidConfiguration) {
            enkfmc_set_error("band of half-bandwidth " + std::to_string(p->max_bw) + " exceeds shared memory");
            return ENKFMC_E_CAPACITY;
        }
        CK(e);
    }
    p->counters[0] += 1;
    return ENKFMC_OK;
}

extern "C" int enkfmc_precision_apply(enkfmc_plan *p, const double *d_T, const double *d_D, const double *d_V,
                                      int64_t ncols, double *d_tmp, double *d_out, void *stream) {
    if (p->ntiles != 1 || p->nfields != 1) {
        enkfmc_set_error("precision_apply needs a single-tile plan");
        return ENKFMC_E_VALUE;
    }
    int rc = ensure_device(p);
    if (rc) return rc;
    DeviceState *d = p->dev;
    CK(launch_precision_apply(d->row_ptr, d->col_idx, d->csc_ptr, d->csc_row, d->csc_src, d_T, d_D, d_V, d_tmp,
                              d_out, p->sum_nlocal(), ncols, (cudaStream_t)stream));
    p->counters[0] += 2;
    return ENKFMC_OK;
}

extern "C" int enkfmc_unit_tri_solve(enkfmc_plan *p, const double *d_T, int transposed, const double *d_scale_in,
                                     const double *d_scale_out, double *d_B, int64_t ncols, void *stream) {
    if (p->ntiles != 1 || p->nfields != 1) {
        enkfmc_set_error("unit_tri_solve needs a single-tile plan");
        return ENKFMC_E_VALUE;
    }
    int rc = ensure_device(p);
    if (rc) return rc;
    DeviceState *d = p->dev;
    if (transposed)
        CK(launch_unit_tri_solve(1, d->csc_ptr, d->csc_row, d->csc_src, d_T, d_scale_in, d_scale_out, d_B, p->sum_nlocal(), ncols,
                                 (cudaStream_t)stream));
    else
        CK(launch_unit_tri_solve(0, d->row_ptr, d->col_idx, nullptr, d_T, d_scale_in, d_scale_out, d_B, p->sum_nlocal(), ncols,
                                 (cudaStream_t)stream));
    p->counters[0] += 1;
    return ENKFMC_OK;
}

extern "C" int enkfmc_advdiff_step(const double *d_in, double *d_out, int64_t nx, int64_t ny, int row_major, int64_t nfields,
                                   int64_t nens, double ux, double uy, double dt, double kappa, void *stream) {
    int rc = check_nens(nens);
    if (rc) return rc;
    if (nx < 1 || ny < 1 || nfields < 1) { enkfmc_set_error("grid extents must be positive"); return ENKFMC_E_VALUE; }
    int dev = 0;
    CK(cudaGetDevice(&dev));
    int sms = 0;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    CK(launch_advdiff_step(d_in, d_out, nx, ny, row_major, nfields, (int)nens, ux, uy, dt, kappa, sms, (cudaStream_t)stream));
    return ENKFMC_OK;
}

extern "C" int enkfmc_letkf_device(const double *d_X, double *d_U, double *d_mean, double *d_Xa, const int32_t *d_obs_of_state,
                                   const double *d_rdiag, const double *d_y, int64_t nx, int64_t ny, int row_major, int periodic,
                                   int64_t nfields, int64_t nens, int64_t zeta, double inflation, int64_t *first_bad, void *stream) {
    int rc = check_nens(nens);
    if (rc) return rc;
    if (nx < 1 || ny < 1 || nfields < 1 || zeta < 0) { enkfmc_set_error("invalid grid extents or radius"); return ENKFMC_E_VALUE; }
    if (!(inflation > 0.0)) { enkfmc_set_error("inflation must be positive, got " + std::to_string(inflation)); return ENKFMC_E_VALUE; }
    int dev = 0;
    CK(cudaGetDevice(&dev));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, dev));
    if (prop.major < 10) { enkfmc_set_error("libenkfmc is built for sm_100a only"); return ENKFMC_E_CUDA; }
    cudaStream_t s = (cudaStream_t)stream;
    unsigned int *counter = nullptr;
    unsigned long long *bad = nullptr;
    CK(cudaMalloc(&counter, sizeof(unsigned int) + sizeof(unsigned long long) + 8));
    bad = reinterpret_cast<unsigned long long *>(reinterpret_cast<char *>(counter) + 8);
    CK(cudaMemsetAsync(counter, 0, 8, s));
    CK(cudaMemsetAsync(bad, 0xff, sizeof(unsigned long long), s));
    LetkfParams L{};
    L.X = d_X; L.U = d_U; L.mean = d_mean; L.Xa = d_Xa; L.obs_of_state = d_obs_of_state; L.rdiag = d_rdiag; L.y = d_y;
    L.nx = nx; L.ny = ny; L.nitems = nx * ny * nfields; L.zeta = zeta; L.row_major = row_major; L.periodic = periodic;
    L.N = (int)nens; L.boxmax = (int)((2 * zeta + 1) * (2 * zeta + 1)); L.inflation = inflation; L.eig_floor = 1e-12;
    L.counter = counter; L.first_bad = bad;
    cudaError_t e = launch_letkf(L, prop.multiProcessorCount, prop.sharedMemPerBlockOptin, s);
    if (e == cudaErrorInvalidConfiguration) {
        cudaFree(counter);
        enkfmc_set_error("LETKF workspace (two " + std::to_string(nens) + " x " + std::to_string(nens) +
                         " matrices per grid point) exceeds shared memory, or the radius exceeds 31");
        return ENKFMC_E_CAPACITY;
    }
    CK(e);
    unsigned long long hb = 0;
    CK(cudaStreamSynchronize(s));
    CK(cudaMemcpy(&hb, bad, sizeof(hb), cudaMemcpyDeviceToHost));
    cudaFree(counter);
    *first_bad = hb == ~0ull ? -1 : (int64_t)hb;
    if (hb != ~0ull) {
        enkfmc_set_error("component " + std::to_string(hb) + ": analysis weight matrix lost positive definiteness");
        return ENKFMC_E_NUMERIC;
    }
    return ENKFMC_OK;
}

extern "C" int enkfmc_plan_read_buffer(const enkfmc_plan *p, int what, void *host_out, int64_t bytes) {
    void *src = enkfmc_plan_device_buffer(p, what);
    if (!src) { enkfmc_set_error("workspace buffer not allocated"); return ENKFMC_E_VALUE; }
    {   // T, D and flags cover the owned tiles only: [nfields][owned count], in the plan's order
        const DeviceState *d = p->dev;
        const int64_t have = what == 0 ? p->nstate2d * p->nfields * d->ws_nens * 8 : what == 1 ? d->ws_nnz * p->nfields * 8 :
                             what == 2 ? d->ws_rows * p->nfields * 8 : what == 3 ? d->ws_rows * p->nfields * 4 : p->ntiles * p->nfields * 4;
        if (bytes > have) {
            enkfmc_set_error("workspace buffer holds " + std::to_string(have) + " bytes (the owned tiles' share), " +
                             std::to_string(bytes) + " requested");
            return ENKFMC_E_VALUE;
        }
    }
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(host_out, src, (size_t)bytes, cudaMemcpyDeviceToHost));
    return ENKFMC_OK;
}
