// Host-side integer index maps of the EnKF-MC analysis step (bit-exact with the reference).
//
// What each routine restates (reference = /root/reference/pkg/src/mcholkf):
//   tiling()            geometry.py:179-193   near-square block grid, ties to smaller pr
//   bands()             geometry.py:195-199   equal bands, remainder to the last
//   axis_window/band()  geometry.py:132-142   clip, or wrap + de-duplicate
//   box / predecessors  geometry.py:145-162
//   build_tiles()       geometry.py:204-221   interior, zeta-ring halo, sorted local_order
//   build_rows()        estimator.py:123-131  predecessors mapped into local positions
//   set_observations()  kernels.py:90-113     restrict_network per (field, tile)
// The rest (physical order, half-bandwidth, column lists, work orders) is new: it is what
// the CUDA kernels need and has no reference counterpart.

#include <algorithm>
#include <cstring>
#include <numeric>
#include <string>
#include <unordered_map>

#include "plan.h"

static thread_local std::string g_last_error;
void enkfmc_set_error(const std::string &msg) { g_last_error = msg; }

extern "C" const char *enkfmc_last_error(void) { return g_last_error.c_str(); }
extern "C" const char *enkfmc_version(void) { return "enkfmc 0.1 (sm_100a)"; }

namespace {

// periodic flag of the C-ABI: 0 clipped, 1 periodic on both axes (the reference's two boundaries, geometry.py:43), 2 periodic
// along x only (columns: longitude periodic, latitude clipped -- BASELINE.json config 1 as worded), 3 along y only.  The
// per-axis forms have no reference counterpart: they apply the reference's per-axis rules (geometry.py:132-142) with one
// flag per axis.
struct Geo {
    int64_t nx, ny;
    bool row_major, periodic_x, periodic_y;
    Geo(int64_t nx_, int64_t ny_, bool rm, int periodic)
        : nx(nx_), ny(ny_), row_major(rm), periodic_x(periodic == 1 || periodic == 2), periodic_y(periodic == 1 || periodic == 3) {}
    int64_t label(int64_t r, int64_t c) const { return row_major ? r * nx + c : c * ny + r; }
    void coords(int64_t lab, int64_t &r, int64_t &c) const {
        if (row_major) { r = lab / nx; c = lab % nx; } else { c = lab / ny; r = lab % ny; }
    }
};

int64_t pmod(int64_t a, int64_t n) { int64_t m = a % n; return m < 0 ? m + n : m; }

// Sorted unique coordinates within zeta of center.
void axis_window(int64_t center, int64_t zeta, int64_t n, bool periodic, std::vector<int64_t> &out) {
    out.clear();
    if (periodic) {
        for (int64_t d = -zeta; d <= zeta; ++d) out.push_back(pmod(center + d, n));
        std::sort(out.begin(), out.end());
        out.erase(std::unique(out.begin(), out.end()), out.end());
    } else {
        for (int64_t v = std::max<int64_t>(0, center - zeta); v < std::min(n, center + zeta + 1); ++v)
            out.push_back(v);
    }
}

// Coordinates within zeta of [lo, hi): `sorted` as the reference returns them, `walk` in
// unwrapped order (the order a band solver wants); walk == sorted when nothing wraps or
// when the band covers the whole axis.
void axis_band(int64_t lo, int64_t hi, int64_t zeta, int64_t n, bool periodic,
               std::vector<int64_t> &sorted, std::vector<int64_t> &walk) {
    sorted.clear();
    walk.clear();
    if (periodic) {
        for (int64_t v = lo - zeta; v < hi + zeta; ++v) walk.push_back(pmod(v, n));
        sorted = walk;
        std::sort(sorted.begin(), sorted.end());
        sorted.erase(std::unique(sorted.begin(), sorted.end()), sorted.end());
        if (sorted.size() != walk.size()) walk = sorted;  // wrapped onto itself: whole axis
    } else {
        for (int64_t v = std::max<int64_t>(0, lo - zeta); v < std::min(n, hi + zeta); ++v)
            sorted.push_back(v);
        walk = sorted;
    }
}

// Sorted labels of rows x cols (both ascending).
void label_product(const Geo &g, const std::vector<int64_t> &rows, const std::vector<int64_t> &cols,
                   std::vector<int64_t> &out) {
    out.clear();
    out.reserve(rows.size() * cols.size());
    if (g.row_major) {
        for (int64_t r : rows) for (int64_t c : cols) out.push_back(g.label(r, c));
    } else {
        for (int64_t c : cols) for (int64_t r : rows) out.push_back(g.label(r, c));
    }
}

void box_members(const Geo &g, int64_t center, int64_t zeta, std::vector<int64_t> &out,
                 std::vector<int64_t> &rows, std::vector<int64_t> &cols) {
    int64_t r, c;
    g.coords(center, r, c);
    axis_window(r, zeta, g.ny, g.periodic_y, rows);
    axis_window(c, zeta, g.nx, g.periodic_x, cols);
    label_product(g, rows, cols, out);
}

int check_geometry(int64_t nx, int64_t ny, int64_t zeta) {
    if (nx < 1 || ny < 1) {
        enkfmc_set_error("grid extents must be positive, got nx=" + std::to_string(nx) + " ny=" + std::to_string(ny));
        return ENKFMC_E_VALUE;
    }
    if (zeta < 0) {
        enkfmc_set_error("zeta must be nonnegative, got " + std::to_string(zeta));
        return ENKFMC_E_VALUE;
    }
    return ENKFMC_OK;
}

int tiling(int64_t nx, int64_t ny, int64_t delta, int64_t &pr, int64_t &pc) {
    if (delta < 1) {
        enkfmc_set_error("delta must be >= 1, got " + std::to_string(delta));
        return ENKFMC_E_CONFIG;
    }
    bool found = false;
    int64_t best_diff = 0, best_pr = 0;
    for (int64_t a = 1; a <= delta; ++a) {
        if (delta % a) continue;
        int64_t b = delta / a;
        if (a > ny || b > nx) continue;
        int64_t diff = a > b ? a - b : b - a;
        if (!found || diff < best_diff || (diff == best_diff && a < best_pr)) {
            found = true; best_diff = diff; best_pr = a;
        }
    }
    if (!found) {
        enkfmc_set_error("delta=" + std::to_string(delta) + " does not tile a " + std::to_string(ny) + "x" +
                         std::to_string(nx) + " grid");
        return ENKFMC_E_CONFIG;
    }
    pr = best_pr;
    pc = delta / best_pr;
    return ENKFMC_OK;
}

void bands(int64_t n, int64_t parts, std::vector<std::pair<int64_t, int64_t>> &out) {
    out.clear();
    int64_t base = n / parts;
    for (int64_t i = 0; i + 1 < parts; ++i) out.push_back({i * base, (i + 1) * base});
    out.push_back({(parts - 1) * base, n});
}

int64_t find_sorted(const int64_t *a, int64_t n, int64_t v) {
    const int64_t *it = std::lower_bound(a, a + n, v);
    return (it != a + n && *it == v) ? (it - a) : -1;
}

// Everything downstream of (tile_ptr, local_order, phys): rows, bandwidths, column lists, orders.
// Predecessors of a local row (estimator.py:123-131): the members of its box with a smaller label that are present in
// the local domain.  With levels (extension) the box is the 2-D box on every level within zeta_v; a lifted local domain
// (tile x all levels) is nlev copies of the same sorted 2-D cover, so positions are level * ncover + 2-D position.
void build_rows_from_geometry(enkfmc_plan &p) {
    Geo g{p.nx, p.ny, p.row_major != 0, p.periodic};
    p.row_ptr.assign(1, 0);
    p.col_idx.clear();
    std::vector<int64_t> box, rows, cols;
    for (int64_t t = 0; t < p.ntiles; ++t) {
        const int64_t base = p.tile_ptr[t], n = p.tile_ptr[t + 1] - base;
        const int64_t *lo = p.local_order.data() + base;
        const int64_t ncover = n / p.nlev;                 // 2-D cover of the tile (nlev == 1: the local domain itself)
        for (int64_t j = 0; j < n; ++j) {
            if (p.zeta > 0 || p.zeta_v > 0) {
                const int64_t lev = lo[j] / p.n2d, lab2 = lo[j] % p.n2d;
                box_members(g, lab2, p.zeta, box, rows, cols);
                for (int64_t l = std::max<int64_t>(0, lev - p.zeta_v); l <= lev; ++l) {
                    for (int64_t lab : box) {
                        if (l == lev && lab >= lab2) break;  // ascending: predecessors first
                        int64_t pos = find_sorted(lo, ncover, lab);   // level 0 block of the local order = the 2-D cover
                        if (pos >= 0) p.col_idx.push_back((int32_t)(l * ncover + pos));
                    }
                }
            }
            p.row_ptr.push_back((int64_t)p.col_idx.size());
        }
    }
}

void finish_plan(enkfmc_plan &p) {
    const int64_t total = p.sum_nlocal();
    p.row_tile.resize(total);
    p.max_nlocal = 0;
    for (int64_t t = 0; t < p.ntiles; ++t) {
        p.max_nlocal = std::max(p.max_nlocal, p.tile_ptr[t + 1] - p.tile_ptr[t]);
        for (int64_t q = p.tile_ptr[t]; q < p.tile_ptr[t + 1]; ++q) p.row_tile[q] = (int32_t)t;
    }
    // inverse physical order
    p.iphys.resize(total);
    for (int64_t t = 0; t < p.ntiles; ++t) {
        const int64_t base = p.tile_ptr[t];
        for (int64_t j = 0; j < p.tile_ptr[t + 1] - base; ++j) p.iphys[base + p.phys[base + j]] = (int32_t)j;
    }
    // tiles whose physical order is the local order (every clipped tile): K3a can stop a row's scan at the pivot entry
    p.tile_mono.assign((size_t)p.ntiles, 1);
    for (int64_t t = 0; t < p.ntiles; ++t) {
        const int64_t base = p.tile_ptr[t];
        for (int64_t j = 0; j < p.tile_ptr[t + 1] - base; ++j)
            if (p.phys[base + j] != (int32_t)j) { p.tile_mono[(size_t)t] = 0; break; }
    }
    // predecessor state rows, max predecessor count, half-bandwidth in physical order
    p.pred_state.resize(p.nnz());
    p.bw.assign(p.ntiles, 0);
    p.max_pred = 0;
    p.max_bw = 0;
    for (int64_t q = 0; q < total; ++q) {
        const int64_t base = p.tile_ptr[p.row_tile[q]];
        int32_t lo = p.phys[q], hi = p.phys[q];
        for (int64_t k = p.row_ptr[q]; k < p.row_ptr[q + 1]; ++k) {
            const int64_t qq = base + p.col_idx[k];
            p.pred_state[k] = p.state_row[qq];
            lo = std::min(lo, p.phys[qq]);
            hi = std::max(hi, p.phys[qq]);
        }
        p.max_pred = std::max(p.max_pred, p.row_ptr[q + 1] - p.row_ptr[q]);
        int32_t &b = p.bw[p.row_tile[q]];
        b = std::max(b, hi - lo);
    }
    for (int32_t b : p.bw) p.max_bw = std::max<int64_t>(p.max_bw, b);
    // column lists (transpose pattern), ascending row inside each column
    p.csc_ptr.assign(total + 1, 0);
    for (int64_t q = 0; q < total; ++q) {
        const int64_t base = p.tile_ptr[p.row_tile[q]];
        for (int64_t k = p.row_ptr[q]; k < p.row_ptr[q + 1]; ++k) p.csc_ptr[base + p.col_idx[k] + 1]++;
    }
    for (int64_t q = 0; q < total; ++q) p.csc_ptr[q + 1] += p.csc_ptr[q];
    p.csc_row.resize(p.nnz());
    p.csc_src.resize(p.nnz());
    std::vector<int64_t> fill(p.csc_ptr.begin(), p.csc_ptr.end() - 1);
    for (int64_t q = 0; q < total; ++q) {
        const int64_t base = p.tile_ptr[p.row_tile[q]];
        for (int64_t k = p.row_ptr[q]; k < p.row_ptr[q + 1]; ++k) {
            int64_t &slot = fill[base + p.col_idx[k]];
            p.csc_row[slot] = (int32_t)(q - base);
            p.csc_src[slot] = k;
            ++slot;
        }
    }
    p.tile_begin = 0;
    p.tile_end = p.ntiles;
    enkfmc_build_orders(p);
}

int validate_increasing(const int64_t *a, int64_t n, const char *name) {
    for (int64_t i = 0; i < n; ++i) {
        if (a[i] < 0) { enkfmc_set_error(std::string(name) + " must be nonnegative"); return ENKFMC_E_VALUE; }
        if (i && a[i] <= a[i - 1]) {
            enkfmc_set_error(std::string(name) + " must be strictly increasing");
            return ENKFMC_E_VALUE;
        }
    }
    return ENKFMC_OK;
}

}  // namespace

// Work orders over the owned tiles [tile_begin, tile_end): regressions with the most
// predecessors first, tiles with the largest solve cost first (stable sorts: deterministic).
void enkfmc_build_orders(enkfmc_plan &p) {
    p.work_order.clear();
    p.tile_order.clear();
    p.regress_order.clear();
    p.alias_row.clear();
    p.alias_rep.clear();
    // identical regressions (same state row, same predecessor list) among the owned rows
    std::unordered_map<uint64_t, std::vector<int32_t>> seen;
    auto row_hash = [&](int64_t q) {
        uint64_t h = 1469598103934665603ull ^ (uint64_t)(uint32_t)p.state_row[q];
        for (int64_t e = p.row_ptr[q]; e < p.row_ptr[q + 1]; ++e) {
            h ^= (uint64_t)(uint32_t)p.pred_state[e];
            h *= 1099511628211ull;
        }
        return h;
    };
    auto same_row = [&](int64_t a, int64_t b) {
        const int64_t n = p.row_ptr[a + 1] - p.row_ptr[a];
        if (p.state_row[a] != p.state_row[b] || n != p.row_ptr[b + 1] - p.row_ptr[b]) return false;
        return std::equal(p.pred_state.begin() + p.row_ptr[a], p.pred_state.begin() + p.row_ptr[a] + n,
                          p.pred_state.begin() + p.row_ptr[b]);
    };
    for (int64_t t = p.tile_begin; t < p.tile_end; ++t) {
        p.tile_order.push_back((int32_t)t);
        for (int64_t q = p.tile_ptr[t]; q < p.tile_ptr[t + 1]; ++q) {
            p.work_order.push_back((int32_t)q);
            auto &bucket = seen[row_hash(q)];
            int32_t rep = -1;
            for (int32_t c : bucket) if (same_row(c, q)) { rep = c; break; }
            if (rep < 0) {
                bucket.push_back((int32_t)q);
                p.regress_order.push_back((int32_t)q);
            } else {
                p.alias_row.push_back((int32_t)q);
                p.alias_rep.push_back(rep);
            }
        }
    }
    auto more_preds = [&](int32_t a, int32_t b) {
        return (p.row_ptr[a + 1] - p.row_ptr[a]) > (p.row_ptr[b + 1] - p.row_ptr[b]);
    };
    std::stable_sort(p.work_order.begin(), p.work_order.end(), more_preds);
    std::stable_sort(p.regress_order.begin(), p.regress_order.end(), more_preds);
    // packed QR block of every representative: R by columns (min(j+1,K) entries), c[K], e2; sized for
    // K = p (the largest block), valid for any ensemble size
    p.rq_ptr.assign((size_t)p.sum_nlocal() + 1, 0);
    {
        std::vector<uint8_t> is_rep((size_t)p.sum_nlocal(), 0);
        for (int32_t q : p.regress_order) is_rep[q] = 1;
        for (int64_t q = 0; q < p.sum_nlocal(); ++q) {
            const int64_t k = p.row_ptr[q + 1] - p.row_ptr[q];
            p.rq_ptr[q + 1] = p.rq_ptr[q] + (is_rep[q] ? k * (k + 1) / 2 + k + 1 : 0);
        }
    }
    std::stable_sort(p.tile_order.begin(), p.tile_order.end(), [&](int32_t a, int32_t b) {
        auto cost = [&](int32_t t) {
            double n = (double)(p.tile_ptr[t + 1] - p.tile_ptr[t]), w = (double)p.bw[t] + 1.0;
            return n * w * w;
        };
        return cost(a) > cost(b);
    });
}

extern "C" int enkfmc_plan_set_tile_range(enkfmc_plan *p, int64_t t0, int64_t t1) {
    if (t0 < 0 || t1 > p->ntiles || t0 > t1) {
        enkfmc_set_error("tile range [" + std::to_string(t0) + ", " + std::to_string(t1) + ") outside [0, " +
                         std::to_string(p->ntiles) + "]");
        return ENKFMC_E_VALUE;
    }
    p->tile_begin = t0;
    p->tile_end = t1;
    enkfmc_build_orders(*p);
    enkfmc_device_invalidate_orders(p);
    return ENKFMC_OK;
}

extern "C" int enkfmc_plan_work(const enkfmc_plan *p, int64_t nens, double *flops3) {
    const double N = (double)nens;
    auto qr_flops = [&](int64_t q) {
        const double k = (double)(p->row_ptr[q + 1] - p->row_ptr[q]);
        return 2.0 * N * k * k - (2.0 / 3.0) * k * k * k + 4.0 * N * k;
    };
    double reg = 0.0, sol = 0.0, reg_distinct = 0.0;
    for (int32_t q : p->work_order) reg += qr_flops(q);
    for (int32_t q : p->regress_order) reg_distinct += qr_flops(q);
    for (int64_t f = 0; f < p->nfields; ++f) {
        for (int64_t t = p->tile_begin; t < p->tile_end; ++t) {
            if (p->have_obs && p->tile_nobs[(size_t)(f * p->ntiles + t)] == 0) continue;
            const double n = (double)(p->tile_ptr[t + 1] - p->tile_ptr[t]), b = (double)p->bw[t];
            sol += n * b * b + 4.0 * n * b * N;
        }
    }
    flops3[0] = reg * (double)p->nfields;
    flops3[1] = sol;
    flops3[2] = reg_distinct * (double)p->nfields;
    return ENKFMC_OK;
}

extern "C" int enkfmc_tiling(int64_t nx, int64_t ny, int64_t delta, int64_t *pr, int64_t *pc) {
    int rc = check_geometry(nx, ny, 0);
    if (rc) return rc;
    return tiling(nx, ny, delta, *pr, *pc);
}

extern "C" int enkfmc_local_box(int64_t nx, int64_t ny, int row_major, int periodic, int64_t center,
                                int64_t zeta, int64_t *out, int64_t *count) {
    int rc = check_geometry(nx, ny, zeta);
    if (rc) return rc;
    if (center < 0 || center >= nx * ny) {
        enkfmc_set_error("index " + std::to_string(center) + " outside [0, " + std::to_string(nx * ny) + ")");
        return ENKFMC_E_VALUE;
    }
    Geo g{nx, ny, row_major != 0, periodic};
    std::vector<int64_t> box, rows, cols;
    box_members(g, center, zeta, box, rows, cols);
    std::copy(box.begin(), box.end(), out);
    *count = (int64_t)box.size();
    return ENKFMC_OK;
}

extern "C" int enkfmc_predecessors(int64_t nx, int64_t ny, int row_major, int periodic, int64_t center,
                                   int64_t zeta, int64_t *out, int64_t *count) {
    int rc = enkfmc_local_box(nx, ny, row_major, periodic, center, zeta, out, count);
    if (rc) return rc;
    int64_t m = 0;
    while (m < *count && out[m] < center) ++m;
    *count = m;
    return ENKFMC_OK;
}

extern "C" int enkfmc_plan_create(int64_t nx, int64_t ny, int row_major, int periodic, int64_t nfields,
                                  int64_t delta, int64_t zeta, enkfmc_plan **out) {
    return enkfmc_plan_create_levels(nx, ny, row_major, periodic, 1, 0, nfields, delta, zeta, out);
}

extern "C" int enkfmc_plan_create_levels(int64_t nx, int64_t ny, int row_major, int periodic, int64_t nlev, int64_t zeta_v,
                                         int64_t nfields, int64_t delta, int64_t zeta, enkfmc_plan **out) {
    *out = nullptr;
    int rc = check_geometry(nx, ny, zeta);
    if (rc) return rc;
    if (nfields < 1) { enkfmc_set_error("nfields must be positive"); return ENKFMC_E_VALUE; }
    if (nlev < 1) { enkfmc_set_error("nlev must be positive, got " + std::to_string(nlev)); return ENKFMC_E_VALUE; }
    if (zeta_v < 0) { enkfmc_set_error("zeta_v must be nonnegative, got " + std::to_string(zeta_v)); return ENKFMC_E_VALUE; }
    int64_t pr, pc;
    if (delta < 1) { enkfmc_set_error("delta must be >= 1, got " + std::to_string(delta)); return ENKFMC_E_CONFIG; }
    rc = tiling(nx, ny, delta, pr, pc);
    if (rc) return rc;
    if (nx * ny * nlev * nfields > INT32_MAX) { enkfmc_set_error("state dimension exceeds 2^31-1"); return ENKFMC_E_CAPACITY; }

    auto *p = new enkfmc_plan();
    p->nx = nx; p->ny = ny; p->row_major = row_major; p->periodic = periodic; p->nfields = nfields;
    p->delta = delta; p->zeta = zeta; p->pr = pr; p->pc = pc; p->kind = 0;
    p->nlev = nlev; p->zeta_v = nlev > 1 ? zeta_v : 0;
    p->ntiles = delta; p->n2d = nx * ny; p->nstate2d = nx * ny * nlev;
    Geo g{nx, ny, row_major != 0, periodic};

    std::vector<std::pair<int64_t, int64_t>> rb, cb;
    bands(ny, pr, rb);
    bands(nx, pc, cb);
    p->tile_ptr.assign(1, 0);
    p->interior_ptr.assign(1, 0);
    p->halo_ptr.assign(1, 0);
    std::vector<int64_t> rows_in, cols_in, rows_s, rows_w, cols_s, cols_w, inter, cover, halo2, ipos2;
    std::vector<int32_t> phys2;
    std::vector<int64_t> rowpos(ny), colpos(nx);
    for (int64_t bi = 0; bi < pr; ++bi) {
        for (int64_t bj = 0; bj < pc; ++bj) {
            rows_in.clear(); cols_in.clear();
            for (int64_t r = rb[bi].first; r < rb[bi].second; ++r) rows_in.push_back(r);
            for (int64_t c = cb[bj].first; c < cb[bj].second; ++c) cols_in.push_back(c);
            label_product(g, rows_in, cols_in, inter);
            axis_band(rb[bi].first, rb[bi].second, zeta, ny, g.periodic_y, rows_s, rows_w);
            axis_band(cb[bj].first, cb[bj].second, zeta, nx, g.periodic_x, cols_s, cols_w);
            label_product(g, rows_s, cols_s, cover);   // == union1d(interior, halo): sorted local_order
            ipos2.clear();
            for (int64_t lab : inter) ipos2.push_back(find_sorted(cover.data(), (int64_t)cover.size(), lab));
            // halo = covered \ interior (both sorted)
            halo2.clear();
            std::set_difference(cover.begin(), cover.end(), inter.begin(), inter.end(), std::back_inserter(halo2));
            // physical order: walk the extended rectangle in unwrapped order
            for (size_t i = 0; i < rows_w.size(); ++i) rowpos[rows_w[i]] = (int64_t)i;
            for (size_t i = 0; i < cols_w.size(); ++i) colpos[cols_w[i]] = (int64_t)i;
            const int64_t h = (int64_t)rows_w.size(), w = (int64_t)cols_w.size();
            phys2.resize(cover.size());
            for (size_t j = 0; j < cover.size(); ++j) {
                int64_t r, c;
                g.coords(cover[j], r, c);
                phys2[j] = (int32_t)(g.row_major ? rowpos[r] * w + colpos[c] : colpos[c] * h + rowpos[r]);
            }
            // the tile spans every level: level-major copies of the 2-D maps (labels ascending: level * n2d + 2-D label)
            const int64_t ncover = (int64_t)cover.size();
            for (int64_t l = 0; l < nlev; ++l) {
                const int64_t off = l * p->n2d;
                for (int64_t lab : cover) p->local_order.push_back(off + lab);
                for (int64_t lab : inter) p->interior.push_back(off + lab);
                for (int64_t q : ipos2) p->interior_pos.push_back(l * ncover + q);
                for (int64_t lab : halo2) p->halo.push_back(off + lab);
                for (int32_t q : phys2) p->phys.push_back((int32_t)(l * ncover) + q);
            }
            p->tile_ptr.push_back((int64_t)p->local_order.size());
            p->interior_ptr.push_back((int64_t)p->interior.size());
            p->halo_ptr.push_back((int64_t)p->halo.size());
        }
    }
    p->is_interior.assign(p->local_order.size(), 0);
    for (int64_t t = 0; t < p->ntiles; ++t)
        for (int64_t k = p->interior_ptr[t]; k < p->interior_ptr[t + 1]; ++k)
            p->is_interior[p->tile_ptr[t] + p->interior_pos[k]] = 1;
    p->state_row.resize(p->local_order.size());
    for (size_t q = 0; q < p->local_order.size(); ++q) p->state_row[q] = (int32_t)p->local_order[q];
    build_rows_from_geometry(*p);
    finish_plan(*p);
    *out = p;
    return ENKFMC_OK;
}

extern "C" int enkfmc_plan_create_local(int64_t nx, int64_t ny, int row_major, int periodic, int64_t zeta,
                                        int64_t n_local, const int64_t *local_order, enkfmc_plan **out) {
    *out = nullptr;
    int rc = check_geometry(nx, ny, zeta);
    if (rc) return rc;
    if (n_local < 0) { enkfmc_set_error("n_local must be nonnegative"); return ENKFMC_E_VALUE; }
    rc = validate_increasing(local_order, n_local, "local_order");
    if (rc) return rc;
    if (n_local && local_order[n_local - 1] >= nx * ny) {
        enkfmc_set_error("local_order contains labels outside the geometry");
        return ENKFMC_E_VALUE;
    }
    auto *p = new enkfmc_plan();
    p->nx = nx; p->ny = ny; p->row_major = row_major; p->periodic = periodic; p->nfields = 1;
    p->delta = 1; p->zeta = zeta; p->kind = 1; p->ntiles = 1; p->n2d = nx * ny; p->nstate2d = n_local;
    p->tile_ptr = {0, n_local};
    p->local_order.assign(local_order, local_order + n_local);
    p->interior = p->local_order;
    p->interior_ptr = {0, n_local};
    p->halo_ptr = {0, 0};
    p->interior_pos.resize(n_local);
    p->phys.resize(n_local);
    p->state_row.resize(n_local);
    p->is_interior.assign(n_local, 1);
    for (int64_t j = 0; j < n_local; ++j) {
        p->interior_pos[j] = j; p->phys[j] = (int32_t)j; p->state_row[j] = (int32_t)j;
    }
    build_rows_from_geometry(*p);
    finish_plan(*p);
    *out = p;
    return ENKFMC_OK;
}

extern "C" int enkfmc_plan_create_csr(int64_t n, const int64_t *indptr, const int64_t *indices,
                                      enkfmc_plan **out) {
    *out = nullptr;
    if (n < 0 || indptr[0] != 0) { enkfmc_set_error("invalid CSR pattern"); return ENKFMC_E_VALUE; }
    for (int64_t j = 0; j < n; ++j) {
        if (indptr[j + 1] < indptr[j]) { enkfmc_set_error("invalid CSR indptr"); return ENKFMC_E_VALUE; }
        for (int64_t k = indptr[j]; k < indptr[j + 1]; ++k) {
            if (indices[k] < 0 || indices[k] >= j) {
                enkfmc_set_error("T must be strictly lower triangular (unit diagonal is implicit)");
                return ENKFMC_E_VALUE;
            }
            if (k > indptr[j] && indices[k] <= indices[k - 1]) {
                enkfmc_set_error("CSR column indices must be strictly increasing per row");
                return ENKFMC_E_VALUE;
            }
        }
    }
    auto *p = new enkfmc_plan();
    p->nx = n; p->ny = 1; p->nfields = 1; p->delta = 1; p->zeta = 0; p->kind = 2; p->ntiles = 1;
    p->n2d = n; p->nstate2d = n;
    p->tile_ptr = {0, n};
    p->local_order.resize(n);
    std::iota(p->local_order.begin(), p->local_order.end(), 0);
    p->interior = p->local_order;
    p->interior_pos = p->local_order;
    p->interior_ptr = {0, n};
    p->halo_ptr = {0, 0};
    p->phys.resize(n);
    p->state_row.resize(n);
    p->is_interior.assign(n, 1);
    for (int64_t j = 0; j < n; ++j) { p->phys[j] = (int32_t)j; p->state_row[j] = (int32_t)j; }
    p->row_ptr.assign(indptr, indptr + n + 1);
    p->col_idx.resize(indptr[n]);
    for (int64_t k = 0; k < indptr[n]; ++k) p->col_idx[k] = (int32_t)indices[k];
    finish_plan(*p);
    *out = p;
    return ENKFMC_OK;
}

extern "C" void enkfmc_plan_destroy(enkfmc_plan *plan) {
    if (!plan) return;
    enkfmc_device_release(plan);
    delete plan;
}

extern "C" int enkfmc_plan_set_observations(enkfmc_plan *p, int64_t nobs, const int64_t *obs) {
    if (nobs < 0) { enkfmc_set_error("nobs must be nonnegative"); return ENKFMC_E_VALUE; }
    int rc = validate_increasing(obs, nobs, "obs_indices");
    if (rc) return rc;
    const int64_t nstate = p->nstate2d * p->nfields;
    if (nobs && obs[nobs - 1] >= nstate) {
        enkfmc_set_error("observation indices exceed the state dimension");
        return ENKFMC_E_VALUE;
    }
    const int64_t total = p->sum_nlocal();
    p->nobs = nobs;
    p->obs_indices.assign(obs, obs + nobs);
    p->obs_slot.assign((size_t)(p->nfields * total), -1);
    p->tile_nobs.assign((size_t)(p->nfields * p->ntiles), 0);
    std::vector<std::vector<std::pair<int64_t, int64_t>>> lists((size_t)(p->nfields * p->ntiles));

    if (p->kind != 0) {
        // single tile, state rows are local positions: every observation is inside
        for (int64_t k = 0; k < nobs; ++k) lists[0].push_back({obs[k], k});
    } else {
        // which block rows / block columns have coordinate v inside their extended band
        Geo g{p->nx, p->ny, p->row_major != 0, p->periodic};
        std::vector<std::pair<int64_t, int64_t>> rb, cb;
        bands(p->ny, p->pr, rb);
        bands(p->nx, p->pc, cb);
        std::vector<std::vector<int32_t>> row_blocks(p->ny), col_blocks(p->nx);
        std::vector<int64_t> s, w;
        for (int64_t bi = 0; bi < p->pr; ++bi) {
            axis_band(rb[bi].first, rb[bi].second, p->zeta, p->ny, g.periodic_y, s, w);
            for (int64_t v : s) row_blocks[v].push_back((int32_t)bi);
        }
        for (int64_t bj = 0; bj < p->pc; ++bj) {
            axis_band(cb[bj].first, cb[bj].second, p->zeta, p->nx, g.periodic_x, s, w);
            for (int64_t v : s) col_blocks[v].push_back((int32_t)bj);
        }
        for (int64_t k = 0; k < nobs; ++k) {
            const int64_t f = obs[k] / p->nstate2d, rem = obs[k] % p->nstate2d;
            const int64_t lev = rem / p->n2d, lab = rem % p->n2d;
            int64_t r, c;
            g.coords(lab, r, c);
            for (int32_t bi : row_blocks[r]) for (int32_t bj : col_blocks[c]) {
                const int64_t t = bi * p->pc + bj, base = p->tile_ptr[t];
                const int64_t ncover = (p->tile_ptr[t + 1] - base) / p->nlev;
                const int64_t pos = find_sorted(p->local_order.data() + base, ncover, lab);
                if (pos >= 0) lists[(size_t)(f * p->ntiles + t)].push_back({lev * ncover + pos, k});
            }
        }
    }
    p->obs_ptr.assign(1, 0);
    p->obs_pos.clear();
    p->obs_row.clear();
    for (int64_t f = 0; f < p->nfields; ++f) {
        for (int64_t t = 0; t < p->ntiles; ++t) {
            auto &lst = lists[(size_t)(f * p->ntiles + t)];
            for (auto &pr_ : lst) {
                p->obs_pos.push_back(pr_.first);
                p->obs_row.push_back(pr_.second);
                p->obs_slot[(size_t)(f * total + p->tile_ptr[t] + pr_.first)] = (int32_t)pr_.second;
            }
            p->tile_nobs[(size_t)(f * p->ntiles + t)] = (int32_t)lst.size();
            p->obs_ptr.push_back((int64_t)p->obs_pos.size());
        }
    }
    p->have_obs = true;
    enkfmc_device_invalidate_obs(p);
    return ENKFMC_OK;
}

extern "C" int64_t enkfmc_plan_size(const enkfmc_plan *p, int what) {
    switch (what) {
        case 0: return p->ntiles;
        case 1: return p->sum_nlocal();
        case 2: return p->nnz();
        case 3: return (int64_t)p->interior.size();
        case 4: return (int64_t)p->halo.size();
        case 5: return p->nobs;
        case 6: return (int64_t)p->obs_pos.size();
        case 7: return p->pr;
        case 8: return p->pc;
        case 9: return p->max_nlocal;
        case 10: return p->max_pred;
        case 11: return p->max_bw;
        case 12: return p->nfields;
        case 13: return p->n2d;
        case 16: return p->nlev;
        case 17: return p->zeta_v;
        case 14: return (int64_t)p->regress_order.size();   // distinct regressions among the owned rows
        case 15: return (int64_t)p->work_order.size();      // owned local rows
        default: return -1;
    }
}

namespace {
template <class V>
int copy_out(const V &v, int64_t *out, int64_t cap) {
    if ((int64_t)v.size() > cap) { enkfmc_set_error("output buffer too small"); return ENKFMC_E_VALUE; }
    for (size_t i = 0; i < v.size(); ++i) out[i] = (int64_t)v[i];
    return ENKFMC_OK;
}
}  // namespace

extern "C" int enkfmc_plan_get(const enkfmc_plan *p, int what, int64_t *out, int64_t cap) {
    switch (what) {
        case 0: return copy_out(p->tile_ptr, out, cap);
        case 1: return copy_out(p->local_order, out, cap);
        case 2: return copy_out(p->interior_ptr, out, cap);
        case 3: return copy_out(p->interior, out, cap);
        case 4: return copy_out(p->interior_pos, out, cap);
        case 5: return copy_out(p->halo_ptr, out, cap);
        case 6: return copy_out(p->halo, out, cap);
        case 7: return copy_out(p->row_ptr, out, cap);
        case 8: return copy_out(p->col_idx, out, cap);
        case 9: return copy_out(p->obs_ptr, out, cap);
        case 10: return copy_out(p->obs_pos, out, cap);
        case 11: return copy_out(p->obs_row, out, cap);
        case 12: return copy_out(p->bw, out, cap);
        case 13: return copy_out(p->phys, out, cap);
        case 14: {   // per local row: the row whose regression it shares (itself for a representative, -1 if not owned)
            std::vector<int64_t> rep((size_t)p->sum_nlocal(), -1);
            for (int32_t q : p->regress_order) rep[q] = q;
            for (size_t a = 0; a < p->alias_row.size(); ++a) rep[p->alias_row[a]] = p->alias_rep[a];
            return copy_out(rep, out, cap);
        }
        default: enkfmc_set_error("unknown map id"); return ENKFMC_E_VALUE;
    }
}
