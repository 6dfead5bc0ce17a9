// Internal plan layout shared by plan.cpp (host index maps) and api.cu (device side).
#pragma once
#include <cstdint>
#include <string>
#include <vector>

#include "enkf_mc.h"

struct DeviceState;  // defined in api.cu

struct enkfmc_plan {
    // geometry.py:22-66 descriptor (+ nfields extension)
    int64_t nx = 0, ny = 0, nfields = 1, delta = 1, zeta = 0, pr = 1, pc = 1;
    int row_major = 1, periodic = 0;
    int kind = 0;  // 0 decompose, 1 explicit local_order, 2 explicit CSR pattern
    int64_t ntiles = 0, n2d = 0, nstate2d = 0;  // nstate2d: rows of one field's state block (= n2d * nlev)
    // vertically coupled fields (extension, BASELINE.json configs 3 / 5 "vertical r = 1"): a field is nlev stacked 2-D
    // levels, row = level * n2d + 2-D label; a component's box spans the levels within zeta_v of its own
    int64_t nlev = 1, zeta_v = 0;

    // tile-major maps, exactly the reference's arrays (int64)
    std::vector<int64_t> tile_ptr, local_order, interior_ptr, interior, interior_pos, halo_ptr, halo;
    std::vector<int64_t> row_ptr;       // sum n_local + 1
    std::vector<int32_t> col_idx;       // nnz, local positions, ascending per row

    // derived maps consumed by the kernels
    std::vector<int32_t> state_row;     // per local row: row inside one field's state block
    std::vector<int32_t> pred_state;    // per nnz: state_row of that predecessor
    std::vector<int32_t> row_tile;      // per local row
    std::vector<int32_t> phys, iphys;   // physical (band) order inside the tile and its inverse
    std::vector<int32_t> bw;            // per tile: half-bandwidth of A in physical order
    std::vector<uint8_t> is_interior;   // per local row
    std::vector<uint8_t> tile_mono;     // per tile: physical order == local order
    std::vector<int64_t> csc_ptr;       // per local row + 1: column lists of T (global offsets)
    std::vector<int32_t> csc_row;       // local row j holding the entry
    std::vector<int64_t> csc_src;       // offset of the entry in the CSR value array
    std::vector<int32_t> work_order;    // owned local rows sorted by predecessor count, descending
    // Halo rows are regressed once per tile holding them (estimator.py:123-159 runs per sub-domain), but two
    // local rows with the same state row and the same predecessor list are the same regression: it is
    // computed once (regress_order, the representatives) and copied to its aliases.
    std::vector<int32_t> regress_order; // representatives among the owned rows, most predecessors first
    std::vector<int32_t> alias_row, alias_rep;   // owned non-representative rows and their representatives
    std::vector<int64_t> rq_ptr;        // per local row + 1: offset of the packed QR block (representatives only)
    std::vector<int32_t> tile_order;    // tiles sorted by solve cost, descending
    int64_t max_nlocal = 0, max_pred = 0, max_bw = 0;

    // observations (kernels.py:90-113), per (field, tile)
    int64_t nobs = 0;
    bool have_obs = false;
    std::vector<int64_t> obs_indices, obs_ptr, obs_pos, obs_row;
    std::vector<int32_t> obs_slot;      // nfields x sum n_local: parent obs row or -1
    std::vector<int32_t> tile_nobs;     // nfields x ntiles

    int64_t tile_begin = 0, tile_end = 0;   // owned tiles (one rank's share)
    bool profile = false;

    DeviceState *dev = nullptr;
    int64_t counters[8] = {0, 0, 0, 0, -1, 0, 0, 0};

    int64_t sum_nlocal() const { return tile_ptr.empty() ? 0 : tile_ptr.back(); }
    int64_t nnz() const { return row_ptr.empty() ? 0 : row_ptr.back(); }
};

void enkfmc_set_error(const std::string &msg);
void enkfmc_device_release(enkfmc_plan *plan);  // api.cu
void enkfmc_device_invalidate_obs(enkfmc_plan *plan);
void enkfmc_device_invalidate_orders(enkfmc_plan *plan);
void enkfmc_build_orders(enkfmc_plan &p);  // plan.cpp
