// fph_grid.cuh -- device-resident spatial grid (see fph_grid.cu).
#pragma once

#include "fph_common.cuh"

namespace fph {

// Device-resident grid: the sorted cloud and cell table, and the Grid
// parameters themselves (d_grid) -- computed on the device from the cloud's
// bounding box, so building a grid never waits for the host.
struct GridStore {
    double* x = nullptr;
    double* y = nullptr;
    double* z = nullptr;
    int* cell_start = nullptr;  // cap + 1 entries (the used prefix: ncells + 1)
    int* idx = nullptr;
    Grid* d_grid = nullptr;     // device copy of the parameters
    long long cap = 0;
    void free_all(cudaStream_t stream);
};

// Bin the device cloud d_pts (n x dim float64, row-major) into gs, all on
// `stream`.  cell_size <= 0 picks the cell edge for about `occupancy` points
// per cell if the cloud filled its bounding box; keep_index also stores each
// sorted point's cloud index (gs->idx, Grid::idx).
int grid_build(const double* d_pts, int n, int dim, double cell_size, double occupancy,
               cudaStream_t stream, GridStore* gs, bool keep_index = false);

}  // namespace fph
