// fph_grid.cuh -- device-resident spatial grid (see fph_grid.cu).
#pragma once

#include "fph_common.cuh"

namespace fph {

struct GridStore {
    double* x = nullptr;
    double* y = nullptr;
    double* z = nullptr;
    int* cell_start = nullptr;
    int* idx = nullptr;
    long long ncells = 0;
    Grid grid{};
    void free_all(cudaStream_t stream);
};

// Default cell edge: about `occupancy` points per cell if the cloud filled
// its bounding box uniformly.
double grid_cell_size(const double lo[3], const double hi[3], int dim, long long n,
                      double occupancy);

// Bin the device cloud d_pts (n x dim float64, row-major) into gs.
// cell_size <= 0 picks grid_cell_size(..., occupancy); keep_index also
// stores each sorted point's cloud index (gs->idx, Grid::idx).
int grid_build(const double* d_pts, int n, int dim, double cell_size, double occupancy,
               cudaStream_t stream, GridStore* gs, bool keep_index = false);

}  // namespace fph
