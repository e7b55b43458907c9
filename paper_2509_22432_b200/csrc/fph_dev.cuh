// fph_dev.cuh -- device helpers shared by the flooding kernels: simplex
// vertices, the reference's barycentric embedding and Ritter ball, the fp32
// error bound of the expanded distance, packed-candidate tile math.
#pragma once

#include "fph_flood.cuh"

namespace fph {

constexpr double kU32 = 5.9604644775390625e-08;  // 2^-24

// ----------------------------------------------------- simplex geometry
struct Verts {
    double v[4][3];
};

__device__ __forceinline__ void load_verts(const FloodArgs& a, int s, Verts& V) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        int id = j <= a.k ? a.simplices[(size_t)s * 4 + j] : -1;
        V.v[j][0] = id >= 0 ? a.landmarks[(size_t)id * 3 + 0] : 0.0;
        V.v[j][1] = id >= 0 ? a.landmarks[(size_t)id * 3 + 1] : 0.0;
        V.v[j][2] = id >= 0 ? a.landmarks[(size_t)id * 3 + 2] : 0.0;
    }
}

// Reference barycentric row: p = w0*v0; p = p + wj*vj (w = c/m), no FMA
// (floodph/geometry.py barycentric_grid + barycentric_grid_template).
__device__ __forceinline__ void embed_row(const Verts& V, int k, ushort4 c, double m,
                                          double p[3]) {
    const unsigned cc[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        double w = __ddiv_rn((double)cc[0], m);
        double acc = __dmul_rn(w, V.v[0][a]);
#pragma unroll
        for (int j = 1; j < 4; ++j) {
            if (j <= k) {
                double wj = __ddiv_rn((double)cc[j], m);
                acc = __dadd_rn(acc, __dmul_rn(wj, V.v[j][a]));
            }
        }
        p[a] = acc;
    }
}

// Ritter ball exactly as reference floodph/geometry.py:123 (first longest
// edge in combinations order, center its midpoint, radius the farthest
// vertex).  Only used to bound candidate sets, kept exact anyway.
__device__ __forceinline__ double ritter(const Verts& V, int k, double c[3]) {
    if (k == 0) {
        c[0] = V.v[0][0];
        c[1] = V.v[0][1];
        c[2] = V.v[0][2];
        return 0.0;
    }
    double best = -1.0;
    double c0 = 0, c1 = 0, c2 = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = i + 1; j < 4; ++j) {
            if (j <= k) {
                double d = sq64(V.v[i][0], V.v[i][1], V.v[i][2], V.v[j][0], V.v[j][1], V.v[j][2]);
                if (d > best) {
                    best = d;
                    c0 = __dmul_rn(0.5, __dadd_rn(V.v[i][0], V.v[j][0]));
                    c1 = __dmul_rn(0.5, __dadd_rn(V.v[i][1], V.v[j][1]));
                    c2 = __dmul_rn(0.5, __dadd_rn(V.v[i][2], V.v[j][2]));
                }
            }
        }
    c[0] = c0;
    c[1] = c1;
    c[2] = c2;
    double mx = -1.0;
#pragma unroll
    for (int i = 0; i < 4; ++i)
        if (i <= k) mx = fmax(mx, sq64(V.v[i][0], V.v[i][1], V.v[i][2], c0, c1, c2));
    return sqrt(mx);
}


// Same row as embed_row with the weights c/m read from a table filled with
// __ddiv_rn (bit-identical, no division per coordinate).
__device__ __forceinline__ void embed_w(const Verts& V, int k, ushort4 c, const double* wt,
                                        double p[3]) {
    const unsigned cc[4] = {c.x, c.y, c.z, c.w};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        double acc = __dmul_rn(wt[cc[0]], V.v[0][a]);
#pragma unroll
        for (int j = 1; j < 4; ++j)
            if (j <= k) acc = __dadd_rn(acc, __dmul_rn(wt[cc[j]], V.v[j][a]));
        p[a] = acc;
    }
}

// Row j of simplex s: explicit coordinates (uniform-random sampler) or the
// template row embedded as the reference does (table weights when given).
__device__ __forceinline__ void sample_row(const FloodArgs& a, const Verts& V, int s, int j,
                                           const double* wt, double p[3]) {
    if (a.explicit_pts) {
        const double* q = a.explicit_pts + ((size_t)s * a.P + j) * 3;
        p[0] = q[0];
        p[1] = q[1];
        p[2] = q[2];
    } else if (wt) {
        embed_w(V, a.k, a.tmpl[j], wt, p);
    } else {
        embed_row(V, a.k, a.tmpl[j], (double)a.m, p);
    }
}

// sample_row for kernels that always hold the weight table (no division
// code is emitted)
__device__ __forceinline__ void sample_row_w(const FloodArgs& a, const Verts& V, int s, int j,
                                             const double* wt, double p[3]) {
    if (a.explicit_pts) {
        const double* q = a.explicit_pts + ((size_t)s * a.P + j) * 3;
        p[0] = q[0];
        p[1] = q[1];
        p[2] = q[2];
    } else {
        embed_w(V, a.k, a.tmpl[j], wt, p);
    }
}

// Rigorous bound on |m32 - d^2| for the expanded fp32 distance
// |a|^2 - 2 a.b + |b|^2 with a, b rounded once from float64 offsets to the
// simplex center: <= 16 u (|b| + d)^2, taken with a 2.5x margin.
__device__ __forceinline__ float err_bound(float m32, float B) {
    const float sv = sqrtf(fmaxf(m32, 0.f)) + B;
    return (float)(40.0 * kU32 * 1.01) * sv * sv;
}

}  // namespace fph
