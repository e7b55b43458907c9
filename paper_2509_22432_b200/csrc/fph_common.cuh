// fph_common.cuh -- shared device helpers for the flood-filtration library.
//
// Exactness contract: every float64 quantity that must match the reference
// bit for bit (farthest-point distances, barycentric grid rows, Ritter balls,
// refined squared distances) is computed with explicit round-to-nearest
// intrinsics (__dadd_rn/__dsub_rn/__dmul_rn) so nvcc can never contract a
// multiply-add into an FMA.  The reference accumulates coordinate by
// coordinate, s = d0*d0; s = s + d1*d1; s = s + d2*d2 (floodph/geometry.py:61,
// floodph/_kernels.py:41); sq64() below is that exact sequence.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#define FPH_OK 0
#define FPH_EARG 1
#define FPH_ECUDA 2
#define FPH_ENOMEM 3
#define FPH_EINTEGRITY 4

namespace fph {

// ------------------------------------------------------------------ errors
void set_error(const char* fmt, ...);

#define FPH_CUDA_TRY(expr)                                                       \
    do {                                                                         \
        cudaError_t _e = (expr);                                                 \
        if (_e != cudaSuccess) {                                                 \
            ::fph::set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr,          \
                             cudaGetErrorString(_e));                            \
            return FPH_ECUDA;                                                    \
        }                                                                        \
    } while (0)

#define FPH_TRY(expr)                                                            \
    do {                                                                         \
        int _rc = (expr);                                                        \
        if (_rc != FPH_OK) return _rc;                                           \
    } while (0)

// Stream-ordered scratch (cudaMallocAsync), freed on every exit path.
struct Scratch {
    cudaStream_t stream;
    std::vector<void*> ptrs;
    explicit Scratch(cudaStream_t s) : stream(s) {}
    Scratch(const Scratch&) = delete;
    Scratch& operator=(const Scratch&) = delete;
    template <class T>
    int alloc(T** p, size_t count) {
        void* q = nullptr;
        cudaError_t e = cudaMallocAsync(&q, count * sizeof(T) + 16, stream);
        if (e != cudaSuccess) {
            set_error("cudaMallocAsync(%zu bytes): %s", count * sizeof(T), cudaGetErrorString(e));
            return FPH_ENOMEM;
        }
        ptrs.push_back(q);
        *p = static_cast<T*>(q);
        return FPH_OK;
    }
    ~Scratch() {
        for (void* p : ptrs) cudaFreeAsync(p, stream);
    }
};

// ------------------------------------------------------- exact float64 ops
__device__ __forceinline__ double sq64(double ax, double ay, double az, double bx,
                                       double by, double bz) {
    double t0 = __dsub_rn(ax, bx);
    double t1 = __dsub_rn(ay, by);
    double t2 = __dsub_rn(az, bz);
    double s = __dmul_rn(t0, t0);
    s = __dadd_rn(s, __dmul_rn(t1, t1));
    s = __dadd_rn(s, __dmul_rn(t2, t2));  // 2-D clouds carry z = 0: s + 0 = s
    return s;
}

// ------------------------------------------------ packed fp32 (sm_100a)
// fma.rn.f32x2 issues one FFMA2 for two lanes; ptxas folds a duplicated
// scalar operand into the ".F32" broadcast form, so per-point scalars need
// no register duplication.
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
    float2 d;
    asm("{.reg .b64 ra, rb, rc, rd;\n\t"
        "mov.b64 ra, {%2,%3};\n\t"
        "mov.b64 rb, {%4,%5};\n\t"
        "mov.b64 rc, {%6,%7};\n\t"
        "fma.rn.f32x2 rd, ra, rb, rc;\n\t"
        "mov.b64 {%0,%1}, rd;}"
        : "=f"(d.x), "=f"(d.y)
        : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
    return d;
}

// three-input min (FMNMX3, sm_100+)
__device__ __forceinline__ float fmin3(float a, float b, float c) {
    float d;
    asm("min.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
    return d;
}

// order-preserving float <-> uint mapping for atomicMin on signed floats
__device__ __forceinline__ unsigned f2ord(float f) {
    unsigned u = __float_as_uint(f);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float ord2f(unsigned u) {
    return __uint_as_float((u & 0x80000000u) ? (u & 0x7fffffffu) : ~u);
}

// ------------------------------------------------------- warp reductions
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ float warp_min_f(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ double warp_min_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ int warp_sum_i(int v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// ------------------------------------------------------- spatial grid
// Points sorted by linear cell id (x fastest), stored as float64 SoA.
struct Grid {
    const double* x;
    const double* y;
    const double* z;
    const int* cell_start;  // ncells + 1
    const int* idx;         // cloud index of each sorted point (only when requested)
    int n;
    int nx, ny, nz;
    double lox, loy, loz;
    double h, inv_h;
    double margin;  // absolute slack added to every box query
};

__device__ __forceinline__ int cell_coord(double v, double lo, double inv_h, int nmax) {
    double f = floor(__dmul_rn(__dsub_rn(v, lo), inv_h));
    int i = (int)fmax(0.0, fmin(f, (double)(nmax - 1)));
    return i;
}

// The cell box of a ball (inclusive bounds).  Binning uses the same
// monotone float64 expression, so every point inside the ball lands in a
// cell of the box.
struct Box {
    int x0, x1, y0, y1, z0, z1;
    __device__ __forceinline__ int ny_b() const { return y1 - y0 + 1; }
    __device__ __forceinline__ int rows() const { return (y1 - y0 + 1) * (z1 - z0 + 1); }
};

__device__ __forceinline__ Box ball_box(const Grid& g, double cx, double cy, double cz,
                                        double rad) {
    Box b;
    double R = rad + g.margin;
    b.x0 = cell_coord(cx - R, g.lox, g.inv_h, g.nx);
    b.x1 = cell_coord(cx + R, g.lox, g.inv_h, g.nx);
    b.y0 = cell_coord(cy - R, g.loy, g.inv_h, g.ny);
    b.y1 = cell_coord(cy + R, g.loy, g.inv_h, g.ny);
    b.z0 = cell_coord(cz - R, g.loz, g.inv_h, g.nz);
    b.z1 = cell_coord(cz + R, g.loz, g.inv_h, g.nz);
    return b;
}

__device__ __forceinline__ Box full_box(const Grid& g) {
    Box b;
    b.x0 = 0; b.x1 = g.nx - 1; b.y0 = 0; b.y1 = g.ny - 1; b.z0 = 0; b.z1 = g.nz - 1;
    return b;
}

// Contiguous run of sorted points for row r of a box, clipped to the
// ball's chord in that row (a superset: the row's yz-rectangle is padded by
// the grid margin).  Returns the run as [begin, end).
__device__ __forceinline__ int2 row_run(const Grid& g, const Box& b, int r, double cx,
                                        double cy, double cz, double rad, bool clip) {
    int ny_b = b.ny_b();
    int iy = b.y0 + r % ny_b;
    int iz = b.z0 + r / ny_b;
    int x0 = b.x0, x1 = b.x1;
    if (clip) {
        double R = rad + g.margin;
        double ylo = g.loy + iy * g.h - g.margin, yhi = g.loy + (iy + 1) * g.h + g.margin;
        double zlo = g.loz + iz * g.h - g.margin, zhi = g.loz + (iz + 1) * g.h + g.margin;
        double dy = fmax(0.0, fmax(ylo - cy, cy - yhi));
        double dz = fmax(0.0, fmax(zlo - cz, cz - zhi));
        double rem = R * R - dy * dy - dz * dz;
        if (rem < 0.0) return make_int2(0, 0);
        double half = sqrt(rem) * (1.0 + 1e-12) + g.margin;
        x0 = max(x0, cell_coord(cx - half, g.lox, g.inv_h, g.nx));
        x1 = min(x1, cell_coord(cx + half, g.lox, g.inv_h, g.nx));
        if (x1 < x0) return make_int2(0, 0);
    }
    int base = (iz * g.ny + iy) * g.nx;
    return make_int2(g.cell_start[base + x0], g.cell_start[base + x1 + 1]);
}

// fp32 version for the search kernel: the same superset contract, with the
// ball center given relative to the grid origin (one float64 subtraction per
// region, not per row) and an absolute slack that dominates every fp32
// rounding of the chord arithmetic.
struct RowClipF {
    float cx, cy, cz;  // center - grid origin
    float R, slack;
};

__device__ __forceinline__ RowClipF make_clip_f(const Grid& g, double cx, double cy, double cz,
                                                double R) {
    RowClipF c;
    const double rx = cx - g.lox, ry = cy - g.loy, rz = cz - g.loz;
    c.cx = (float)rx;
    c.cy = (float)ry;
    c.cz = (float)rz;
    c.R = (float)R;
    c.slack = (float)(2e-5 * (fabs(rx) + fabs(ry) + fabs(rz) + R + g.h) + 1e-3 * g.h + g.margin);
    return c;
}

__device__ __forceinline__ int2 row_run_f(const Grid& g, const Box& b, int r, const RowClipF& c) {
    const int ny_b = b.ny_b();
    const int iy = b.y0 + r % ny_b;
    const int iz = b.z0 + r / ny_b;
    const float h = (float)g.h, ih = (float)g.inv_h;
    const float ylo = iy * h - c.slack, yhi = (iy + 1) * h + c.slack;
    const float zlo = iz * h - c.slack, zhi = (iz + 1) * h + c.slack;
    const float dy = fmaxf(0.f, fmaxf(ylo - c.cy, c.cy - yhi));
    const float dz = fmaxf(0.f, fmaxf(zlo - c.cz, c.cz - zhi));
    const float Rs = c.R + c.slack;
    const float rem = Rs * Rs - dy * dy - dz * dz;
    if (rem < 0.f) return make_int2(0, 0);
    const float half = sqrtf(rem) * 1.0001f + c.slack;
    const int x0 = max(b.x0, (int)floorf((c.cx - half) * ih));
    const int x1 = min(b.x1, (int)floorf((c.cx + half) * ih));
    if (x1 < x0) return make_int2(0, 0);
    const int base = (iz * g.ny + iy) * g.nx;
    return make_int2(g.cell_start[base + x0], g.cell_start[base + x1 + 1]);
}

}  // namespace fph
