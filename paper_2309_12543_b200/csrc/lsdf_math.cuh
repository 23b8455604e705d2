// lsdf_math.cuh — scalar arithmetic of the hot path, written once for device
// (and, for the host-side recipe check in tests/native, for the CPU).
//
// Every function reproduces the reference's numpy expression in the same
// operation order, with explicit rounding intrinsics so nvcc cannot contract
// a*b+c into an FMA where numpy does not, and does use one where OpenBLAS
// does (np.matmul / dgemm, verified in SURVEY.md §7.3 and DESIGN.md §Parity):
//
//   np.matmul 3x3 / (V,3)@(3,3)   : fma(a2,b2, fma(a1,b1, a0*b0))
//   np.einsum "cij,cj"/"cij,j"    : (a0*b0 + a2*b2) + a1*b1     (no FMA)
//   np.einsum "bj,bjk->bk"        : (a0*b0 + a1*b1) + a2*b2     (no FMA)
//   (n,3) @ (3,)  (dgemv)         : fma(a2,b2, fma(a0,b0, a1*b1))
//   np.linalg.norm(axis=-1)       : sqrt((x0*x0 + x1*x1) + x2*x2)
#pragma once
#include <stdint.h>

#if defined(__CUDACC__)
#define LSDF_HD __host__ __device__ __forceinline__
#else
#define LSDF_HD inline
#endif

#if defined(__CUDA_ARCH__)
#define DFMA(a, b, c) __fma_rn((a), (b), (c))
#define DMUL(a, b) __dmul_rn((a), (b))
#define DADD(a, b) __dadd_rn((a), (b))
#define DSUB(a, b) __dsub_rn((a), (b))
#define DDIV(a, b) __ddiv_rn((a), (b))
#define DSQRT(a) __dsqrt_rn(a)
#define FMUL(a, b) __fmul_rn((a), (b))
#define FADD(a, b) __fadd_rn((a), (b))
#define FSUB(a, b) __fsub_rn((a), (b))
#else
#include <cmath>
#define DFMA(a, b, c) std::fma((a), (b), (c))
#define DMUL(a, b) ((double)(a) * (double)(b))
#define DADD(a, b) ((double)(a) + (double)(b))
#define DSUB(a, b) ((double)(a) - (double)(b))
#define DDIV(a, b) ((double)(a) / (double)(b))
#define DSQRT(a) std::sqrt(a)
#define FMUL(a, b) ((float)(a) * (float)(b))
#define FADD(a, b) ((float)(a) + (float)(b))
#define FSUB(a, b) ((float)(a) - (float)(b))
#endif

namespace lsdf {

// ---------------------------------------------------------------- small linalg
// C = A @ B for row-major 3x3 (np.matmul -> dgemm, FMA chain over k).
LSDF_HD void mm33(const double* A, const double* B, double* C) {
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int k = 0; k < 3; ++k)
            C[3 * i + k] = DFMA(A[3 * i + 2], B[6 + k], DFMA(A[3 * i + 1], B[3 + k], DMUL(A[3 * i], B[k])));
}

// out_i = sum_j A_ij v_j  (np.einsum "cij,cj->ci" / "cij,j->ci")
LSDF_HD void mv_einsum(const double* A, const double* v, double* out) {
#pragma unroll
    for (int i = 0; i < 3; ++i)
        out[i] = DADD(DADD(DMUL(A[3 * i], v[0]), DMUL(A[3 * i + 2], v[2])), DMUL(A[3 * i + 1], v[1]));
}

// Rodrigues (robot.py:35-46): c*I + s*K + (1-c)*kk^T, elementwise in that order.
LSDF_HD void rodrigues(const double* skew, const double* outer, double c, double s, double* M) {
    const double omc = DSUB(1.0, c);
#pragma unroll
    for (int e = 0; e < 9; ++e) {
        const double eye = (e == 0 || e == 4 || e == 8) ? 1.0 : 0.0;
        M[e] = DADD(DADD(DMUL(c, eye), DMUL(s, skew[e])), DMUL(omc, outer[e]));
    }
}

// x / r correctly rounded from rinv = RN(1 / r) without a division:
// q0 = RN(x rinv), the exact residual x - q0 r by FMA, one correction step
// (Markstein; also checked on 3.2e8 random operands,
// tests/test_hostcheck.py::test_division_recipe).  Normal operands only.
LSDF_HD double div_rn(double x, double r, double rinv) {
    const double q0 = DMUL(x, rinv);
    return DFMA(DFMA(-q0, r, x), rinv, q0);
}

// ---------------------------------------------------------------- alignment
// placement.py:60-99 for one position. Returns true when the window overlaps.
// rinv (optional): RN(1 / res) per axis, so the floor quotient needs no division.
LSDF_HD bool align_one(const double* pos, const double* ext, const double* res,
                       const int32_t* dims, const int32_t* W, int32_t* anchor, double* delta,
                       const double* rinv = nullptr) {
    const double eps = 2.220446049250313e-16;  // np.finfo(np.float64).eps
    bool overlap = true;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const double x = DADD(pos[a], ext[a]);
        double jf = floor(rinv ? div_rn(x, res[a], rinv[a]) : DDIV(x, res[a]));
        int64_t j = (int64_t)jf;
        // centers: -e + (j + 0.5) * r   (grids.py:80-83)
        double cen = DADD(-ext[a], DMUL(DADD((double)j, 0.5), res[a]));
        double d = DSUB(pos[a], cen);
        const double half = DMUL(0.5, res[a]);
        const double slack = DMUL(32.0 * eps, ext[a] > 1.0 ? ext[a] : 1.0);
        if (d >= half) j += 1;
        if (d < DSUB(-half, slack)) j -= 1;
        cen = DADD(-ext[a], DMUL(DADD((double)j, 0.5), res[a]));
        delta[a] = DSUB(pos[a], cen);
        const int64_t k = j - W[a] / 2;
        anchor[a] = (int32_t)k;
        if (k >= dims[a] || k + W[a] <= 0) overlap = false;
    }
    return overlap;
}

// dt_inv_k = -((dt0/e)*R0k + (dt1/e)*R1k + (dt2/e)*R2k)   (placement.py:165)
// e_rinv (optional, > 0): RN(1 / e_r), so the three quotients need no division.
LSDF_HD void shift_inverse(const double* R, const double* dt, double e_r, double* out, double e_rinv = 0.0) {
    const double a0 = e_rinv > 0.0 ? div_rn(dt[0], e_r, e_rinv) : DDIV(dt[0], e_r);
    const double a1 = e_rinv > 0.0 ? div_rn(dt[1], e_r, e_rinv) : DDIV(dt[1], e_r);
    const double a2 = e_rinv > 0.0 ? div_rn(dt[2], e_r, e_rinv) : DDIV(dt[2], e_r);
#pragma unroll
    for (int k = 0; k < 3; ++k)
        out[k] = -DADD(DADD(DMUL(a0, R[k]), DMUL(a1, R[3 + k])), DMUL(a2, R[6 + k]));
}

// ---------------------------------------------------------------- trilinear
struct GridView {
    const float* v;
    int32_t nx, ny, nz;
    float d_far;
    double ex, ey, ez;
    double rx, ry, rz;
};

// grids.py:155-191 at one link-frame point (fp64 coordinates, fp32 lerps).
template <typename Load>
LSDF_HD float trilinear_at(const GridView& g, double px, double py, double pz, Load load) {
    const double ux = DSUB(DDIV(DADD(px, g.ex), g.rx), 0.5);
    const double uy = DSUB(DDIV(DADD(py, g.ey), g.ry), 0.5);
    const double uz = DSUB(DDIV(DADD(pz, g.ez), g.rz), 0.5);
    const double hx = (double)(g.nx - 1), hy = (double)(g.ny - 1), hz = (double)(g.nz - 1);
    const bool inside = (ux >= 0.0) && (ux <= hx) && (uy >= 0.0) && (uy <= hy) && (uz >= 0.0) && (uz <= hz);
    if (!inside) return g.d_far;
    int ix = (int)ux, iy = (int)uy, iz = (int)uz;  // trunc == floor, u >= 0
    ix = ix < g.nx - 2 ? ix : g.nx - 2;
    iy = iy < g.ny - 2 ? iy : g.ny - 2;
    iz = iz < g.nz - 2 ? iz : g.nz - 2;
    const float fx = (float)DSUB(ux, (double)ix);
    const float fy = (float)DSUB(uy, (double)iy);
    const float fz = (float)DSUB(uz, (double)iz);
    const float gx = FSUB(1.0f, fx), gy = FSUB(1.0f, fy), gz = FSUB(1.0f, fz);
    const int64_t sy = g.nx, sz = (int64_t)g.nx * g.ny;
    const int64_t b = ix + sy * iy + sz * iz;
    const float v000 = load(b), v100 = load(b + 1);
    const float v010 = load(b + sy), v110 = load(b + 1 + sy);
    const float v001 = load(b + sz), v101 = load(b + 1 + sz);
    const float v011 = load(b + sy + sz), v111 = load(b + 1 + sy + sz);
    const float c00 = FADD(FMUL(v000, gx), FMUL(v100, fx));
    const float c10 = FADD(FMUL(v010, gx), FMUL(v110, fx));
    const float c01 = FADD(FMUL(v001, gx), FMUL(v101, fx));
    const float c11 = FADD(FMUL(v011, gx), FMUL(v111, fx));
    const float c0 = FADD(FMUL(c00, gy), FMUL(c10, fy));
    const float c1 = FADD(FMUL(c01, gy), FMUL(c11, fy));
    return FADD(FMUL(c0, gz), FMUL(c1, fz));
}

// Link-frame sample point of a window cell (placement.py:164-167 then the
// `g * window.extent` of placement.py:301-302):
//   g_k = (P R)_k + dt_inv_k ;  point_k = g_k * e_r
LSDF_HD void window_point(double px, double py, double pz, const double* R, const double* dtinv,
                          double e_r, double* out) {
#pragma unroll
    for (int k = 0; k < 3; ++k) {
        const double g = DFMA(pz, R[6 + k], DFMA(py, R[3 + k], DMUL(px, R[k])));
        out[k] = DMUL(DADD(g, dtinv[k]), e_r);
    }
}

// ---------------------------------------------------------------- reduction key
// Orderable 64-bit key: (value, position, link) lexicographic, -0.0 == +0.0.
LSDF_HD uint32_t orderable(float v) {
    if (v == 0.0f) v = 0.0f;
#if defined(__CUDA_ARCH__)
    uint32_t b = __float_as_uint(v);
#else
    uint32_t b;
    __builtin_memcpy(&b, &v, 4);
#endif
    return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}
LSDF_HD float from_orderable(uint32_t k) {
    uint32_t b = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
#if defined(__CUDA_ARCH__)
    return __uint_as_float(b);
#else
    float v;
    __builtin_memcpy(&v, &b, 4);
    return v;
#endif
}

// ---------------------------------------------------------------- primitives
// meshes.py:64-82, one point.
LSDF_HD double norm3(double x, double y, double z) {
    return DSQRT(DADD(DADD(DMUL(x, x), DMUL(y, y)), DMUL(z, z)));
}

LSDF_HD double primitive_at(int kind, const double* p, double x, double y, double z) {
    if (kind == 0) {  // sphere: p0 radius, p1..3 center
        return DSUB(norm3(DSUB(x, p[1]), DSUB(y, p[2]), DSUB(z, p[3])), p[0]);
    } else if (kind == 1) {  // capsule: p0 radius, p1 half length, p2..4 axis
        double t = DFMA(z, p[4], DFMA(x, p[2], DMUL(y, p[3])));
        const double hl = p[1];
        t = t < -hl ? -hl : (t > hl ? hl : t);
        return DSUB(norm3(DSUB(x, DMUL(t, p[2])), DSUB(y, DMUL(t, p[3])), DSUB(z, DMUL(t, p[4]))), p[0]);
    } else {  // box: p0..2 half extents
        const double qx = DSUB(fabs(x), p[0]), qy = DSUB(fabs(y), p[1]), qz = DSUB(fabs(z), p[2]);
        const double out = norm3(qx > 0.0 ? qx : 0.0, qy > 0.0 ? qy : 0.0, qz > 0.0 ? qz : 0.0);
        double m = qx > qy ? qx : qy;
        m = m > qz ? m : qz;
        return DADD(out, m < 0.0 ? m : 0.0);
    }
}

// ---------------------------------------------------------------- meshes
// einsum "ntj,tj->nt" (a0*b0 + a2*b2) + a1*b1
LSDF_HD double dot3(double a0, double a1, double a2, double b0, double b1, double b2) {
    return DADD(DADD(DMUL(a0, b0), DMUL(a2, b2)), DMUL(a1, b1));
}

struct Tri {
    double a[3], b[3], c[3];
};

// meshes.py:144-214 for one (point, triangle): squared distance.
LSDF_HD double closest_sq(const double* p, const double* a, const double* b, const double* c) {
    const double ab0 = DSUB(b[0], a[0]), ab1 = DSUB(b[1], a[1]), ab2 = DSUB(b[2], a[2]);
    const double ac0 = DSUB(c[0], a[0]), ac1 = DSUB(c[1], a[1]), ac2 = DSUB(c[2], a[2]);
    const double bc0 = DSUB(c[0], b[0]), bc1 = DSUB(c[1], b[1]), bc2 = DSUB(c[2], b[2]);
    const double ap0 = DSUB(p[0], a[0]), ap1 = DSUB(p[1], a[1]), ap2 = DSUB(p[2], a[2]);
    const double bp0 = DSUB(p[0], b[0]), bp1 = DSUB(p[1], b[1]), bp2 = DSUB(p[2], b[2]);
    const double cp0 = DSUB(p[0], c[0]), cp1 = DSUB(p[1], c[1]), cp2 = DSUB(p[2], c[2]);
    const double d1 = dot3(ap0, ap1, ap2, ab0, ab1, ab2);
    const double d2 = dot3(ap0, ap1, ap2, ac0, ac1, ac2);
    const double d3 = dot3(bp0, bp1, bp2, ab0, ab1, ab2);
    const double d4 = dot3(bp0, bp1, bp2, ac0, ac1, ac2);
    const double d5 = dot3(cp0, cp1, cp2, ab0, ab1, ab2);
    const double d6 = dot3(cp0, cp1, cp2, ac0, ac1, ac2);
    const double va = DSUB(DMUL(d3, d6), DMUL(d5, d4));
    const double vb = DSUB(DMUL(d5, d2), DMUL(d1, d6));
    const double vc = DSUB(DMUL(d1, d4), DMUL(d3, d2));
    double q0, q1, q2;
    const double d43 = DSUB(d4, d3), d56 = DSUB(d5, d6);
    if (d1 <= 0.0 && d2 <= 0.0) {
        q0 = a[0]; q1 = a[1]; q2 = a[2];
    } else if (d3 >= 0.0 && d4 <= d3) {
        q0 = b[0]; q1 = b[1]; q2 = b[2];
    } else if (vc <= 0.0 && d1 >= 0.0 && d3 <= 0.0) {
        double t = DDIV(d1, DSUB(d1, d3));
        if (!(t == t)) t = 0.0;  // nan_to_num (inf cannot occur on this branch's use)
        q0 = DADD(a[0], DMUL(t, ab0)); q1 = DADD(a[1], DMUL(t, ab1)); q2 = DADD(a[2], DMUL(t, ab2));
    } else if (d6 >= 0.0 && d5 <= d6) {
        q0 = c[0]; q1 = c[1]; q2 = c[2];
    } else if (vb <= 0.0 && d2 >= 0.0 && d6 <= 0.0) {
        double t = DDIV(d2, DSUB(d2, d6));
        if (!(t == t)) t = 0.0;
        q0 = DADD(a[0], DMUL(t, ac0)); q1 = DADD(a[1], DMUL(t, ac1)); q2 = DADD(a[2], DMUL(t, ac2));
    } else if (va <= 0.0 && d43 >= 0.0 && d56 >= 0.0) {
        double t = DDIV(d43, DADD(d43, d56));
        if (!(t == t)) t = 0.0;
        q0 = DADD(b[0], DMUL(t, bc0)); q1 = DADD(b[1], DMUL(t, bc1)); q2 = DADD(b[2], DMUL(t, bc2));
    } else {
        double den = DADD(DADD(va, vb), vc);
        if (den == 0.0) den = 1.0;
        const double v = DDIV(vb, den), w = DDIV(vc, den);
        q0 = DADD(DADD(a[0], DMUL(v, ab0)), DMUL(w, ac0));
        q1 = DADD(DADD(a[1], DMUL(v, ab1)), DMUL(w, ac1));
        q2 = DADD(DADD(a[2], DMUL(v, ab2)), DMUL(w, ac2));
    }
    const double e0 = DSUB(p[0], q0), e1 = DSUB(p[1], q1), e2 = DSUB(p[2], q2);
    return dot3(e0, e1, e2, e0, e1, e2);
}

// np.cross(a, b) component order (numpy linalg: a1*b2 - a2*b1, ...)
LSDF_HD void cross3(const double* a, const double* b, double* o) {
    o[0] = DSUB(DMUL(a[1], b[2]), DMUL(a[2], b[1]));
    o[1] = DSUB(DMUL(a[2], b[0]), DMUL(a[0], b[2]));
    o[2] = DSUB(DMUL(a[0], b[1]), DMUL(a[1], b[0]));
}

// Per-triangle ray constants along one direction (meshes.py:265-271).
struct RayTri {
    double a[3], e1[3], e2[3], h[3], det;  // det == 1.0 and parallel flag packed
    int parallel;
};

// One (point, triangle) crossing test (meshes.py:277-287).
// Returns 0 no hit, 1 hit, 2 hit near an edge (suspect).
LSDF_HD int ray_cross(const double* p, const RayTri& t, const double* dir) {
    if (t.parallel) return 0;
    const double s[3] = {DSUB(p[0], t.a[0]), DSUB(p[1], t.a[1]), DSUB(p[2], t.a[2])};
    const double u = DDIV(dot3(s[0], s[1], s[2], t.h[0], t.h[1], t.h[2]), t.det);
    double q[3];
    cross3(s, t.e1, q);
    const double v = DDIV(dot3(q[0], q[1], q[2], dir[0], dir[1], dir[2]), t.det);
    const double tt = DDIV(dot3(q[0], q[1], q[2], t.e2[0], t.e2[1], t.e2[2]), t.det);
    const bool hit = (u >= 0.0) && (v >= 0.0) && (DADD(u, v) <= 1.0) && (tt > 0.0);
    if (!hit) return 0;
    const double eps = 1e-9;
    const bool near = (u < eps) || (v < eps) || (DADD(u, v) > 1.0 - eps) || (fabs(tt) < eps);
    return near ? 2 : 1;
}

}  // namespace lsdf
