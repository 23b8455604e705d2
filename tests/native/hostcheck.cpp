// hostcheck.cpp — TEST-ONLY host build of the kernels' scalar arithmetic.
//
// Compiles paper_2309_12543_b200/csrc/lsdf_math.cuh as plain C++ (std::fma,
// -ffp-contract=off) so the CPU test suite can check, without a GPU, that the
// operation orders the CUDA kernels use reproduce the reference's numpy
// results bit-for-bit (golden fixtures).  Never loaded by the product package.
#include <cmath>
#include <cstdint>
#include <cstring>

#include "../../include/linksdf_b200.h"
#include "../../paper_2309_12543_b200/csrc/lsdf_math.cuh"

using namespace lsdf;

extern "C" {

// Same chain walk as fk_align_kernel (lsdf_query.cu), one configuration at a time.
void hc_fk(const lsdf_link* links, int n_links, const double* q, int64_t C, int D, double* R_out, double* T_out) {
    double rl[LSDF_MAX_LINKS][9], tl[LSDF_MAX_LINKS][3], R[LSDF_MAX_LINKS][9], T[LSDF_MAX_LINKS][3];
    for (int64_t c = 0; c < C; ++c) {
        const double* qc = q + c * D;
        for (int li = 0; li < n_links; ++li) {
            const lsdf_link& L = links[li];
            if (L.kind == 1) {
                double M[9];
                const double a = qc[L.q_col];
                rodrigues(L.skew, L.outer, std::cos(a), std::sin(a), M);
                mm33(L.joint_R, M, rl[li]);
                for (int k = 0; k < 3; ++k) tl[li][k] = L.joint_t[k];
            } else {
                for (int e = 0; e < 9; ++e) rl[li][e] = L.joint_R[e];
                for (int k = 0; k < 3; ++k)
                    tl[li][k] = L.kind == 2 ? DADD(L.joint_t[k], DMUL(qc[L.q_col], L.R_axis[k])) : L.joint_t[k];
            }
        }
        for (int li = 0; li < n_links; ++li) {
            const lsdf_link& L = links[li];
            double rj[9], tj[3], tmp[3];
            if (L.kind == 0) {
                const double I[9] = {1, 0, 0, 0, 1, 0, 0, 0, 1};
                std::memcpy(rj, I, sizeof(I));
                tj[0] = tj[1] = tj[2] = 0.0;
            } else {
                mm33(R[L.parent], rl[li], rj);
                mv_einsum(R[L.parent], tl[li], tmp);
                for (int k = 0; k < 3; ++k) tj[k] = DADD(T[L.parent][k], tmp[k]);
            }
            mm33(rj, L.link_R, R[li]);
            mv_einsum(rj, L.link_t, tmp);
            for (int k = 0; k < 3; ++k) T[li][k] = DADD(tj[k], tmp[k]);
            std::memcpy(R_out + (c * n_links + li) * 9, R[li], sizeof(R[li]));
            std::memcpy(T_out + (c * n_links + li) * 3, T[li], sizeof(T[li]));
        }
    }
}

int hc_align(const double* T, int64_t n, const lsdf_env_grid* env, const int32_t* W, int32_t* anchor, double* dt) {
    int bad = 0;
    for (int64_t i = 0; i < n; ++i)
        bad += !align_one(T + 3 * i, env->extent, env->resolution, env->dims, W, anchor + 3 * i, dt + 3 * i);
    return bad;
}

// the same with the reciprocal-multiply quotient the FK kernels use
int hc_align_rinv(const double* T, int64_t n, const lsdf_env_grid* env, const int32_t* W, int32_t* anchor,
                  double* dt) {
    const double rinv[3] = {1.0 / env->resolution[0], 1.0 / env->resolution[1], 1.0 / env->resolution[2]};
    int bad = 0;
    for (int64_t i = 0; i < n; ++i)
        bad += !align_one(T + 3 * i, env->extent, env->resolution, env->dims, W, anchor + 3 * i, dt + 3 * i, rinv);
    return bad;
}

// shift_inverse with and without the reciprocal (n rotations): the max |difference| (expect 0)
double hc_shift_diff(const double* R, const double* dt, int64_t n, double e_r) {
    double worst = 0.0;
    for (int64_t i = 0; i < n; ++i) {
        double a[3], b[3];
        shift_inverse(R + 9 * i, dt + 3 * i, e_r, a);
        shift_inverse(R + 9 * i, dt + 3 * i, e_r, b, 1.0 / e_r);
        for (int k = 0; k < 3; ++k) worst = std::fmax(worst, std::fabs(a[k] - b[k]) + (a[k] != b[k] ? 1.0 : 0.0));
    }
    return worst;
}

// Same per-cell math as place_windows_kernel: all W^3 cells of one (R, dt).
void hc_window(const double* R, const double* dt, const float* grid, const int32_t* gdims, const double* gext,
               const double* gres, float d_far, const double* P, int Wmax, const int32_t* W, const uint8_t* mask,
               double e_r, float* out) {
    GridView g{grid, gdims[0], gdims[1], gdims[2], d_far, gext[0], gext[1], gext[2], gres[0], gres[1], gres[2]};
    auto load = [&](int64_t i) { return grid[i]; };
    double dtinv[3];
    shift_inverse(R, dt, e_r, dtinv);
    const int n = W[0] * W[1] * W[2];
    for (int cell = 0; cell < n; ++cell) {
        if (!mask[cell]) {
            out[cell] = d_far;
            continue;
        }
        const int mx = cell % W[0], my = (cell / W[0]) % W[1], mz = cell / (W[0] * W[1]);
        double pt[3];
        window_point(P[mx], P[Wmax + my], P[2 * Wmax + mz], R, dtinv, e_r, pt);
        out[cell] = trilinear_at(g, pt[0], pt[1], pt[2], load);
    }
}

void hc_trilinear(const float* grid, const int32_t* gdims, const double* gext, const double* gres, float d_far,
                  const double* pts, int64_t n, float* out) {
    GridView g{grid, gdims[0], gdims[1], gdims[2], d_far, gext[0], gext[1], gext[2], gres[0], gres[1], gres[2]};
    auto load = [&](int64_t i) { return grid[i]; };
    for (int64_t i = 0; i < n; ++i) out[i] = trilinear_at(g, pts[3 * i], pts[3 * i + 1], pts[3 * i + 2], load);
}

void hc_primitive_grid(int kind, const double* prm, const double* ext, const double* res, const int32_t* dims,
                       float* out) {
    const int64_t n = (int64_t)dims[0] * dims[1] * dims[2];
    for (int64_t cell = 0; cell < n; ++cell) {
        const int64_t ix = cell % dims[0], iy = (cell / dims[0]) % dims[1], iz = cell / ((int64_t)dims[0] * dims[1]);
        const double x = DADD(-ext[0], DMUL(DADD((double)ix, 0.5), res[0]));
        const double y = DADD(-ext[1], DMUL(DADD((double)iy, 0.5), res[1]));
        const double z = DADD(-ext[2], DMUL(DADD((double)iz, 0.5), res[2]));
        out[cell] = (float)primitive_at(kind, prm, x, y, z);
    }
}

static const double kDirs[4][3] = {
    {0.577350269, 0.577350269, 0.577350269},
    {0.267261242, 0.534522484, 0.801783726},
    {-0.455842306, 0.569802882, 0.683763459},
    {0.816496581, -0.408248290, 0.408248290},
};

void hc_mesh_grid(const double* tri, int n_tri, int is_signed, const double* ext, const double* res,
                  const int32_t* dims, float* out) {
    RayTri* rays = new RayTri[4 * n_tri];
    for (int d = 0; d < 4; ++d)
        for (int t = 0; t < n_tri; ++t) {
            const double* a = tri + 9 * t;
            RayTri& r = rays[d * n_tri + t];
            for (int k = 0; k < 3; ++k) {
                r.a[k] = a[k];
                r.e1[k] = DSUB(a[3 + k], a[k]);
                r.e2[k] = DSUB(a[6 + k], a[k]);
            }
            cross3(kDirs[d], r.e2, r.h);
            const double det = dot3(r.e1[0], r.e1[1], r.e1[2], r.h[0], r.h[1], r.h[2]);
            r.parallel = std::fabs(det) < 1e-12;
            r.det = r.parallel ? 1.0 : det;
        }
    const int64_t n = (int64_t)dims[0] * dims[1] * dims[2];
    for (int64_t cell = 0; cell < n; ++cell) {
        const int64_t ix = cell % dims[0], iy = (cell / dims[0]) % dims[1], iz = cell / ((int64_t)dims[0] * dims[1]);
        const double p[3] = {DADD(-ext[0], DMUL(DADD((double)ix, 0.5), res[0])),
                             DADD(-ext[1], DMUL(DADD((double)iy, 0.5), res[1])),
                             DADD(-ext[2], DMUL(DADD((double)iz, 0.5), res[2]))};
        double best = INFINITY;
        for (int t = 0; t < n_tri; ++t) {
            const double* tr = tri + 9 * t;
            const double d2 = closest_sq(p, tr, tr + 3, tr + 6);
            best = d2 < best ? d2 : best;
        }
        double d = std::sqrt(best);
        if (is_signed) {
            bool inside = false;
            for (int dir = 0; dir < 4; ++dir) {
                int count = 0;
                bool suspect = false;
                for (int t = 0; t < n_tri; ++t) {
                    const int h = ray_cross(p, rays[dir * n_tri + t], kDirs[dir]);
                    count += h != 0;
                    suspect |= h == 2;
                }
                if (!suspect) {
                    inside = count & 1;
                    break;
                }
            }
            if (inside) d = -d;
        }
        out[cell] = (float)d;
    }
    delete[] rays;
}

void hc_mlp(const float* w1, const float* b1, const float* w2, const float* b2, int H, int64_t n_out,
            const double* R, int64_t B, float* y) {
    float h[64];
    for (int64_t r = 0; r < B; ++r) {
        for (int j = 0; j < H; ++j) {
            float acc = (float)R[r * 9] * w1[j];
            for (int k = 1; k < 9; ++k) acc = std::fma((float)R[r * 9 + k], w1[k * H + j], acc);
            acc = acc + b1[j];
            h[j] = acc > 0.0f ? acc : 0.0f;
        }
        for (int64_t n = 0; n < n_out; ++n) {
            float acc = h[0] * w2[n];
            for (int k = 1; k < H; ++k) acc = std::fma(h[k], w2[(int64_t)k * n_out + n], acc);
            y[r * n_out + n] = acc + b2[n];
        }
    }
}

}  // extern "C"
