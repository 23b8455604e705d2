/*
 * abi_demo.c — one real-time distance cycle driven through the C ABI alone.
 *
 * Plain C99 against include/linksdf_b200.h and the CUDA runtime: no Python,
 * no torch in the process.  This is what a C/C++ host of the checker (a
 * robot controller, a planner) links: it uploads the link SDF grids and the
 * window tables once, then per cycle runs
 *     lsdf_fk_align -> lsdf_voxelize -> lsdf_query_direct
 * (forward_kinematics_batch robot.py:305-347 + compute_alignment
 * placement.py:60-99, voxelize_pointcloud query.py:106-125, the fused
 * query_min_distances query.py:128-150) and writes d / link / voxel.
 *
 * The host-side constants (chain table, window tables, segment bounds) come
 * from a scene file written by tests/native/abi_scene.py — the same numpy
 * recipes the Python facade uses; tests/test_gpu_parity.py compares the
 * output with the oracle bit for bit.
 *
 *   abi_demo scene.bin out.bin
 *
 * Scene file: "LSDFABI1", then sections of (u64 nbytes, bytes):
 *   header {i32 n_links, n_geo, C, D, N, repeat; f64 d_far_global}
 *   lsdf_link[n_links], limits f64 (D, 2), lsdf_env_grid
 *   per geometry link: lsdf_link_grid (pointers zero), values f32
 *   lsdf_window (pointers zero), P f64, zrange i16 (may be empty),
 *   mask_bits u32, shell_cells u32, shell_radius f32
 *   q f64 (C, D), points f32 or f64 (N, 3) (told apart by the section size)
 * Output: d f32 (C), link i32 (C), voxel i32 (C), flags i32 (2).
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime.h>

#include "linksdf_b200.h"

#define DIE(...) do { fprintf(stderr, __VA_ARGS__); fputc('\n', stderr); exit(1); } while (0)
#define CUDA(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) DIE("%s: %s", #x, cudaGetErrorString(e_)); } while (0)
#define LSDF(x) do { int s_ = (x); if (s_ != LSDF_OK) DIE("%s -> %d: %s", #x, s_, lsdf_last_error()); } while (0)

typedef struct {
    int32_t n_links, n_geo, C, D, N, repeat;
    double d_far_global;
} scene_header;

static void* read_section(FILE* f, uint64_t* nbytes) {
    uint64_t n;
    if (fread(&n, 8, 1, f) != 1) DIE("truncated scene file");
    void* buf = malloc(n ? n : 1);
    if (!buf) DIE("out of host memory");
    if (n && fread(buf, 1, n, f) != n) DIE("truncated scene section");
    *nbytes = n;
    return buf;
}

static void* read_exact(FILE* f, uint64_t want, const char* what) {
    uint64_t n;
    void* buf = read_section(f, &n);
    if (n != want) DIE("section %s: %llu bytes, expected %llu", what, (unsigned long long)n,
                       (unsigned long long)want);
    return buf;
}

/* host section -> fresh device buffer (NULL for an empty section) */
static void* upload(FILE* f, uint64_t* nbytes) {
    void* host = read_section(f, nbytes);
    void* dev = NULL;
    if (*nbytes) {
        CUDA(cudaMalloc(&dev, *nbytes));
        CUDA(cudaMemcpy(dev, host, *nbytes, cudaMemcpyHostToDevice));
    }
    free(host);
    return dev;
}

int main(int argc, char** argv) {
    if (argc != 3) DIE("usage: %s scene.bin out.bin", argv[0]);
    FILE* f = fopen(argv[1], "rb");
    if (!f) DIE("cannot open %s", argv[1]);
    char magic[8];
    if (fread(magic, 1, 8, f) != 8 || memcmp(magic, "LSDFABI1", 8) != 0) DIE("not a scene file");
    printf("%s\n", lsdf_version());

    scene_header* h = (scene_header*)read_exact(f, sizeof(scene_header), "header");
    const int64_t C = h->C;
    lsdf_link* links = (lsdf_link*)read_exact(f, sizeof(lsdf_link) * (uint64_t)h->n_links, "links");
    uint64_t nb;
    double* limits_dev = (double*)upload(f, &nb);
    lsdf_env_grid* env = (lsdf_env_grid*)read_exact(f, sizeof(lsdf_env_grid), "env");

    cudaStream_t stream;
    CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));

    lsdf_link_grid grids[LSDF_MAX_LINKS];
    if (h->n_geo > LSDF_MAX_LINKS) DIE("too many geometry links");
    for (int g = 0; g < h->n_geo; ++g) {
        lsdf_link_grid* s = (lsdf_link_grid*)read_exact(f, sizeof(lsdf_link_grid), "link grid");
        grids[g] = *s;
        free(s);
        grids[g].values_dev = (const float*)upload(f, &nb);
        const int64_t cells = (int64_t)(grids[g].dims[0] - 1) * (grids[g].dims[1] - 1) * (grids[g].dims[2] - 1);
        float* packed = NULL;
        CUDA(cudaMalloc((void**)&packed, (size_t)cells * 8 * sizeof(float)));
        LSDF(lsdf_pack_corners(grids[g].values_dev, grids[g].dims, packed, stream));
        grids[g].packed_dev = packed;
    }

    lsdf_window* w = (lsdf_window*)read_exact(f, sizeof(lsdf_window), "window");
    w->P_dev = (const double*)upload(f, &nb);
    w->zrange_dev = (const int16_t*)upload(f, &nb);
    w->mask_bits_dev = (const uint32_t*)upload(f, &nb);
    w->shell_cells_dev = (const uint32_t*)upload(f, &nb);
    w->shell_radius_dev = (const float*)upload(f, &nb);

    double* q_dev = (double*)upload(f, &nb);
    if (nb != sizeof(double) * (uint64_t)C * h->D) DIE("q section size");
    void* pts_dev = upload(f, &nb);
    const int32_t pts_f32 = nb == sizeof(float) * 3 * (uint64_t)h->N;
    if (!pts_f32 && nb != sizeof(double) * 3 * (uint64_t)h->N) DIE("points section size");
    fclose(f);

    /* per-cycle buffers: allocated once, reused by every cycle */
    const int64_t G = h->n_geo;
    double *R_geo, *dt_geo;
    int32_t *anchor_geo, *flags, *link, *voxel;
    float* d;
    void *occ, *ws;
    CUDA(cudaMalloc((void**)&R_geo, sizeof(double) * 9 * C * G));
    CUDA(cudaMalloc((void**)&dt_geo, sizeof(double) * 3 * C * G));
    CUDA(cudaMalloc((void**)&anchor_geo, sizeof(int32_t) * 3 * C * G));
    CUDA(cudaMalloc((void**)&flags, sizeof(int32_t) * 4));
    CUDA(cudaMalloc((void**)&d, sizeof(float) * C));
    CUDA(cudaMalloc((void**)&link, sizeof(int32_t) * C));
    CUDA(cudaMalloc((void**)&voxel, sizeof(int32_t) * C));
    const int64_t occ_bytes = lsdf_occupancy_bytes(env);
    const int64_t ws_bytes = lsdf_query_workspace_bytes(C, h->n_geo);
    if (occ_bytes <= 0 || ws_bytes <= 0) DIE("workspace sizing: %s", lsdf_last_error());
    CUDA(cudaMalloc(&occ, (size_t)occ_bytes));
    CUDA(cudaMalloc(&ws, (size_t)ws_bytes));
    CUDA(cudaMemsetAsync(ws, 0, (size_t)ws_bytes, stream)); /* zeroed once; each query re-zeroes it */

    int32_t h_flags[4];
    const uint64_t launches0 = lsdf_launch_count();
    for (int cycle = 0; cycle < (h->repeat > 0 ? h->repeat : 1); ++cycle) {
        LSDF(lsdf_fk_align(links, h->n_links, h->n_geo, q_dev, C, h->D, limits_dev, env, w->W,
                           NULL, NULL, R_geo, dt_geo, anchor_geo, flags, stream));
        LSDF(lsdf_voxelize(pts_dev, pts_f32, h->N, env, occ, NULL, stream));
        LSDF(lsdf_query_direct(R_geo, dt_geo, anchor_geo, C, h->n_geo, grids, w, env, occ,
                               0, h->d_far_global, ws, d, link, voxel, NULL, stream));
    }
    CUDA(cudaMemcpyAsync(h_flags, flags, sizeof(h_flags), cudaMemcpyDeviceToHost, stream));
    CUDA(cudaStreamSynchronize(stream));
    printf("cycles %d, kernels enqueued %llu, limit violations %d, windows off-grid %d\n",
           h->repeat > 0 ? h->repeat : 1, (unsigned long long)(lsdf_launch_count() - launches0),
           h_flags[0], h_flags[1]);

    float* hd = (float*)malloc(sizeof(float) * C);
    int32_t* hl = (int32_t*)malloc(sizeof(int32_t) * C);
    int32_t* hv = (int32_t*)malloc(sizeof(int32_t) * C);
    CUDA(cudaMemcpy(hd, d, sizeof(float) * C, cudaMemcpyDeviceToHost));
    CUDA(cudaMemcpy(hl, link, sizeof(int32_t) * C, cudaMemcpyDeviceToHost));
    CUDA(cudaMemcpy(hv, voxel, sizeof(int32_t) * C, cudaMemcpyDeviceToHost));
    FILE* o = fopen(argv[2], "wb");
    if (!o) DIE("cannot write %s", argv[2]);
    fwrite(hd, sizeof(float), (size_t)C, o);
    fwrite(hl, sizeof(int32_t), (size_t)C, o);
    fwrite(hv, sizeof(int32_t), (size_t)C, o);
    fwrite(h_flags, sizeof(int32_t), 2, o);
    fclose(o);
    float dmin = hd[0];
    for (int64_t c = 1; c < C; ++c) dmin = hd[c] < dmin ? hd[c] : dmin;
    printf("%lld waypoints, min distance %.6f m\n", (long long)C, dmin);
    return 0;
}
