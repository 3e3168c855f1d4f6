/*
 * biodiff_oracle.c — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C, single-threaded restatement of the reference's LOD diffusion
 * step and cell source/sink step (arxiv 2110.13368 re-implementation,
 * /root/reference/proj/src/core). It is the CHECKER for the CUDA product
 * path: only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg
 * may load it. Nothing in paper_2110_13368_b200/ links or calls it.
 *
 * Parity pinning: tests/test_oracle.py checks this file bit-for-bit against
 * the reference itself compiled from /root/reference (oracle/_ref, built by
 * oracle/Makefile) and against the committed fixtures in tests/golden/
 * (generated from oracle/_ref by tests/golden/make_golden.py).
 *
 * Floating point: compiled with -O2 -ffp-contract=off so every a*b+c is two
 * rounded operations, matching the reference Release build (no -march, so no
 * FMA on x86-64; SURVEY.md §7 hard part 1). Operand order below follows the
 * C++ expressions literally (left-to-right evaluation).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

/* solver.cpp:47-97 precompute_thomas_coefficients (one axis).
 * q[s] = dt*D/(h*h); decay = 1 + dt*lambda/dims;
 * diag(i): n==1 -> decay; ends -> decay+q; interior -> decay+2q  (solver.cpp:79-82)
 * denom_inv[0] = 1/diag(0); c_back[0] = n>1 ? q*denom_inv[0] : 0   (solver.cpp:84-87)
 * i>=1: denom = diag(i) - q*c_back[i-1]; denom_inv[i] = 1/denom;
 *       c_back[i] = q*denom_inv[i] for i < n-1, else 0             (solver.cpp:88-94)
 * Returns 0, or 1 on invalid arguments (solver.cpp:51-56). */
int orc_precompute(int n, int S, const double* D, const double* lambda, double h, double dt, int dims,
                   double* off_diag, double* denom_inv, double* c_back)
{
    if (!(dt > 0.0) || dims < 1 || dims > 3 || S < 1 || n < 1) return 1;
    memset(denom_inv, 0, sizeof(double) * (size_t)n * S);
    memset(c_back, 0, sizeof(double) * (size_t)n * S);
    for (int s = 0; s < S; ++s) {
        const double q = dt * D[s] / (h * h);
        const double decay = 1.0 + dt * lambda[s] / (double)dims;
        off_diag[s] = q;
        double denom = (n == 1) ? decay : decay + q;
        denom_inv[s] = 1.0 / denom;
        c_back[s] = (n > 1) ? q * denom_inv[s] : 0.0;
        for (int i = 1; i < n; ++i) {
            const double diag = (i == n - 1) ? decay + q : decay + 2.0 * q;
            denom = diag - q * c_back[(size_t)(i - 1) * S + s];
            const double dinv = 1.0 / denom;
            denom_inv[(size_t)i * S + s] = dinv;
            if (i < n - 1) c_back[(size_t)i * S + s] = q * dinv;
        }
    }
    return 0;
}

/* One strided line: element m lives at v[m*stride]. The per-element ops are
 * solver.cpp:17-19 (fwd_first, fwd, bwd); the loop shape is thomas_solve
 * solver.cpp:99-126 restated for one substrate. */
static void line_solve(double* v, long stride, int n, int S, int s, double q, const double* dinv, const double* cb)
{
    v[0] = v[0] * dinv[s];
    for (int i = 1; i < n; ++i)
        v[(long)i * stride] = (v[(long)i * stride] + q * v[(long)(i - 1) * stride]) * dinv[(size_t)i * S + s];
    for (int i = n - 2; i >= 0; --i)
        v[(long)i * stride] = v[(long)i * stride] + cb[(size_t)i * S + s] * v[(long)(i + 1) * stride];
}

/* solver.cpp:130-244 sweep_x / sweep_y / sweep_z. Lines are disjoint so the
 * per-line restatement is bitwise equal to the reference's chunked loops
 * (backend.hpp:28-33). axis: 0=x, 1=y, 2=z.
 * Layout (mesh.hpp:59-61): rho[(i + j*nx + k*nx*ny)*S + s]. */
void orc_sweep(double* rho, int nx, int ny, int nz, int S, int axis,
               const double* q, const double* dinv, const double* cb)
{
    const long row = (long)nx * S, plane = row * ny;
    if (axis == 0) {
        for (long k = 0; k < nz; ++k)
            for (long j = 0; j < ny; ++j)
                for (int s = 0; s < S; ++s)
                    line_solve(rho + k * plane + j * row + s, S, nx, S, s, q[s], dinv, cb);
    } else if (axis == 1) {
        for (long k = 0; k < nz; ++k)
            for (long i = 0; i < nx; ++i)
                for (int s = 0; s < S; ++s)
                    line_solve(rho + k * plane + i * S + s, row, ny, S, s, q[s], dinv, cb);
    } else {
        for (long j = 0; j < ny; ++j)
            for (long i = 0; i < nx; ++i)
                for (int s = 0; s < S; ++s)
                    line_solve(rho + j * row + i * S + s, plane, nz, S, s, q[s], dinv, cb);
    }
}

/* solver.cpp:267-275 apply_dirichlet_conditions: masked overwrite per entry. */
void orc_dirichlet(double* rho, int S, int64_t count, const int64_t* voxel, const uint8_t* mask, const double* values)
{
    for (int64_t e = 0; e < count; ++e)
        for (int s = 0; s < S; ++s)
            if (mask[e * S + s]) rho[voxel[e] * S + s] = values[e * S + s];
}

/* mesh.cpp:72-88 nearest_voxel: floor((p-min)/h) clamped to [0, n-1].
 * Returns -1 when the position is outside [min, max] (mesh.cpp:66-70). */
int64_t orc_nearest_voxel(const double* bounds /* xmin,xmax,ymin,ymax,zmin,zmax */, const double* h,
                          const int* n, const double* p)
{
    for (int a = 0; a < 3; ++a)
        if (!(p[a] >= bounds[2 * a] && p[a] <= bounds[2 * a + 1])) return -1;
    int64_t idx[3];
    for (int a = 0; a < 3; ++a) {
        int c = (int)floor((p[a] - bounds[2 * a]) / h[a]);
        if (c < 0) c = 0;
        if (c > n[a] - 1) c = n[a] - 1;
        idx[a] = c;
    }
    return idx[0] + idx[1] * n[0] + idx[2] * (int64_t)n[0] * n[1];
}

typedef struct { int64_t voxel, id, index; } orc_key;
static int key_cmp(const void* a, const void* b)
{
    const orc_key* x = (const orc_key*)a;
    const orc_key* y = (const orc_key*)b;
    if (x->voxel != y->voxel) return x->voxel < y->voxel ? -1 : 1;
    if (x->id != y->id) return x->id < y->id ? -1 : 1;
    return 0;
}

/* agents.cpp:56-73 rebuild_voxel_grouping: sort agent indices by
 * (voxel, id), then cut into groups of equal voxel.
 * Outputs: group_voxel[G], group_offsets[G+1], order[N] (agent indices in
 * group order). Returns G, or -1 when an agent lies outside the mesh. */
int64_t orc_group(int64_t n_agents, const int64_t* ids, const double* positions, const double* bounds,
                  const double* h, const int* n, int64_t* group_voxel, int64_t* group_offsets, int64_t* order)
{
    orc_key* keys = (orc_key*)malloc(sizeof(orc_key) * (size_t)(n_agents > 0 ? n_agents : 1));
    for (int64_t a = 0; a < n_agents; ++a) {
        keys[a].voxel = orc_nearest_voxel(bounds, h, n, positions + 3 * a);
        if (keys[a].voxel < 0) { free(keys); return -1; }
        keys[a].id = ids[a];
        keys[a].index = a;
    }
    qsort(keys, (size_t)n_agents, sizeof(orc_key), key_cmp);
    int64_t G = 0;
    for (int64_t a = 0; a < n_agents; ++a) {
        if (G == 0 || group_voxel[G - 1] != keys[a].voxel) {
            group_voxel[G] = keys[a].voxel;
            group_offsets[G] = a;
            ++G;
        }
        order[a] = keys[a].index;
    }
    group_offsets[G] = n_agents;
    free(keys);
    return G;
}

/* agents.cpp:75-112 cell_sources_sinks_step. Agents are indexed through
 * order[] (group order); per-agent arrays are in the caller's agent order.
 * inv_voxel_volume = 1/((dx*dy)*dz) (agents.cpp:82, mesh.hpp:34);
 * f = dt*volume*inv (agents.cpp:102);
 * rho = (rho + f*sec*target) / (1 + f*(sec+upt)) (agents.cpp:106-107). */
void orc_sources(double* rho, int S, int64_t G, const int64_t* group_voxel, const int64_t* group_offsets,
                 const int64_t* order, const double* volume, const double* secretion, const double* uptake,
                 const double* saturation, double dt, double inv_voxel_volume)
{
    for (int64_t g = 0; g < G; ++g) {
        double* r = rho + group_voxel[g] * S;
        for (int64_t m = group_offsets[g]; m < group_offsets[g + 1]; ++m) {
            const int64_t a = order[m];
            const double f = dt * volume[a] * inv_voxel_volume;
            for (int s = 0; s < S; ++s) {
                const double sec = secretion[a * S + s];
                const double upt = uptake[a * S + s];
                r[s] = (r[s] + f * sec * saturation[a * S + s]) / (1.0 + f * (sec + upt));
            }
        }
    }
}

/* solver.cpp:289-299 diffuse_decay_step: x, y if ny>1, z if nz>1, then the
 * Dirichlet clamp. ws_* point at the per-axis (q, dinv, cb) arrays. */
void orc_diffuse_decay_step(double* rho, int nx, int ny, int nz, int S,
                            const double* qx, const double* dx_, const double* cx,
                            const double* qy, const double* dy_, const double* cy,
                            const double* qz, const double* dz_, const double* cz,
                            int64_t n_dir, const int64_t* dir_voxel, const uint8_t* dir_mask, const double* dir_values)
{
    orc_sweep(rho, nx, ny, nz, S, 0, qx, dx_, cx);
    if (ny > 1) orc_sweep(rho, nx, ny, nz, S, 1, qy, dy_, cy);
    if (nz > 1) orc_sweep(rho, nx, ny, nz, S, 2, qz, dz_, cz);
    orc_dirichlet(rho, S, n_dir, dir_voxel, dir_mask, dir_values);
}
