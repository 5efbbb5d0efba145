/*
 * CPU oracle (C restatement) of the shallow-water hot path.
 * TEST INFRASTRUCTURE ONLY: loaded by tests/, __graft_entry__.smoke() and
 * bench.py's CPU-baseline / --impl reference legs.  Never linked into the
 * product library.
 *
 * Restates oracle/sw_oracle.py:wave_advance (the DSL kernel
 * kernels/wave_advance.fk under refinterp semantics) with
 * the SAME per-op IEEE order, so results are bit-identical to the numpy
 * oracle (checked in tests/test_oracle.py).  Compile with
 * -ffp-contract=off and without -ffast-math (see oracle/Makefile).
 * Boundary fill follows oracle/sw_oracle.py:apply_boundary.
 *
 * Layout: row-major full arrays (ny+2) x pitch, element (x,y) at
 * y*pitch + x, halo [1,1,1,1] (field.py:25-60, region.py:1-6).
 * Rows are split into bands over POSIX threads.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>
#include <pthread.h>
#include <unistd.h>

#define DEFINE_STEP(T, SUF)                                                      \
static inline T fxu_##SUF(T g2, T h, T q) { return ((q * q) / h) + ((g2 * h) * h); } \
static inline T cross_##SUF(T h, T u, T v) { return (u * v) / h; }              \
                                                                                 \
static void band_##SUF(int nx, long pitch, int y0, int y1,                       \
                       const T* H, const T* U, const T* V,                       \
                       T* oH, T* oU, T* oV, T half, T cx2, T cy2, T cx, T cy,   \
                       T g2, T* fx, T* fyA, T* fyB)                              \
{                                                                                \
    /* fyA: y-face below current row (3 x nx: Vy, cross(Hy,Uy,Vy), fxu(Hy,Vy)) */ \
    T* ydn = fyA; T* yup = fyB;                                                  \
    for (int y = y0; y <= y1; ++y) {                                             \
        /* y-face between rows y and y+1 (row y is "dn") */                      \
        const T *Hd = H + (long)y * pitch, *Ud = U + (long)y * pitch,           \
                *Vd = V + (long)y * pitch;                                       \
        const T *Hu = Hd + pitch, *Uu = Ud + pitch, *Vu = Vd + pitch;            \
        for (int x = 1; x <= nx; ++x) {                                          \
            T hD = Hd[x], uD = Ud[x], vD = Vd[x];                                \
            T hU = Hu[x], uU = Uu[x], vU = Vu[x];                                \
            T Hy = (half * (hD + hU)) + (cy2 * (vD - vU));                       \
            T Uy = (half * (uD + uU)) + (cy2 * (cross_##SUF(hD, uD, vD) - cross_##SUF(hU, uU, vU))); \
            T Vy = (half * (vD + vU)) + (cy2 * (fxu_##SUF(g2, hD, vD) - fxu_##SUF(g2, hU, vU))); \
            yup[x - 1] = Vy;                                                     \
            yup[nx + x - 1] = cross_##SUF(Hy, Uy, Vy);                           \
            yup[2 * nx + x - 1] = fxu_##SUF(g2, Hy, Vy);                         \
        }                                                                        \
        if (y >= y0 + 1) {                                                       \
            /* update row yc = y (interior row) using faces y-1/2 (ydn), y+1/2 (yup) */ \
            int yc = y;                                                          \
            const T *Hc = H + (long)yc * pitch, *Uc = U + (long)yc * pitch,     \
                    *Vc = V + (long)yc * pitch;                                  \
            for (int x = 0; x <= nx; ++x) { /* x-face between x and x+1 */      \
                T hL = Hc[x], uL = Uc[x], vL = Vc[x];                            \
                T hR = Hc[x + 1], uR = Uc[x + 1], vR = Vc[x + 1];                \
                T Hx = (half * (hL + hR)) + (cx2 * (uL - uR));                   \
                T Ux = (half * (uL + uR)) + (cx2 * (fxu_##SUF(g2, hL, uL) - fxu_##SUF(g2, hR, uR))); \
                T Vx = (half * (vL + vR)) + (cx2 * (cross_##SUF(hL, uL, vL) - cross_##SUF(hR, uR, vR))); \
                fx[x] = Ux;                                                      \
                fx[nx + 1 + x] = fxu_##SUF(g2, Hx, Ux);                          \
                fx[2 * (nx + 1) + x] = cross_##SUF(Hx, Ux, Vx);                  \
            }                                                                    \
            T *ph = oH + (long)yc * pitch, *pu = oU + (long)yc * pitch,         \
              *pv = oV + (long)yc * pitch;                                       \
            for (int x = 1; x <= nx; ++x) {                                      \
                ph[x] = (Hc[x] + (cx * (fx[x - 1] - fx[x]))) +                   \
                        (cy * (ydn[x - 1] - yup[x - 1]));                        \
                pu[x] = (Uc[x] + (cx * (fx[nx + 1 + x - 1] - fx[nx + 1 + x]))) + \
                        (cy * (ydn[nx + x - 1] - yup[nx + x - 1]));              \
                pv[x] = (Vc[x] + (cx * (fx[2 * (nx + 1) + x - 1] - fx[2 * (nx + 1) + x]))) + \
                        (cy * (ydn[2 * nx + x - 1] - yup[2 * nx + x - 1]));      \
            }                                                                    \
        }                                                                        \
        T* t_ = ydn; ydn = yup; yup = t_;                                        \
    }                                                                            \
}                                                                                \
                                                                                 \
static void boundary_##SUF(int nx, int ny, long p, T* H, T* U, T* V, int bc)    \
{                                                                                \
    if (bc == 0) { /* reflective */                                              \
        for (int y = 1; y <= ny; ++y) {                                          \
            long r = (long)y * p;                                                \
            H[r] = H[r + 1];           H[r + nx + 1] = H[r + nx];               \
            U[r] = -U[r + 1];          U[r + nx + 1] = -U[r + nx];              \
            V[r] = V[r + 1];           V[r + nx + 1] = V[r + nx];               \
        }                                                                        \
        long t = (long)(ny + 1) * p;                                             \
        for (int x = 0; x <= nx + 1; ++x) {                                      \
            H[x] = H[p + x];   H[t + x] = H[t - p + x];                          \
            U[x] = U[p + x];   U[t + x] = U[t - p + x];                          \
            V[x] = -V[p + x];  V[t + x] = -V[t - p + x];                         \
        }                                                                        \
    } else { /* periodic */                                                      \
        T* A[3] = {H, U, V};                                                     \
        for (int k = 0; k < 3; ++k) {                                            \
            T* a = A[k];                                                         \
            for (int y = 1; y <= ny; ++y) {                                      \
                long r = (long)y * p;                                            \
                a[r] = a[r + nx]; a[r + nx + 1] = a[r + 1];                      \
            }                                                                    \
            long t = (long)(ny + 1) * p;                                         \
            for (int x = 0; x <= nx + 1; ++x) {                                  \
                a[x] = a[(long)ny * p + x]; a[t + x] = a[p + x];                \
            }                                                                    \
        }                                                                        \
    }                                                                            \
}                                                                                \
                                                                                 \
struct job_##SUF {                                                               \
    int nx; long pitch; int r0, r1;                                              \
    const T *H, *U, *V; T *oH, *oU, *oV;                                         \
    T half, cx2, cy2, cx, cy, g2; int err;                                       \
};                                                                               \
static void* run_job_##SUF(void* p)                                              \
{                                                                                \
    struct job_##SUF* j = (struct job_##SUF*)p;                                  \
    int nx = j->nx;                                                              \
    T* s = (T*)malloc(sizeof(T) * (size_t)(3 * (nx + 1) + 6 * nx));             \
    if (!s) { j->err = 1; return NULL; }                                         \
    band_##SUF(nx, j->pitch, j->r0 - 1, j->r1, j->H, j->U, j->V, j->oH, j->oU,  \
               j->oV, j->half, j->cx2, j->cy2, j->cx, j->cy, j->g2, s,          \
               s + 3 * (nx + 1), s + 3 * (nx + 1) + 3 * nx);                     \
    free(s);                                                                     \
    j->err = 0;                                                                  \
    return NULL;                                                                 \
}                                                                                \
                                                                                 \
int sw_oracle_step_##SUF(int nx, int ny, long pitch,                            \
                         const T* H, const T* U, const T* V,                     \
                         T* oH, T* oU, T* oV, T dx, T dy, T dt, T g, int bc,    \
                         int nthreads)                                           \
{                                                                                \
    if (nx < 1 || ny < 1 || pitch < nx + 2) return 2;                            \
    T half = (T)0.5;                                                             \
    T cx2 = (half * dt) / dx, cy2 = (half * dt) / dy;                            \
    T cx = dt / dx, cy = dt / dy, g2 = half * g;                                 \
    int nt = nthreads > 0 ? nthreads : 1;                                        \
    if (nt > ny) nt = ny;                                                        \
    if (nt > 256) nt = 256;                                                      \
    struct job_##SUF jobs[256];                                                  \
    pthread_t tids[256];                                                         \
    int err = 0;                                                                 \
    for (int b = 0; b < nt; ++b) {                                               \
        struct job_##SUF j = {nx, pitch, 1 + (int)((long)ny * b / nt),           \
                              (int)((long)ny * (b + 1) / nt), H, U, V, oH, oU, oV, \
                              half, cx2, cy2, cx, cy, g2, 0};                     \
        jobs[b] = j;                                                             \
    }                                                                            \
    for (int b = 1; b < nt; ++b)                                                 \
        if (pthread_create(&tids[b], NULL, run_job_##SUF, &jobs[b])) jobs[b].err = -1; \
    run_job_##SUF(&jobs[0]);                                                     \
    for (int b = 1; b < nt; ++b) {                                               \
        if (jobs[b].err == -1) { run_job_##SUF(&jobs[b]); continue; }           \
        pthread_join(tids[b], NULL);                                             \
    }                                                                            \
    for (int b = 0; b < nt; ++b) err |= jobs[b].err;                             \
    if (err) return 3;                                                           \
    boundary_##SUF(nx, ny, pitch, oH, oU, oV, bc);                               \
    return 0;                                                                    \
}                                                                                \
                                                                                 \
int sw_oracle_boundary_##SUF(int nx, int ny, long pitch, T* H, T* U, T* V, int bc) \
{                                                                                \
    boundary_##SUF(nx, ny, pitch, H, U, V, bc);                                  \
    return 0;                                                                    \
}

DEFINE_STEP(float, f32)
DEFINE_STEP(double, f64)

int sw_oracle_max_threads(void)
{
    long n = sysconf(_SC_NPROCESSORS_ONLN);
    return n > 0 ? (int)n : 1;
}
