// sw_resident.cuh -- the whole time loop of a SMALL grid in one launch:
// a thread-block cluster (up to 16 CTAs, one per SM) keeps the state in
// shared memory and iterates the steps on chip.
//
// Why: below ~512^2 a step is a few microseconds of work, and a launch per
// step -- even replayed from a CUDA graph -- costs about as much as the work
// (B200: 128^2 runs 2.3 us / step in a graph, profiles/r01/grid_sweep.json).
// Here a step costs its arithmetic plus one cluster barrier (~0.2 us).
//
// Work split.  CTA b of the cluster owns a band of R_b consecutive rows
// (full width).  Its shared memory holds the band plus one halo row above
// and below (S: h, hu, hv records), the x-faces of the band rows (FX) and
// the y-faces between them (FY).  A step is two CTA-wide phases separated
// by __syncthreads:
//   B  every face once: x-faces (nx+1 per band row), y-faces (nx per row
//      boundary, including the two band edges), the cell quantities they
//      need computed in registers;
//   C  the conservative update of the band cells IN PLACE (only phase C
//      reads S's interior, and each thread reads then writes its own cells),
//      the column halos per boundary condition, the fused reductions, and
//      the band's first / last rows pushed into the neighbouring CTAs'
//      halo-row buffers through distributed shared memory (DSMEM), double-
//      buffered by step parity so a neighbour still reading the current
//      step's halo is never overwritten.
// One cluster barrier (release / acquire) ends the step; with a CFL-chosen
// dt every CTA then reads the cluster's minimum bound from the CTAs' slots
// (DSMEM, parity-buffered) -- no host and no global-memory round trip.
//
// Arithmetic: the same per-cell / per-face functions as every other kernel
// (sw_math.cuh cell_q / x_face / y_face / update_cell; exact mode with IEEE
// division), so exact mode is bit-identical to the oracle.  The reductions
// of each step go to the caller's slot rows exactly like the step kernels'.
// The final state is written to the buffer fkc_sw_advance_n's double-
// buffering contract names; the host then fills its halo rows / corners
// with the boundary kernel (== apply_boundary of the new state).
#pragma once
#include "sw_kernels.cuh"

namespace fkc {

#ifndef FKC_RES_THREADS
#define FKC_RES_THREADS 512
#endif
constexpr int RES_THREADS = FKC_RES_THREADS;
enum { FKC_RES_ERR_DEPTH = 1u, FKC_RES_ERR_NONFINITE = 2u, FKC_RES_ERR_FACE = 8u };   // include/fkc_sw.h fkc_err_bits
constexpr int RES_MAX_CLUSTER = 16;

// A cell / face record in shared memory: (h, hu, hv) or (F_h, F_hu, F_hv)
// plus a pad word, so one 16-byte vector access moves it (f32; two for f64)
// and the fields need one address between them.
template <class T> struct alignas(4 * sizeof(T)) Q4 {
    T a, b, c, d;
};

// shared-memory layout of one CTA (record offsets; every CTA of the cluster
// uses the same layout, so a local address is valid in DSMEM too)
struct ResLayout {
    int nx, R, W;                  // interior width, rows of the largest band, row length nx + 2
    int s, fx, fy, hb, n;          // bases (records) and total
    __host__ __device__ ResLayout(int nx_, int R_) : nx(nx_), R(R_), W(nx_ + 2) {
        s = 0;                                   // state S: (R + 2) x W
        fx = s + (R + 2) * W;                    // x-faces: R x (nx + 1)
        fy = fx + R * (nx + 1);                  // y-faces: (R + 1) x nx
        hb = fy + (R + 1) * nx;                  // halo rows [parity][side 0 bottom / 1 top][x - 1]
        n = hb + 2 * 2 * nx;
    }
    __host__ __device__ int S(int j, int x) const { return s + j * W + x; }
    __host__ __device__ int FX(int j, int i) const { return fx + j * (nx + 1) + i; }
    __host__ __device__ int FY(int j, int x) const { return fy + j * nx + x; }
    __host__ __device__ int HB(int p, int side, int x) const { return hb + (p * 2 + side) * nx + x; }
};

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t dsmem_addr(uint32_t local, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
    return r;
}
template <class T>
__device__ __forceinline__ void st_dsmem(uint32_t a, T v) {
    if constexpr (sizeof(T) == 4) asm volatile("st.shared::cluster.f32 [%0], %1;" :: "r"(a), "f"(v) : "memory");
    else asm volatile("st.shared::cluster.f64 [%0], %1;" :: "r"(a), "d"(v) : "memory");
}
template <class T>
__device__ __forceinline__ void st_dsmem_q(uint32_t a, const Q4<T>& q) {
    if constexpr (sizeof(T) == 4) {
        asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};" :: "r"(a), "f"(q.a), "f"(q.b), "f"(q.c), "f"(q.d)
                     : "memory");
    } else {
        asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" :: "r"(a), "d"(q.a), "d"(q.b) : "memory");
        asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" :: "r"(a + 16), "d"(q.c), "d"(q.d) : "memory");
    }
}
template <class T>
__device__ __forceinline__ T ld_dsmem(uint32_t a) {
    T v;
    if constexpr (sizeof(T) == 4) asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(a) : "memory");
    else asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ void cluster_barrier() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// (row, column) walk over a region `w` columns wide with stride nt without
// a division per element: thread tid starts at element tid
struct RegionIter {
    int j, x, dj, dx, w;
    __device__ __forceinline__ RegionIter(int tid, int nt, int w_) : w(w_) {
        j = tid / w; x = tid % w; dj = nt / w; dx = nt % w;
    }
    __device__ __forceinline__ void next() {
        j += dj; x += dx;
        if (x >= w) { x -= w; ++j; }
    }
};

template <class T, int D>
__device__ __forceinline__ CellQ<T> rcq(const Q4<T>& s, const Coef<T>& c, bool& ok) {
    return cell_q<T, D>(s.a, s.b, s.c, c, ok);
}

struct ResArgs {
    int nx, ny;
    int64_t pitch;
    const void* in[3];     // state at global step `first` (fresh halos)
    void* out[3];          // buffer that receives the final state
    double dx, dy, g, dt, cfl;
    int dt_from_slots, want_cfl;
    BCs bc;
    int64_t first, steps;
    unsigned long long* slots;   // 5 words per state row (mass, max|hu|, max|hv|, cfl bound, err), or null
};

template <class T, int DM>
__global__ void __launch_bounds__(RES_THREADS, 1) sw_resident(const __grid_constant__ ResArgs a) {
    using Q = Q4<T>;
    extern __shared__ __align__(32) uint8_t res_smem[];
    Q* sm = (Q*)res_smem;
    __shared__ T s_cfl[2];                           // this CTA's CFL bound of the last two states
    __shared__ double s_mass[RES_THREADS / 32];      // warp partials
    __shared__ unsigned long long s_mx[RES_THREADS / 32][2];
    __shared__ T s_b[RES_THREADS / 32];
    __shared__ uint32_t s_err[RES_THREADS / 32];
    using B = typename std::conditional<sizeof(T) == 4, uint32_t, unsigned long long>::type;
    const int nb = (int)gridDim.x;                   // the grid is exactly one cluster
    const int b = (int)cluster_rank();
    const int nx = a.nx, ny = a.ny;
    const int base = ny / nb, extra = ny % nb;
    const int R = base + (b < extra ? 1 : 0);              // rows of this band
    const int r0 = 1 + b * base + min(b, extra);            // its first interior row
    const ResLayout L(nx, base + (extra ? 1 : 0));
    const int tid = threadIdx.x, nt = blockDim.x;
    const int lane = tid & 31, warp = tid >> 5;
    const T dx = T(a.dx), dy = T(a.dy), g = T(a.g), dmin = dx < dy ? dx : dy;
    const int below = b > 0 ? b - 1 : (a.bc.s[SIDE_D] == BC_PER ? nb - 1 : -1);
    const int above = b < nb - 1 ? b + 1 : (a.bc.s[SIDE_U] == BC_PER ? 0 : -1);
    const T* in[3] = {(const T*)a.in[0], (const T*)a.in[1], (const T*)a.in[2]};

    // initial load: band rows (columns 0 .. nx+1) into S, the two halo rows
    // (columns 1 .. nx) into the halo buffers of parity 0
    for (RegionIter it(tid, nt, L.W); it.j < R + 2; it.next()) {
        const int64_t go = (int64_t)(r0 - 1 + it.j) * a.pitch + it.x;
        const Q v{in[0][go], in[1][go], in[2][go], T(0)};
        if (it.j == 0 || it.j == R + 1) {
            if (it.x >= 1 && it.x <= nx) sm[L.HB(0, it.j ? 1 : 0, it.x - 1)] = v;
        } else {
            sm[L.S(it.j, it.x)] = v;
        }
    }
    if (tid < 2) s_cfl[tid] = T(INFINITY);
    T dt = T(a.dt);
    if (a.dt_from_slots) dt = Ar<T, false>::mul(T(a.cfl), T(__longlong_as_double((long long)a.slots[5 * a.first + 3])));
    __syncthreads();

    for (int64_t k = 0; k < a.steps; ++k) {
        const int p = (int)(k & 1);
        const Coef<T> c = make_coef<T>(dx, dy, dt, g);
        bool ok = true;
        // phase B: every face once -- the thread of corner (x, j), x = 0 .. nx,
        // j = 0 .. R, takes the x-face right of cell (x, j) (band rows) and
        // the y-face above it (interior columns); the cell quantities of its
        // cell, the right and the upper neighbour are computed in registers
        // (rows 0 and R+1 -- the halo rows -- live in the halo buffers of parity p)
        T fdep = T(INFINITY);
        auto corner = [&](int j, int x) {
            const bool xf = j >= 1, yf = x >= 1;
            if (!xf && !yf) return;
            const Q sc = j == 0 ? sm[L.HB(p, 0, x - 1)] : sm[L.S(j, x)];
            if constexpr (DM == DIV_GUARD) {
                // exact mode: the guarded shared-reciprocal division; a corner
                // that saw a non-benign operand redoes its faces with DIV_FIXUP
                bool okg = true;
                const CellQ<T> C = rcq<T, DIV_GUARD>(sc, c, okg);
                FaceF<T> fx, fy;
                if (xf) fx = x_face<T, DIV_GUARD>(C, rcq<T, DIV_GUARD>(sm[L.S(j, x + 1)], c, okg), c, okg);
                const Q su = yf ? (j == R ? sm[L.HB(p, 1, x - 1)] : sm[L.S(j + 1, x)]) : sc;
                if (yf) fy = y_face<T, DIV_GUARD>(C, rcq<T, DIV_GUARD>(su, c, okg), c, okg);
                if (!okg) {
                    bool okf = true;
                    const CellQ<T> C2 = rcq<T, DIV_FIXUP>(sc, c, okf);
                    if (xf) fx = x_face<T, DIV_FIXUP>(C2, rcq<T, DIV_FIXUP>(sm[L.S(j, x + 1)], c, okf), c, okf);
                    if (yf) fy = y_face<T, DIV_FIXUP>(C2, rcq<T, DIV_FIXUP>(su, c, okf), c, okf);
                }
                if (xf) { sm[L.FX(j - 1, x)] = Q{fx.fh, fx.fu, fx.fv, T(0)}; fdep = fmin(fdep, fx.hd); }
                if (yf) { sm[L.FY(j, x - 1)] = Q{fy.fh, fy.fu, fy.fv, T(0)}; fdep = fmin(fdep, fy.hd); }
            } else {
                const CellQ<T> C = rcq<T, DM>(sc, c, ok);
                if (xf) {
                    const FaceF<T> f = x_face<T, DM>(C, rcq<T, DM>(sm[L.S(j, x + 1)], c, ok), c, ok);
                    sm[L.FX(j - 1, x)] = Q{f.fh, f.fu, f.fv, T(0)};
                    fdep = fmin(fdep, f.hd);
                }
                if (yf) {
                    const Q su = j == R ? sm[L.HB(p, 1, x - 1)] : sm[L.S(j + 1, x)];
                    const FaceF<T> f = y_face<T, DM>(C, rcq<T, DM>(su, c, ok), c, ok);
                    sm[L.FY(j, x - 1)] = Q{f.fh, f.fu, f.fv, T(0)};
                    fdep = fmin(fdep, f.hd);
                }
            }
        };
        {
            // two corners per iteration (independent chains: ILP)
            RegionIter i1(tid, 2 * nt, nx + 1), i2(tid + nt, 2 * nt, nx + 1);
            for (; i1.j < R + 1; i1.next(), i2.next()) {
                corner(i1.j, i1.x);
                if (i2.j < R + 1) corner(i2.j, i2.x);
            }
        }
        __syncthreads();
        // phase C: update in place + column halos + row pushes + reductions
        const int q = 1 - p;                     // halo parity the next step reads
        double mass = 0.0;
        B mu = 0, mv = 0;
        T hmin = T(INFINITY), bmin = T(INFINITY);
        const bool want_red = a.slots != nullptr || a.dt_from_slots;
        auto cell = [&](int j, int x) {
            const Q o = sm[L.S(j, x)];
            const Q fl = sm[L.FX(j - 1, x - 1)], fr = sm[L.FX(j - 1, x)];
            const Q fd = sm[L.FY(j - 1, x - 1)], fu = sm[L.FY(j, x - 1)];
            T h, u, v;
            update_cell<T, DM>(o.a, o.b, o.c, FaceF<T>{fl.a, fl.b, fl.c, T(1)}, FaceF<T>{fr.a, fr.b, fr.c, T(1)},
                               FaceF<T>{fd.a, fd.b, fd.c, T(1)}, FaceF<T>{fu.a, fu.b, fu.c, T(1)}, c, h, u, v);
            const Q nw{h, u, v, T(0)};
            sm[L.S(j, x)] = nw;
            // column halos (apply_boundary columns)
            if (x == 1) {
                if (a.bc.s[SIDE_L] == BC_REFL) sm[L.S(j, 0)] = Q{h, -u, v, T(0)};
                if (a.bc.s[SIDE_R] == BC_PER) sm[L.S(j, nx + 1)] = nw;
            }
            if (x == nx) {
                if (a.bc.s[SIDE_R] == BC_REFL) sm[L.S(j, nx + 1)] = Q{h, -u, v, T(0)};
                if (a.bc.s[SIDE_L] == BC_PER) sm[L.S(j, 0)] = nw;
            }
            // the band's first / last row: the neighbour's halo row for the next step
            // (reflective domain edge: this CTA's own halo row, the mirror image)
            if (j == 1) {
                if (below >= 0) st_dsmem_q<T>(dsmem_addr((uint32_t)__cvta_generic_to_shared(&sm[L.HB(q, 1, x - 1)]), below), nw);
                else sm[L.HB(q, 0, x - 1)] = Q{h, u, -v, T(0)};
            }
            if (j == R) {
                if (above >= 0) st_dsmem_q<T>(dsmem_addr((uint32_t)__cvta_generic_to_shared(&sm[L.HB(q, 0, x - 1)]), above), nw);
                else sm[L.HB(q, 1, x - 1)] = Q{h, u, -v, T(0)};
            }
            // reductions of the new state (RowRed semantics of the step kernels:
            // maxima as the bit patterns of |value| -- NaN / Inf sort on top)
            if (!want_red) return;
            mass += (double)h;
            mu = max(mu, RowRed<T, false, 1>::absbits(u));
            mv = max(mv, RowRed<T, false, 1>::absbits(v));
            hmin = fmin(hmin, h);
            if (a.want_cfl) bmin = fmin(bmin, cfl_bound(h, u, v, g, dmin));
        };
        {
            RegionIter i1(tid, 2 * nt, nx), i2(tid + nt, 2 * nt, nx);
            for (; i1.j < R; i1.next(), i2.next()) {
                cell(i1.j + 1, i1.x + 1);
                if (i2.j < R) cell(i2.j + 1, i2.x + 1);
            }
        }
        // block reduction -> the CTA's CFL slot and the step's slot row
        // (skipped when nobody reads them: no slots, fixed dt)
        if (!want_red) {
            cluster_barrier();
            continue;
        }
        const double wm = warp_sum(mass);
        const B wu = RowRed<T, false, 1>::warp_max_bits(mu), wv = RowRed<T, false, 1>::warp_max_bits(mv);
        const T wh = warp_min(hmin), wb = warp_min(bmin), wf = warp_min(fdep);
        if (lane == 0) {
            uint32_t e = 0;
            if (!(wh > T(0)) && !isnan(wh)) e |= FKC_RES_ERR_DEPTH;
            if (!(wf > T(0)) && !isnan(wf)) e |= FKC_RES_ERR_FACE;
            s_mass[warp] = wm;
            s_mx[warp][0] = dbits((double)RowRed<T, false, 1>::frombits(wu));
            s_mx[warp][1] = dbits((double)RowRed<T, false, 1>::frombits(wv));
            s_b[warp] = wb;
            s_err[warp] = e;
        }
        __syncthreads();
        if (warp == 0) {
            const bool has = lane < nt / 32;
            double m = warp_sum(has ? s_mass[lane] : 0.0);
            unsigned long long xu = has ? s_mx[lane][0] : 0ull, xv = has ? s_mx[lane][1] : 0ull;
            for (int o = 16; o > 0; o >>= 1) {
                xu = max(xu, (unsigned long long)__shfl_xor_sync(0xffffffffu, xu, o));
                xv = max(xv, (unsigned long long)__shfl_xor_sync(0xffffffffu, xv, o));
            }
            const T bb = warp_min(has ? s_b[lane] : T(INFINITY));
            uint32_t ee = __reduce_or_sync(0xffffffffu, has ? s_err[lane] : 0u);
            if (!isfinite(m) || xu >= 0x7ff0000000000000ull || xv >= 0x7ff0000000000000ull) ee |= FKC_RES_ERR_NONFINITE;
            if (lane == 0) s_cfl[p] = bb;
            if (lane == 0 && a.slots) {
                unsigned long long* row = a.slots + 5 * (a.first + k + 1);
                atomicAdd((double*)row, m);
                atomicMax(row + 1, xu);
                atomicMax(row + 2, xv);
                if (a.want_cfl) atomicMin(row + 3, dbits((double)bb));
                if (ee) atomicOr((unsigned int*)(row + 4), ee);
            }
        }
        cluster_barrier();   // every CTA's pushes, column halos and CFL slot are visible
        if (a.dt_from_slots) {
            T bm = T(INFINITY);
            for (int r = 0; r < nb; ++r)
                bm = fmin(bm, ld_dsmem<T>(dsmem_addr((uint32_t)__cvta_generic_to_shared(&s_cfl[p]), r)));
            dt = Ar<T, false>::mul(T(a.cfl), bm);
        }
    }
    // final state: band rows incl. column halos (the host fills row halos / corners)
    T* out[3] = {(T*)a.out[0], (T*)a.out[1], (T*)a.out[2]};
    for (RegionIter it(tid, nt, L.W); it.j < R; it.next()) {
        const int64_t go = (int64_t)(r0 + it.j) * a.pitch + it.x;
        const Q o = sm[L.S(it.j + 1, it.x)];
        out[0][go] = o.a; out[1][go] = o.b; out[2][go] = o.c;
    }
    cluster_barrier();   // no CTA exits while a neighbour may still read its CFL slot
}

}  // namespace fkc
