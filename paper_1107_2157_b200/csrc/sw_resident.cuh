// sw_resident.cuh -- the whole time loop of a SMALL grid in one launch:
// a thread-block cluster (up to 16 CTAs, one per SM) keeps the state in
// shared memory and iterates the steps on chip.
//
// Why: below ~512^2 a step is a few microseconds of work, and a launch per
// step -- even replayed from a CUDA graph -- costs about as much as the work
// (B200: 128^2 runs 2.5 us / step in a graph).  Here a step costs its
// arithmetic plus one cluster barrier.
//
// Work split.  CTA b of the cluster owns a band of R_b consecutive rows
// (full width).  Its shared memory holds the band plus one halo row above
// and below, TWICE (state k is read from buffer k&1, state k+1 written to
// the other), as three field planes laid out exactly like one TMA stage of
// the per-step kernel (sw_tma.cuh): plane column c = full column x + LEAD,
// so strip j's lane l reads its CPL cells of a row with one 16-byte vector
// load at column OWN j + CPL l.  The warps of the CTA are (strip, row
// group) pairs; each sweeps its rows with the SAME row engines as the per-
// step TMA kernel (sw_pair.cuh: PairEngine for f32 fast, ExactPairEngine2
// for f32 bit-exact, ScalarEngine for f64) -- cell quantities once per
// cell, x-faces through shuffles with ghost lanes, y-faces carried in
// registers -- reading rows from the resident buffer instead of a TMA ring.
// Each updated row goes to the other buffer; the band's first / last row
// is also pushed into the neighbouring CTA's halo row of that buffer
// through distributed shared memory (DSMEM), and the boundary images
// (column halos; row halos at the domain edges) are written alongside.
// Buffers are never read and written in the same step, so one cluster
// barrier (release / acquire) per step is the only synchronisation.  With a
// CFL-chosen dt every CTA then reads the cluster's minimum bound from the
// CTAs' slots (DSMEM, parity-buffered) -- no host, no global round trip; the
// per-step diagnostics rows are committed to global memory after the
// barrier (off the critical path).
//
// Arithmetic: the per-step kernels' row engines, so exact mode is
// bit-identical to the oracle.  The final state is written to the buffer
// fkc_sw_advance_n's double-buffering contract names; the host then fills
// its row halos / corners with the boundary kernel (== apply_boundary).
#pragma once
#include "sw_tma.cuh"

namespace fkc {

// warps per CTA: the f32 exact engine fits 168 registers (12 warps: 4 x 3
// per SM sub-partition); the fast pair engine and the f64 engines do not
// without spills, so they run 8 warps (255 registers)
constexpr int RES_MAX_WARPS = 12;
#ifndef FKC_RES_FAST_WARPS
#define FKC_RES_FAST_WARPS 8
#endif
template <class T, bool FAST> constexpr int res_warps() {
    return sizeof(T) == 8 ? 8 : (FAST ? FKC_RES_FAST_WARPS : 12);
}
constexpr int RES_MAX_CLUSTER = 16;
#ifndef FKC_RES_FAST_UNROLL
#define FKC_RES_FAST_UNROLL 2            // fast mode: rows of the sweep unrolled (register window renamed)
#endif
// rows per warp's sweep (row group) targeted by the host plan, capped by
// the warps per CTA; B200 (profiles/r02/resident_variants.txt): fast 1
// (128^2 1.93 vs 2.10 us / step at 4), exact 2 (3.15 vs 3.61)
#ifndef FKC_RES_GROUP_ROWS_FAST
#define FKC_RES_GROUP_ROWS_FAST 1
#endif
#ifndef FKC_RES_GROUP_ROWS_EXACT
#define FKC_RES_GROUP_ROWS_EXACT 2
#endif

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
__device__ __forceinline__ T ld_dsmem(uint32_t a) {
    T v;
    if constexpr (sizeof(T) == 4) asm volatile("ld.shared::cluster.f32 %0, [%1];" : "=f"(v) : "r"(a) : "memory");
    else asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
    return v;
}
// one lane's 16-byte row vector into (possibly another CTA's) shared memory
template <class T, int CPL>
__device__ __forceinline__ void st_cluster_vec(uint32_t a, const T (&v)[CPL], T sgn = T(1)) {
    if constexpr (sizeof(T) == 4)
        asm volatile("st.shared::cluster.v4.f32 [%0], {%1, %2, %3, %4};" ::"r"(a), "f"(sgn * v[0]),
                     "f"(sgn * v[1]), "f"(sgn * v[2]), "f"(sgn * v[3]) : "memory");
    else
        asm volatile("st.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(a), "d"(sgn * v[0]), "d"(sgn * v[1])
                     : "memory");
}
__device__ __forceinline__ void cluster_barrier() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// shared-memory geometry of one CTA (every CTA uses the same, so a local
// address is valid in DSMEM too): planes [buffer][field][row 0..R+1][column]
template <class T> struct ResGeo {
    static constexpr int CPL = tma::Geo<T>::CPL, OWN = tma::Geo<T>::OWN, LEAD = tma::Geo<T>::LEAD;
    int ns, rowe, R;                 // strips, elements per plane row, rows of the largest band
    __host__ __device__ ResGeo(int nx, int R_) : R(R_) {
        ns = (nx + OWN - 1) / OWN;
        rowe = OWN * (ns - 1) + 32 * CPL;
    }
    __host__ __device__ int plane() const { return (R + 2) * rowe; }
    __host__ __device__ size_t bytes() const { return (size_t)6 * plane() * sizeof(T); }
    // element offset of (buffer p, field f, band row j, full column x)
    __host__ __device__ int at(int p, int f, int j, int x) const { return (p * 3 + f) * plane() + j * rowe + x + LEAD; }
};

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
    int groups;                  // row groups per band (warps = strips x groups)
};

template <class T, bool FAST, int RED>
__global__ void __launch_bounds__(res_warps<T, FAST>() * 32, 1) sw_resident(const __grid_constant__ ResArgs a) {
    using G = tma::Geo<T>;
    constexpr int CPL = G::CPL;
    constexpr int DM = FAST ? DIV_FAST : DIV_GUARD;
    constexpr bool EXACT2 = !FAST && sizeof(T) == 4;
    using Engine = typename std::conditional<
        FAST && sizeof(T) == 4, PairEngine,
        typename std::conditional<EXACT2, ExactPairEngine2, ScalarEngine<T, CPL>>::type>::type;
    using RR = RowRed<T, FAST, RED>;
    using B = typename RR::B;
    constexpr int RES_UNR = FAST ? FKC_RES_FAST_UNROLL : 1;
    extern __shared__ __align__(128) uint8_t res_smem[];
    T* sm = (T*)res_smem;
    __shared__ T s_cfl[2];                                  // this CTA's CFL bound of the last two states
    __shared__ double s_mass[RES_MAX_WARPS];
    __shared__ B s_mu[RES_MAX_WARPS], s_mv[RES_MAX_WARPS];
    __shared__ T s_dmax[RES_MAX_WARPS], s_h[RES_MAX_WARPS], s_f[RES_MAX_WARPS];
    __shared__ double s_tot_mass;
    __shared__ unsigned long long s_tot_u, s_tot_v, s_tot_b;
    __shared__ uint32_t s_tot_err;

    const int nb = (int)gridDim.x;                          // the grid is exactly one cluster
    const int b = (int)cluster_rank();
    const int nx = a.nx, ny = a.ny;
    const int base = ny / nb, extra = ny % nb;
    const int R = base + (b < extra ? 1 : 0);               // rows of this band
    const int r0 = 1 + b * base + min(b, extra);            // its first interior row
    auto band_rows = [&](int bb) { return base + (bb < extra ? 1 : 0); };
    const ResGeo<T> L(nx, base + (extra ? 1 : 0));
    const int tid = threadIdx.x, nt = blockDim.x;
    const int lane = tid & 31, warp = warp_index();   // provably warp-uniform (sw_tma.cuh)
    const T dx = T(a.dx), dy = T(a.dy), g = T(a.g), dmin = dx < dy ? dx : dy;
    const int below = b > 0 ? b - 1 : (a.bc.s[SIDE_D] == BC_PER ? nb - 1 : -1);
    const int above = b < nb - 1 ? b + 1 : (a.bc.s[SIDE_U] == BC_PER ? 0 : -1);
    const bool want_red = a.slots != nullptr;

    // both buffers: a lake at rest everywhere (cells outside the grid stay
    // benign for the branch-free sweeps), then the band's rows 0..R+1,
    // columns 0..nx+1 of the input into buffer 0
    for (int i = tid; i < 2 * L.plane(); i += nt) {
        const int p = i / L.plane(), r = i - p * L.plane();
        sm[(p * 3 + 0) * L.plane() + r] = T(1);
        sm[(p * 3 + 1) * L.plane() + r] = T(0);
        sm[(p * 3 + 2) * L.plane() + r] = T(0);
    }
    __syncthreads();
    {
        const T* in[3] = {(const T*)a.in[0], (const T*)a.in[1], (const T*)a.in[2]};
        const int w = nx + 2;
        for (int i = tid; i < (R + 2) * w; i += nt) {
            const int j = i / w, x = i - j * w;
            const int64_t go = (int64_t)(r0 - 1 + j) * a.pitch + x;
#pragma unroll
            for (int f = 0; f < 3; ++f) sm[L.at(0, f, j, x)] = in[f][go];
        }
    }
    if (tid < 2) s_cfl[tid] = T(INFINITY);
    T dt = T(a.dt);
    if (a.dt_from_slots) dt = Ar<T, false>::mul(T(a.cfl), T(__longlong_as_double((long long)a.slots[5 * a.first + 3])));
    __syncthreads();
    cluster_barrier();                      // every CTA's buffers are initialised before any DSMEM push

    // this warp's strip and row group
    const int ns = L.ns;
    const int strip = warp % ns, grp = warp / ns;
    const bool active = grp < a.groups;
    const int gbase = R / a.groups, gext = R % a.groups;
    const int ga = 1 + grp * gbase + min(grp, gext);        // first band row of the group
    const int nrows = active ? gbase + (grp < gext ? 1 : 0) : 0;
    const int xs = 1 + strip * G::OWN - CPL;                // full column of the lane-0 cell
    const int X = xs + CPL * lane;                          // this lane's first cell
    const bool owner = (lane >= 1) && (lane <= 30) && (X <= nx);
    const uint32_t smem0 = smem_u32(res_smem);

    for (int64_t k = 0; k < a.steps; ++k) {
        const int p = (int)(k & 1), q = p ^ 1;
        const Coef<T> c = make_coef<T>(dx, dy, dt, g);
        RR rr;
        rr.init();
        T fdep = T(INFINITY);
        if (active && nrows > 0) {
            Engine eng;
            eng.init(c);
            // store of the updated band row y (owner lanes): the other buffer,
            // the column images, the neighbour's halo row / the domain-edge image
            auto store_row = [&](int y, T (&oh)[CPL], T (&ou)[CPL], T (&ov)[CPL]) {
                T* dst[3] = {sm + L.at(q, 0, y, X), sm + L.at(q, 1, y, X), sm + L.at(q, 2, y, X)};
                stg_vec<T, CPL>(dst[0], oh);
                stg_vec<T, CPL>(dst[1], ou);
                stg_vec<T, CPL>(dst[2], ov);
                // column halos (apply_boundary columns)
                if (X == 1) {
                    if (a.bc.s[SIDE_L] == BC_REFL) {
                        sm[L.at(q, 0, y, 0)] = oh[0]; sm[L.at(q, 1, y, 0)] = -ou[0]; sm[L.at(q, 2, y, 0)] = ov[0];
                    } else if (a.bc.s[SIDE_R] == BC_PER) {
                        sm[L.at(q, 0, y, nx + 1)] = oh[0]; sm[L.at(q, 1, y, nx + 1)] = ou[0]; sm[L.at(q, 2, y, nx + 1)] = ov[0];
                    }
                }
                if (X + CPL - 1 == nx) {
                    if (a.bc.s[SIDE_R] == BC_REFL) {
                        sm[L.at(q, 0, y, nx + 1)] = oh[CPL - 1]; sm[L.at(q, 1, y, nx + 1)] = -ou[CPL - 1];
                        sm[L.at(q, 2, y, nx + 1)] = ov[CPL - 1];
                    } else if (a.bc.s[SIDE_L] == BC_PER) {
                        sm[L.at(q, 0, y, 0)] = oh[CPL - 1]; sm[L.at(q, 1, y, 0)] = ou[CPL - 1]; sm[L.at(q, 2, y, 0)] = ov[CPL - 1];
                    }
                }
                // row halos: the band's first / last row is the neighbour's halo
                // row (DSMEM push); at a reflective domain edge the image goes
                // into this CTA's own halo row
                if (y == 1) {
                    if (below >= 0) {
                        const int jt = band_rows(below) + 1;
                        st_cluster_vec<T, CPL>(dsmem_addr(smem0 + (uint32_t)(L.at(q, 0, jt, X) * sizeof(T)), below), oh);
                        st_cluster_vec<T, CPL>(dsmem_addr(smem0 + (uint32_t)(L.at(q, 1, jt, X) * sizeof(T)), below), ou);
                        st_cluster_vec<T, CPL>(dsmem_addr(smem0 + (uint32_t)(L.at(q, 2, jt, X) * sizeof(T)), below), ov);
                    } else {
                        stg_vec<T, CPL>(sm + L.at(q, 0, 0, X), oh);
                        stg_vec<T, CPL>(sm + L.at(q, 1, 0, X), ou);
                        stg_vec<T, CPL>(sm + L.at(q, 2, 0, X), ov, T(-1));
                    }
                }
                if (y == R) {
                    if (above >= 0) {
                        st_cluster_vec<T, CPL>(dsmem_addr(smem0 + (uint32_t)(L.at(q, 0, 0, X) * sizeof(T)), above), oh);
                        st_cluster_vec<T, CPL>(dsmem_addr(smem0 + (uint32_t)(L.at(q, 1, 0, X) * sizeof(T)), above), ou);
                        st_cluster_vec<T, CPL>(dsmem_addr(smem0 + (uint32_t)(L.at(q, 2, 0, X) * sizeof(T)), above), ov);
                    } else {
                        stg_vec<T, CPL>(sm + L.at(q, 0, R + 1, X), oh);
                        stg_vec<T, CPL>(sm + L.at(q, 1, R + 1, X), ou);
                        stg_vec<T, CPL>(sm + L.at(q, 2, R + 1, X), ov, T(-1));
                    }
                }
                if constexpr (RED > 0) rr.template add_row<CPL>(oh, ou, ov, g);
            };
            // the sweep of band rows ga-1 .. ga+nrows (loaded row n = band row ga-1+n)
            const int nload = nrows + 2;
#pragma unroll RES_UNR
            for (int n = 0; n < nload; ++n) {
                const int j = ga - 1 + n;
                const uint32_t sr = smem0 + (uint32_t)(L.at(p, 0, j, X) * sizeof(T));
                const uint32_t fb = (uint32_t)(L.plane() * sizeof(T));
                auto load_row = [&](VecF<T>& hv, VecF<T>& uv, VecF<T>& vv) {
                    hv = lds_vec<T>(sr);
                    uv = lds_vec<T>(sr + fb);
                    vv = lds_vec<T>(sr + 2 * fb);
                };
                VecF<T> hv, uv, vv;
                load_row(hv, uv, vv);
                const bool have_prev = n >= 1;
                const bool want_x = (n >= 1) && (n <= nrows);
                const bool upd = n >= 2;
                const int y_upd = ga + n - 2;
                bool ok = true;
                if constexpr (EXACT2) {
                    eng.template cells_y<DIV_GUARD>(hv, uv, vv, have_prev, ok);
                    if (__any_sync(0xffffffffu, !ok)) {
                        VecF<T> h2, u2, v2;
                        asm volatile("" ::: "memory");
                        load_row(h2, u2, v2);
                        eng.template cells_y<DIV_FIXUP>(h2, u2, v2, have_prev, ok);
                    }
                    if (upd) {
                        T oh[CPL], ou[CPL], ov[CPL];
                        eng.template update<DM>(c, oh, ou, ov);
                        if (owner) store_row(y_upd, oh, ou, ov);
                    }
                    bool okx = true;
                    eng.template xfaces<DIV_GUARD>(want_x, okx);
                    if (__any_sync(0xffffffffu, !okx)) eng.template xfaces<DIV_FIXUP>(want_x, okx);
                } else {
                    if constexpr (FAST) {
                        eng.template row<DIV_FAST>(hv, uv, vv, true, true, c, ok);
                    } else {
                        eng.template row<DIV_GUARD>(hv, uv, vv, have_prev, want_x, c, ok);
                        if (__any_sync(0xffffffffu, !ok)) {
                            VecF<T> h2, u2, v2;
                            asm volatile("" ::: "memory");
                            load_row(h2, u2, v2);
                            eng.template row<DIV_FIXUP>(h2, u2, v2, have_prev, want_x, c, ok);
                        }
                    }
                    if (upd) {
                        T oh[CPL], ou[CPL], ov[CPL];
                        eng.template update<DM>(c, oh, ou, ov);
                        if (owner) store_row(y_upd, oh, ou, ov);
                    }
                }
                if constexpr (RED > 0) {
                    // face depths of the faces owned cells use (NonPositiveDepth)
                    const bool xrow = (n >= 1) && (n <= nrows);
                    const bool yrow = n >= 1;
                    eng.track(fdep, owner && xrow, lane == 0 && xrow, owner && yrow);
                }
                eng.shift();
            }
        }
        if constexpr (RED > 0) {
            // warp partials -> CTA totals (warp 0) -> the CTA's CFL slot; the
            // diagnostics row goes to global memory after the barrier
            const double wm = warp_sum(rr.mass);
            const B wu = RR::warp_max_bits(rr.mu), wv = RR::warp_max_bits(rr.mv);
            const T wh = warp_min(rr.hmin), wd = warp_max(rr.dmax), wf = warp_min(fdep);
            if (lane == 0) {
                s_mass[warp] = wm; s_mu[warp] = wu; s_mv[warp] = wv;
                s_h[warp] = wh; s_dmax[warp] = wd; s_f[warp] = wf;
            }
            __syncthreads();
            if (warp == 0) {
                const bool has = lane < nt / 32;
                const double m = warp_sum(has ? s_mass[lane] : 0.0);
                const B bu = RR::warp_max_bits(has ? s_mu[lane] : B(0)), bv = RR::warp_max_bits(has ? s_mv[lane] : B(0));
                const T hm = warp_min(has ? s_h[lane] : T(INFINITY));
                const T dm = warp_max(has ? s_dmax[lane] : T(0));
                const T fm = warp_min(has ? s_f[lane] : T(INFINITY));
                if (lane == 0) {
                    uint32_t e = 0;
                    if (!(hm > T(0)) && !isnan(hm)) e |= 1u;
                    if (!isfinite(m) || bu >= RR::absbits(T(INFINITY)) || bv >= RR::absbits(T(INFINITY))) e |= 2u;
                    if (!(fm > T(0)) && !isnan(fm)) e |= 8u;
                    const T bound = (RED >= 2 && dm > T(0)) ? Ar<T, false>::div(dmin, dm) : T(INFINITY);
                    s_cfl[p] = bound;
                    s_tot_mass = m;
                    s_tot_u = dbits((double)RR::frombits(bu));
                    s_tot_v = dbits((double)RR::frombits(bv));
                    s_tot_b = dbits((double)bound);
                    s_tot_err = e;
                }
            }
        }
        cluster_barrier();   // the other buffer (pushes, images) and the CFL slots are complete
        if constexpr (RED > 0) {
            if (tid == 0 && want_red) {
                unsigned long long* row = a.slots + 5 * (a.first + k + 1);
                atomicAdd((double*)row, s_tot_mass);
                atomicMax(row + 1, s_tot_u);
                atomicMax(row + 2, s_tot_v);
                if (RED >= 2) atomicMin(row + 3, s_tot_b);
                if (s_tot_err) atomicOr((unsigned int*)(row + 4), s_tot_err);
            }
            if (a.dt_from_slots) {
                // lane r of every warp reads CTA r's bound (one remote load
                // latency), the warp takes the minimum
                const T br = lane < nb ? ld_dsmem<T>(dsmem_addr(smem_u32(&s_cfl[p]), lane)) : T(INFINITY);
                dt = Ar<T, false>::mul(T(a.cfl), warp_min(br));
            }
        }
    }
    // final state: band rows incl. column halos (the host fills row halos / corners)
    {
        const int pf = (int)(a.steps & 1);
        T* out[3] = {(T*)a.out[0], (T*)a.out[1], (T*)a.out[2]};
        const int w = nx + 2;
        for (int i = tid; i < R * w; i += nt) {
            const int j = i / w, x = i - j * w;
            const int64_t go = (int64_t)(r0 + j) * a.pitch + x;
#pragma unroll
            for (int f = 0; f < 3; ++f) out[f][go] = sm[L.at(pf, f, j + 1, x)];
        }
    }
    cluster_barrier();   // no CTA exits while a neighbour may still read its CFL slot
}

}  // namespace fkc
