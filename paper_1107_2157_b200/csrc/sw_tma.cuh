// sw_tma.cuh -- the product kernel: per-warp TMA y-sweep of the fused
// two-step Lax-Wendroff step (f32 and f64; fast and bit-exact modes; fused
// boundary halos, reductions and multi-GPU halo exchange).
//
// Geometry.  A warp owns a strip of OWN = 30*CPL columns and `seg` rows.
// It loads LOAD = 32*CPL columns (the strip plus CPL columns on each side):
// lane l holds CPL consecutive cells of every row; lanes 0 and 31 are
// "ghost" lanes whose cells lie outside the strip -- they exist so that
// every x-face an owned lane (1..30) needs is produced in SIMD by a
// neighbouring lane (no divergent edge work, no separate halo loads).
//
// Pipeline.  Lane 0 streams the strip's rows of H, U, V through a private
// S-stage shared-memory ring (R rows per stage, one cp.async.bulk.tensor box
// per field, completion on an mbarrier with expect_tx); the warp never waits
// for another warp.  Each row is read once from shared memory (one vector
// LDS per field), its cell quantities (fxu, cross) are computed once, the
// y-face below it is carried in registers from the previous row, the x-face
// right of lane's last cell uses lane+1's first cell (shfl.down) and the face
// left of its first cell is lane-1's last face (shfl.up).  The row above is
// then updated and stored with vector stores; the output halo (boundary
// conditions) and optional reductions are emitted in the same pass.
//
// The per-row arithmetic lives in the row engines of sw_pair.cuh
// (PairEngine: f32 fast on the packed FP32 pipe; ExactPairEngine: f32
// bit-exact; ScalarEngine: f64).  In fast mode odd segments sweep the mirror
// image top-down (L2 reuse of the rows shared by neighbouring segments).
//
// Schedule (host side, fkc_sw.cu): a 2-D grid of CTAs = bands of 4 strips x
// row segments; the last wave's segments are half length (SegMap::tail),
// successive launches on a stream lay the segments out bottom-up and
// top-down in turn (SegMap::rev: a step starts on the rows its predecessor
// wrote last), and launches are programmatic (pdl_wait before the first read
// of the previous step's output).
#pragma once
#include "sw_pair.cuh"

namespace fkc {
namespace tma {
#ifndef FKC_TMA_R
#define FKC_TMA_R 4
#endif
#ifndef FKC_TMA_S
#define FKC_TMA_S 3
#endif
#ifndef FKC_TMA_CTAS_FAST
#define FKC_TMA_CTAS_FAST 3   // fast kernel: <= 168 registers -> 12 warps per SM
#endif
#ifndef FKC_TMA_CTAS_FAST_RED
#define FKC_TMA_CTAS_FAST_RED 3  // fast kernel with fused reductions
#endif
#ifndef FKC_TMA_CTAS_F64
#define FKC_TMA_CTAS_F64 2    // f64 kernels (~190-210 registers)
#endif
#ifndef FKC_EXACT_WARPS
#define FKC_EXACT_WARPS 12    // exact kernel: resident warps per SM (12: <= 168 registers; even)
#endif
constexpr int R = FKC_TMA_R;             // rows per stage
constexpr int S = FKC_TMA_S;             // ring stages per warp
// T = float (4 cells per lane) or double (2 cells per lane): one 16-byte
// vector per lane and row either way.
#ifndef FKC_F64_CPL
#define FKC_F64_CPL 2     // f64 cells per lane: 2 (one 16-B vector) or 1 (8 B lanes, half the register
                          // window: 154-168 registers, 3 CTAs per SM -- correct, but measured 14 % slower
                          // in fast mode, 9 % in exact: per-row overheads over half the cells)
#endif
template <class T> struct Geo {
    static constexpr int CPL = sizeof(T) == 8 ? FKC_F64_CPL : 4;   // cells per lane
    static constexpr int VEC = CPL * (int)sizeof(T);      // bytes per lane and row
    static constexpr int LEAD = 16 / (int)sizeof(T) - 1;  // tensor column = full column + LEAD (fkc_sw.cu get_map)
    static constexpr int LOAD = 32 * CPL;                 // columns loaded per strip
    static constexpr int OWN = 30 * CPL;                  // columns owned per strip
    // TMA box starts must be 16-B aligned.  With 16-B lanes every strip's
    // first loaded column is; with 8-B lanes (f64, CPL 1) every other strip
    // starts one column late, so the box takes 2 extra columns and the lanes
    // read from column `shift` (0 or 1) of it.
    static constexpr int BOXW = VEC == 16 ? LOAD : LOAD + 2;          // columns per TMA box
    static constexpr int ROWB = BOXW * (int)sizeof(T);                // bytes per staged row
    static constexpr int FIELD_BYTES = (R * ROWB + 127) / 128 * 128;  // 128-B aligned TMA destinations
    static constexpr int STAGE_BYTES = 3 * FIELD_BYTES;
    static constexpr int TX_BYTES = 3 * R * ROWB;                     // bytes a stage's 3 boxes deliver
    static constexpr int WARP_RING = S * STAGE_BYTES;
    // resident warps per SM (the FKC_TMA_CTAS_* macros count CTAs of 4 warps):
    // f32 12 (<= 168 registers), f64 8
    template <bool FAST, int RED = 0> static constexpr int warps_per_sm() {
        return sizeof(T) == 8 ? 4 * FKC_TMA_CTAS_F64
                              : (FAST ? 4 * (RED ? FKC_TMA_CTAS_FAST_RED : FKC_TMA_CTAS_FAST) : FKC_EXACT_WARPS);
    }
    static_assert(FIELD_BYTES % 128 == 0, "TMA destinations must stay 128-B aligned");
};
// A CTA of NW independent warps (strips): 1, 2 or 4 (host picks per size and
// mode, fkc_sw.cu).  Smaller CTAs = finer scheduling granularity for the
// hardware's CTA scheduler (shorter tail), larger = fewer CTA launches.
template <class T, int NW> struct Blk {
    static constexpr int THREADS = NW * 32;
    static constexpr int SMEM_BYTES = NW * Geo<T>::WARP_RING + NW * S * 8 + 128;
    template <bool FAST, int RED = 0> static constexpr int ctas_per_sm() {
        return Geo<T>::template warps_per_sm<FAST, RED>() / NW;
    }
};
#ifndef FKC_EXACT_ALWAYS_FIXUP
#define FKC_EXACT_ALWAYS_FIXUP 0
#endif
#ifndef FKC_TMA_PAIR
#define FKC_TMA_PAIR 1        // f32 fast mode on the packed FP32 pipe (FFMA2 / FADD2 / FMUL2)
#endif
#ifndef FKC_TMA_EXACT_PAIR
#define FKC_TMA_EXACT_PAIR 2  // f32 exact mode: 2 = every op on the packed pipe, row-level guards
                              // (ExactPairEngine2); 1 = packed multiplies only (ExactPairEngine); 0 = scalar
#endif
#ifndef FKC_FAST_UNROLL
#define FKC_FAST_UNROLL 2     // rows of a stage unrolled in fast mode (even: the register window renames)
#endif
#ifndef FKC_FIX_PERSIST
#define FKC_FIX_PERSIST 0     // exact mode: rows that stay on the fixup variant after a guard failure
#endif
#ifndef FKC_EXACT_ROWSYNC
#define FKC_EXACT_ROWSYNC 0
#endif
#ifndef FKC_EXACT_UNROLL
#define FKC_EXACT_UNROLL 1    // exact f32 rows unrolled (1: the loop body stays in the I-cache)
#endif
#ifndef FKC_EXACT_UNROLL_F64
#define FKC_EXACT_UNROLL_F64 4    // f64 exact: unrolled rows rename the (large) register window (measured +6 %)
#endif
}  // namespace tma

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint32_t b, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(b), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(b), "r"(bytes) : "memory");
}
__device__ __forceinline__ bool mbar_try_wait(uint32_t b, uint32_t parity) {
    uint32_t ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok) : "r"(b), "r"(parity) : "memory");
    return ok != 0;
}
// Bounded wait: a lost TMA transaction (a bug, never expected) sets the
// watchdog bit and traps after ~2 s instead of hanging the GPU.
__device__ __noinline__ void watchdog_fire(uint32_t* err) {
    atomicOr(err ? err : &g_watchdog_flag, 4u);
    __threadfence_system();
    asm volatile("trap;");
}
__device__ __forceinline__ void mbar_wait(uint32_t b, uint32_t parity, uint32_t* err) {
    if (mbar_try_wait(b, parity)) return;
    const long long t0 = clock64();
    for (uint32_t spins = 1;; ++spins) {
        if (mbar_try_wait(b, parity)) return;
        if ((spins & 255u) == 0 && clock64() - t0 > 4000000000ll) watchdog_fire(err);
    }
}
#ifndef FKC_L2_HINTS
#define FKC_L2_HINTS 0
#endif
// L2 eviction hints (FKC_L2_HINTS, off): inputs streamed in evict-first,
// the new state stored evict-last, so that the rows of step n's output left
// in L2 at its end are not displaced by step n's input lines and step n+1
// (which starts with them, see SegMap::rev) hits them.  Measured on B200:
// no gain at 2048^2 .. 4096^2 and 8-10 % slower from 5792^2 up (fast mode).
__device__ __forceinline__ uint64_t l2_policy_evict_first() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ uint64_t l2_policy_evict_last() {
    uint64_t p;
    asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
    return p;
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int x, int y, uint32_t bar) {
#if FKC_L2_HINTS
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.L2::cache_hint"
        " [%0], [%1, {%2, %3}], [%4], %5;"
        :: "r"(dst), "l"((uint64_t)map), "r"(x), "r"(y), "r"(bar), "l"(l2_policy_evict_first()) : "memory");
#else
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3}], [%4];"
        :: "r"(dst), "l"((uint64_t)map), "r"(x), "r"(y), "r"(bar) : "memory");
#endif
}

// One lane's 16-byte vector of a row (4 floats or 2 doubles): shared-memory
// load, global store.
#ifndef FKC_LDS_PLAIN
#define FKC_LDS_PLAIN 1   // f32: plain 128-bit shared loads (ptxas allocates the quad where the math wants it)
#endif
template <class T>
__device__ __forceinline__ VecF<T> lds_vec(uint32_t a) {
    VecF<T> r;
    if constexpr (sizeof(T) == 4 && FKC_LDS_PLAIN) {
        float4 q;
        asm("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(q.x), "=f"(q.y), "=f"(q.z), "=f"(q.w) : "r"(a) : "memory");
        r.v[0] = q.x; r.v[1] = q.y; r.v[2] = q.z; r.v[3] = q.w;
    } else if constexpr (sizeof(T) == 4)
        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                     : "=f"(r.v[0]), "=f"(r.v[1]), "=f"(r.v[2]), "=f"(r.v[3]) : "r"(a));
    else if constexpr (tma::Geo<T>::CPL == 2)
        asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(r.v[0]), "=d"(r.v[1]) : "r"(a));
    else
        asm volatile("ld.shared.f64 %0, [%1];" : "=d"(r.v[0]) : "r"(a));
    return r;
}
template <class T, int CPL>
__device__ __forceinline__ void stg_vec(T* p, const T (&v)[CPL], T sgn = T(1)) {
    if constexpr (sizeof(T) == 4)
        *(float4*)p = make_float4(sgn * v[0], sgn * v[1], sgn * v[2], sgn * v[3]);
    else if constexpr (CPL == 2)
        *(double2*)p = make_double2(sgn * v[0], sgn * v[1]);
    else
        *p = sgn * v[0];
}
// the new state's row store (evict-last with FKC_L2_HINTS)
template <class T, int CPL>
__device__ __forceinline__ void stg_row(T* p, const T (&v)[CPL]) {
#if FKC_L2_HINTS
    static_assert(sizeof(T) == 4 || CPL == 2, "L2 hints: 16-B vectors only");
    if constexpr (sizeof(T) == 4)
        asm volatile("st.global.L2::cache_hint.v4.f32 [%0], {%1, %2, %3, %4}, %5;"
                     :: "l"(p), "f"(v[0]), "f"(v[1]), "f"(v[2]), "f"(v[3]), "l"(l2_policy_evict_last()) : "memory");
    else
        asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;"
                     :: "l"(p), "d"(v[0]), "d"(v[1]), "l"(l2_policy_evict_last()) : "memory");
#else
    stg_vec<T, CPL>(p, v);
#endif
}

// One stage = R rows x LOAD columns of H, U, V (3 boxes), completing on `bar`.
template <class T>
__device__ __forceinline__ void issue_stage(uint32_t st, uint32_t bar, const CUtensorMap* mH,
                                            const CUtensorMap* mU, const CUtensorMap* mV, int tx, int ty) {
    constexpr int FB = tma::Geo<T>::FIELD_BYTES;
    mbar_expect_tx(bar, tma::Geo<T>::TX_BYTES);
    tma_load_2d(st, mH, tx, ty, bar);
    tma_load_2d(st + FB, mU, tx, ty, bar);
    tma_load_2d(st + 2 * FB, mV, tx, ty, bar);
}

// Row segments of the CTA grid's y dimension: segments 0 .. jt-1 are `seg`
// rows, the rest `tail` rows (tail = 0: all `seg`).  Short tail segments are
// launched last, so the CTAs of the final, partial wave are short and the
// idle tail of the step shrinks ("guided" segmentation).  With `rev` the
// segments are laid out from the top row down (the mirror image), so a step
// starts where the previous one ended: its first CTAs read rows the previous
// step wrote last, which are still in L2 (the host alternates `rev` per
// launch on a stream).
// The segments tile the row window [ybase, ybase + nyw) -- the whole
// interior (ybase 1, nyw = ny) for a time step, a band of it for the
// streamed host run (fkc_sw_run_host), whose bands advance as a wavefront.
struct SegMap {
    int seg, tail, jt, rev;
    int ybase, nyw;
};
__device__ __forceinline__ void seg_rows(const SegMap& m, int j, int& y0, int& nrows) {
    const int r0 = (m.tail == 0 || j < m.jt) ? j * m.seg : m.jt * m.seg + (j - m.jt) * m.tail;
    nrows = min((m.tail == 0 || j < m.jt) ? m.seg : m.tail, m.nyw - r0);
    y0 = m.rev ? m.ybase + m.nyw - r0 - nrows : m.ybase + r0;     // rows y0 .. y0 + nrows - 1
}

template <class T, int CPL> struct Row3 {
    T h[CPL], u[CPL], v[CPL];
};

// Output halo of one new row segment of CPL cells (x = X .. X+CPL-1, row y)
// on the tile edge: reflective / periodic images (apply_boundary of the new
// state, corners included) and the neighbour tiles' halo lines (fused
// exchange).  Rare (edge lanes only), so it lives out of the sweep loop.
template <class T, int CPL>
__device__ __noinline__ void edge_stores(T* oH, T* oU, T* oV, int64_t pitch, int nx, int ny, int X, int y,
                                         const BCs& bc, const Peers& P, Row3<T, CPL> o) {
    if (y == 1 || y == ny) {
        // row images of the new row: the bottom halo row (row 0) is the image
        // of row 1 (reflective) or of row ny (periodic), the top one (row
        // ny+1) of row ny (reflective) or row 1 (periodic) -- decided per
        // image, so a one-row tile (y == 1 == ny) writes both
#pragma unroll
        for (int img = 0; img < 2; ++img) {          // 0: bottom halo row, 1: top halo row
            const int side = img == 0 ? SIDE_D : SIDE_U;
            const bool refl = bc.s[side] == BC_REFL && y == (img == 0 ? 1 : ny);
            const bool per = bc.s[side] == BC_PER && y == (img == 0 ? ny : 1);
            if (refl || per) {
                const int64_t o2 = (int64_t)(img == 0 ? 0 : ny + 1) * pitch + X;
                stg_vec<T, CPL>(oH + o2, o.h);
                stg_vec<T, CPL>(oU + o2, o.u);
                stg_vec<T, CPL>(oV + o2, o.v, refl ? T(-1) : T(1));
            }
        }
        // fused halo exchange: the new row goes straight into the neighbour
        // tile's halo row (row lines: stride 1)
#pragma unroll
        for (int side = SIDE_D; side <= SIDE_U; ++side) {
            const PeerLine& pl = P.s[side];
            if (pl.p[0] && (side == SIDE_D ? y == 1 : y == ny)) {
                stg_vec<T, CPL>((T*)pl.p[0] + X, o.h);
                stg_vec<T, CPL>((T*)pl.p[1] + X, o.u);
                stg_vec<T, CPL>((T*)pl.p[2] + X, o.v);
            }
        }
    }
    if (X == 1) {
        emit_halos<T>(oH, oU, oV, pitch, nx, ny, bc, 1, y, o.h[0], o.u[0], o.v[0], false);
        if (P.s[SIDE_L].p[0]) peer_store<T>(P.s[SIDE_L], y, o.h[0], o.u[0], o.v[0]);
    }
    if (X + CPL - 1 == nx) {
        emit_halos<T>(oH, oU, oV, pitch, nx, ny, bc, nx, y, o.h[CPL - 1], o.u[CPL - 1], o.v[CPL - 1], false);
        if (P.s[SIDE_R].p[0]) peer_store<T>(P.s[SIDE_R], y, o.h[CPL - 1], o.u[CPL - 1], o.v[CPL - 1]);
    }
}

// The warp's index in its CTA as a value the compiler can prove warp-uniform
// (a lane-0 broadcast): with a plain threadIdx.x >> 5 it cannot for CTAs of
// several warps, and every shuffle / vote after a branch on the strip (the
// early exit of strips that own nothing) then compiles to a
// WARPSYNC.COLLECTIVE fallback -- +20 % code in the sweep loop and 6-8 %
// slower mid-size steps (measured).
__device__ __forceinline__ int warp_index() {
    return __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0);
}

// Persistent time loop (sw_loop_tma below): control block and the
// neighbour ordering between its steps.
// a loop has no peer tiles (zero-initialised constant bank: no local copy)
__constant__ Peers c_no_peers;
__constant__ SyncArgs c_no_sync;
struct LoopBufs {
    void* a[3];      // buffer A (H, U, V): the input of even global steps
    void* b[3];      // buffer B
};
struct LoopCtl {
    int64_t first, steps;
    unsigned long long* slots;   // 5 words per state row, or null
    int dt_from_slots, want_cfl;
    uint32_t* flags;             // per warp: steps completed (zeroed), index seg * nstrips + strip
    uint32_t* bar;               // 32 arrival sub-counters + 1 top counter (zeroed; CFL mode)
    int nstrips;
    int per_lr, per_du;          // periodic left / right, down / up
    double dt, cfl;
};
__device__ __forceinline__ void st_release_gpu(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" :: "l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_relaxed_gpu(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// Poll with relaxed loads (an ld.acquire compiles to an L1 invalidate per
// poll -- measured: 28 % of the loop's stall samples), then one acquire
// fence once the counter is reached.
__device__ __forceinline__ void spin_until(const uint32_t* p, uint32_t target, uint32_t* err) {
    if ((int32_t)(ld_relaxed_gpu(p) - target) < 0) {
        const long long t0 = clock64();
        while ((int32_t)(ld_relaxed_gpu(p) - target) < 0) {
            __nanosleep(32);
            if (clock64() - t0 > 4000000000ll) watchdog_fire(err);
        }
    }
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
}
// Before a loop step's first load: lanes 0..3 each wait (acquire, gpu
// scope) until one direct neighbour warp -- left / right strip of the
// segment, segment below / above in the strip, the periodic wrap partners
// at the domain edges -- completed `target` steps; the four polls run in
// parallel and __syncwarp orders them before lane 0's TMA issue.
// Neighbours are re-derived here (a few integer ops once per step) rather
// than kept in registers across the sweep.
__device__ __forceinline__ void loop_nbr_wait(const LoopCtl& c, int strip, uint32_t target, int lane, uint32_t* err) {
    if (lane < 4) {
        const int ns = c.nstrips, seg = (int)blockIdx.y, nseg = (int)gridDim.y;
        int sg = seg, st = strip;
        if (lane == 0) st = strip > 0 ? strip - 1 : (c.per_lr ? ns - 1 : strip);
        else if (lane == 1) st = strip < ns - 1 ? strip + 1 : (c.per_lr ? 0 : strip);
        else if (lane == 2) sg = seg > 0 ? seg - 1 : (c.per_du ? nseg - 1 : seg);
        else sg = seg < nseg - 1 ? seg + 1 : (c.per_du ? 0 : seg);
        if (sg != seg || st != strip) spin_until(c.flags + sg * ns + st, target, err);
    }
    __syncwarp();
}

// Tensor coordinates: the maps are encoded with base = &field(1 - CPL, 0)
// so that full-array column x is tensor column x + CPL - 1 (16-B aligned
// boxes: cell 1 is 128-B aligned).  Strip j owns columns
// [1 + OWN j, OWN (j+1)] and loads full columns [1 + OWN j - CPL,
// OWN (j+1) + CPL] (ghost lanes 0 and 31 on either side).
//
// One warp's sweep of its (strip, row segment) for one step: the body of
// the step kernel sw_step_tma, and of every step of the persistent loop
// sw_loop_tma.  `kb` = ring stages the warp consumed before (mbarrier slot
// and phase continue across the steps of a loop); returns the stages this
// sweep consumed (0: the strip owns nothing).
template <class T, bool FAST, int RED, int NW, bool STEP = false>
__device__ __forceinline__ int tma_sweep(const CUtensorMap* tmH, const CUtensorMap* tmU, const CUtensorMap* tmV,
                                         int nx, int ny, int64_t pitch, const SegMap& sm, int alt,
                                         T* __restrict__ oH, T* __restrict__ oU, T* __restrict__ oV, T dx, T dy,
                                         const DtSrc& dts, T g, const BCs& bc, const RedPtrs& red, const Peers& P,
                                         const SyncArgs& sy, uint32_t sbase, uint32_t kb,
                                         const LoopCtl* lc = nullptr, uint32_t target = 0u) {
    using namespace tma;
    using G = Geo<T>;
    constexpr int CPL = G::CPL;
    // one 16-byte vector per lane keeps every TMA box start (tensor column
    // OWN j, i.e. 480 j bytes) 16-byte aligned
    constexpr int DM = FAST ? DIV_FAST : DIV_GUARD;

    const int warp = warp_index();
    const int lane = threadIdx.x & 31;
    const int strip = blockIdx.x * NW + warp;
    const int xs = 1 + strip * G::OWN - CPL;             // full column of the first loaded column (ghost lane 0)
    const int txl = xs + G::LEAD;                        // its tensor column
    const int tx = G::VEC == 16 ? txl : (txl & ~1);      // box start (16-B aligned)
    if (xs + CPL > nx) return 0;                         // strip owns nothing (ragged last band)
    int y0, nrows;                                       // first interior row of the segment, rows
    seg_rows(sm, blockIdx.y, y0, nrows);
    const int nload = nrows + 2;                         // rows y0-1 .. y0+nrows
    const int nstages = (nload + R - 1) / R;
    // Sweep direction (fast mode): with `alt`, odd segments sweep top-down,
    // so the two rows a segment shares with each neighbour segment are loaded
    // by both CTAs at about the same time (both at their start or both at
    // their end) and the second load hits L2 instead of HBM.  A top-down
    // sweep runs the SAME code on the mirror image y -> -y of the segment:
    // rows are consumed in reverse order and hv enters negated; the scheme
    // is mirror-symmetric and every IEEE operation is odd under negation, so
    // the mirrored step yields exactly the negated hv' (and the same h', hu')
    // -- up to the sign of zero results, which is why exact mode (bit-exact
    // contract) always sweeps bottom-up.
    const bool down = FAST && alt && (blockIdx.y & 1);
    const int ytop = y0 + nrows;                         // top loaded row (halo above the segment)
    auto stage_y = [&](int k) { return down ? ytop - k * R - (R - 1) : y0 - 1 + k * R; };
    const T vsign = down ? T(-1) : T(1);
    const int row_bytes = down ? -G::ROWB : G::ROWB;    // stage row step
    const uint32_t ring = sbase + warp * G::WARP_RING;
    const uint32_t full = sbase + NW * G::WARP_RING + warp * tma::S * 8;

    // tile sides this warp exchanges with neighbour tiles (fused halo exchange)
    uint32_t sides = 0;
    if (sync_on(sy)) {
        if (y0 == 1) sides |= 1u << SIDE_D;
        if (y0 + nrows - 1 == ny) sides |= 1u << SIDE_U;
        if (strip == 0) sides |= 1u << SIDE_L;
        if (G::OWN * (strip + 1) >= nx) sides |= 1u << SIDE_R;
    }
    if constexpr (STEP) {
        // the step kernel: programmatic launch and the ring's barriers here,
        // after the geometry (the order the code generator handles best)
        pdl_launch_dependents();
        if (lane == 0) {
            for (int s2 = 0; s2 < tma::S; ++s2) mbar_init(full + 8 * s2, 1);
            asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        }
        __syncwarp();                             // the barriers are initialised before any lane uses them
        pdl_wait();                               // the previous step's output is complete
    }
    if (lc) loop_nbr_wait(*lc, strip, target, lane, red.err);
    if (lane == 0) {
        if (sides) peer_wait(sy, sides, red.err);   // before the first halo load
        // the neighbours' generic-proxy stores are read by TMA (async proxy)
        if (lc) asm volatile("fence.proxy.async.global;" ::: "memory");
        // ring slots are free: the previous sweep's generic reads of them are
        // ordered before the new TMA writes
        if (kb) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        for (int k = 0; k < tma::S - 1 && k < nstages; ++k) {
            const int sl = ((int)kb + k) % tma::S;
            issue_stage<T>(ring + sl * G::STAGE_BYTES, full + 8 * sl, tmH, tmU, tmV, tx, stage_y(k));
        }
    }
    __syncwarp();
    // the rank boards only serve steps that also reduce the next bound (the
    // SPEC run's CFL steps): other instantiations keep the plain path
    T dt;
    if constexpr (RED >= 2) dt = resolve_dt_sync<T>(dts, sy, lane, red.err, lc != nullptr);
    else dt = resolve_dt<T>(dts, lc != nullptr);
    const Coef<T> c = make_coef<T>(dx, dy, dt, g);
    const T dmin = dx < dy ? dx : dy;
    const int X = xs + CPL * lane;             // full column of cell 0 of this lane
    const bool owner = (lane >= 1) && (lane <= 30) && (X <= nx);   // nx % CPL == 0
    // cells whose loaded data is not part of the grid (padding left of column
    // 0 in strip 0, zero-fill right of column nx+1) are replaced by a lake at
    // rest so they cannot trip the exact-division guard; they feed no owned cell
    int bad = 0;
#pragma unroll
    for (int i = 0; i < CPL; ++i)
        if (X + i < 0 || X + i > nx + 1) bad |= 1 << i;
    const bool any_bad = __any_sync(0xffffffffu, bad != 0);
    const bool edge_rows = (y0 == 1) || (y0 + nrows - 1 == ny);
    const bool edge_cols = owner && ((X == 1) || (X + CPL - 1 == nx));
    const uint32_t lane_off = (uint32_t)G::VEC * lane + (uint32_t)((txl - tx) * (int)sizeof(T));

    // the y-sweep's register window: packed-pair engine for f32 fast mode
    // (sw_pair.cuh), scalar engine otherwise
    constexpr bool PAIR = FAST && sizeof(T) == 4 && FKC_TMA_PAIR;
    constexpr bool EXACT_PAIR = !FAST && sizeof(T) == 4 && FKC_TMA_EXACT_PAIR;
    using ExactEngine = typename std::conditional<FKC_TMA_EXACT_PAIR == 2, ExactPairEngine2, ExactPairEngine>::type;
    using Engine = typename std::conditional<
        PAIR, PairEngine,
        typename std::conditional<EXACT_PAIR, ExactEngine, ScalarEngine<T, CPL>>::type>::type;
    Engine eng;
    eng.init(c);
    // element offset of the row updated at loaded-row index n (lane's cell 0),
    // advanced by one row per loaded row
    const int64_t row_step = down ? -pitch : pitch;
    int64_t row_off = (int64_t)(down ? ytop + 1 : y0 - 2) * pitch + X;
    RowRed<T, FAST, RED> rr;
    rr.init();
    T fdep = T(INFINITY);              // min face depth (fused reductions only)
    bool fix_mode = false;             // exact mode: current division variant (warp-uniform)
    int fix_rows = 0;
    constexpr int UNR = FAST ? FKC_FAST_UNROLL : (sizeof(T) == 8 ? FKC_EXACT_UNROLL_F64 : FKC_EXACT_UNROLL);
    constexpr bool EXACT2 = EXACT_PAIR && FKC_TMA_EXACT_PAIR == 2;
    // stores of an updated row (owner lanes): the three 16-B row vectors,
    // then -- tile-edge lanes only, out of line to keep the sweep loop small --
    // the output halo (boundary conditions) and the fused halo exchange, and
    // the fused reductions
    auto store_row = [&](int y, T (&oh)[CPL], T (&ou)[CPL], T (&ov)[CPL]) {
        const int64_t off = row_off;
        stg_row<T, CPL>(oH + off, oh);
        stg_row<T, CPL>(oU + off, ou);
        stg_row<T, CPL>(oV + off, ov);
        if ((edge_rows && (y == 1 || y == ny)) || edge_cols) {
            Row3<T, CPL> o;
#pragma unroll
            for (int i = 0; i < CPL; ++i) { o.h[i] = oh[i]; o.u[i] = ou[i]; o.v[i] = ov[i]; }
            edge_stores<T, CPL>(oH, oU, oV, pitch, nx, ny, X, y, bc, P, o);
        }
        if constexpr (RED > 0) rr.template add_row<CPL>(oh, ou, ov, g);
    };

    // The loop bound is re-derived from %ctaid.y (a volatile read the
    // compiler cannot hoist) instead of being kept live: in the reduction
    // variants at the 168-register cap it was otherwise spilled, and with
    // 3 x 74 KB of shared memory per SM the local-memory reload went to L2
    // every stage.
    auto stages_left = [&](int k) {
        uint32_t cy;
        asm volatile("mov.u32 %0, %%ctaid.y;" : "=r"(cy));
        int yy0, nr;
        seg_rows(sm, (int)cy, yy0, nr);
        return k < (nr + 2 + R - 1) / R;
    };
    for (int k = 0; stages_left(k); ++k) {
        const int kg = (int)kb + k;                    // ring stage index over the warp's lifetime
        const int s = kg % tma::S;
        // refill the slot freed by stage k-1 (every lane finished reading it)
        if (lane == 0 && k + tma::S - 1 < nstages) {
            const int kn = k + tma::S - 1;
            const int sl = ((int)kb + kn) % tma::S;
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue_stage<T>(ring + sl * G::STAGE_BYTES, full + 8 * sl, tmH, tmU, tmV, tx, stage_y(kn));
        }
        mbar_wait(full + 8 * s, (kg / tma::S) & 1, red.err);
        // cells whose loaded data is not part of the grid become a lake at
        // rest IN SHARED MEMORY (the lane's own 16-B slots of the stage, read
        // back by the same lane: program order suffices; the slot's next TMA
        // refill is ordered by the fence.proxy.async above) -- keeps the row
        // loop free of a conditional overwrite of the loaded registers
        if (any_bad && bad) {
            const uint32_t s0 = ring + s * G::STAGE_BYTES + lane_off;
#pragma unroll
            for (int rr2 = 0; rr2 < R; ++rr2)
#pragma unroll
                for (int f = 0; f < 3; ++f)
#pragma unroll
                    for (int i = 0; i < CPL; ++i)
                        if (bad & (1 << i)) {
                            const uint32_t a = s0 + rr2 * G::ROWB + f * G::FIELD_BYTES + i * (uint32_t)sizeof(T);
                            if constexpr (sizeof(T) == 4)
                                asm volatile("st.shared.f32 [%0], %1;" :: "r"(a), "f"(f == 0 ? 1.0f : 0.0f) : "memory");
                            else
                                asm volatile("st.shared.f64 [%0], %1;" :: "r"(a), "d"(f == 0 ? 1.0 : 0.0) : "memory");
                        }
        }
        // first row of the stage in sweep order (boxes are stored bottom-up)
        const uint32_t st = ring + s * G::STAGE_BYTES + lane_off + (down ? (R - 1) * G::ROWB : 0);
#pragma unroll UNR
        for (int r = 0; r < R; ++r) {
            const int n = k * R + r;              // loaded row index; row y0-1+n (top-down: ytop-n)
            const uint32_t sr = st + r * row_bytes;
            // the row's H, U, V vectors from shared memory (re-read, not kept
            // live, when exact mode redoes the row: 12 registers fewer)
            auto load_row = [&](VecF<T>& hv, VecF<T>& uv, VecF<T>& vv) {
                hv = lds_vec<T>(sr);
                uv = lds_vec<T>(sr + G::FIELD_BYTES);
                vv = lds_vec<T>(sr + 2 * G::FIELD_BYTES);
                if (FAST) {
#pragma unroll
                    for (int i = 0; i < CPL; ++i) vv.v[i] *= vsign;   // mirror image (top-down sweep)
                }
            };
            VecF<T> hv, uv, vv;
            load_row(hv, uv, vv);
            const bool have_prev = n >= 1;
            const bool want_x = (n >= 1) && (n <= nrows);
            const bool upd = (n >= 2) && (n <= nrows + 1);
            const int y_upd = down ? ytop - n + 1 : y0 + n - 2;   // row updated at this step
            bool ok = true;
            if constexpr (EXACT2) {
                // exact mode, two guarded phases per row (sw_pair.cuh
                // ExactPairEngine2); a phase that saw a non-benign operand or a
                // subnormal tie in any lane is redone with DIV_FIXUP
                eng.template cells_y<DIV_GUARD>(hv, uv, vv, have_prev, ok);
                if (__any_sync(0xffffffffu, !ok)) {
                    VecF<T> h2, u2, v2;
                    asm volatile("" ::: "memory");       // a fresh shared load, not the first one kept live
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
                if constexpr (RED > 0) {
                    const bool xrow = (n >= 1) && (n <= nrows);
                    const bool yrow = (n >= 1) && (n <= nrows + 1);
                    eng.track(fdep, owner && xrow, lane == 0 && xrow, owner && yrow);
                }
                row_off += row_step;
                eng.shift();
#if FKC_EXACT_ROWSYNC
                __syncwarp();      // keeps ptxas from interleaving unrolled rows (register peak)
#endif
                continue;
            }
            if constexpr (FAST) {
                // branch-free: the faces of the first loaded row / of rows past the
                // segment are computed on benign or discarded data, never stored
                eng.template row<DIV_FAST>(hv, uv, vv, true, true, c, ok);
            } else {
                // exact mode, warp-uniform per row: lean guarded division;
                // if any lane saw a non-benign operand, redo the row with the
                // never-failing DIV_FIXUP variant (scaled tiny numerators,
                // per-numerator __fdiv_rn for the rest).  Tiny-valued regions
                // are contiguous along the sweep, so after a row needed the
                // fixup variant the next rows start with it and the lean
                // variant is retried every 16 rows.
                if (!fix_mode && !FKC_EXACT_ALWAYS_FIXUP) {
                    eng.template row<DIV_GUARD>(hv, uv, vv, have_prev, want_x, c, ok);
                    if (__any_sync(0xffffffffu, !ok)) {
                        fix_mode = FKC_FIX_PERSIST > 0;
                        fix_rows = 0;
                        VecF<T> h2, u2, v2;
                        asm volatile("" ::: "memory");   // a fresh shared load, not the first one kept live
                        load_row(h2, u2, v2);
                        eng.template row<DIV_FIXUP>(h2, u2, v2, have_prev, want_x, c, ok);
                    }
                } else {
                    eng.template row<DIV_FIXUP>(hv, uv, vv, have_prev, want_x, c, ok);
                    if (++fix_rows >= FKC_FIX_PERSIST) fix_mode = false;
                }
            }
            if constexpr (RED > 0) {
                // face depths of the faces owned cells use (NonPositiveDepth:
                // any face or cell h <= 0): x-faces of the
                // segment's rows, y-faces from below its first row to above
                // its last
                const bool xrow = (n >= 1) && (n <= nrows);
                const bool yrow = (n >= 1) && (n <= nrows + 1);
                eng.track(fdep, owner && xrow, lane == 0 && xrow, owner && yrow);
            }
            // full-step update of the previous row (row y0 + n - 2; top-down: ytop - n + 1)
            if (FAST || upd) {
                T oh[CPL], ou[CPL], ov[CPL];
                eng.template update<DM>(c, oh, ou, ov);
                if (FAST) {
#pragma unroll
                    for (int i = 0; i < CPL; ++i) ov[i] *= vsign;   // back from the mirror image
                }
                if (owner && upd) store_row(y_upd, oh, ou, ov);
            }
            row_off += row_step;
            // shift the register window (renamed away by the unrolled loop)
            eng.shift();
        }
        __syncwarp();
    }
    if (sides) {
        __threadfence_system();
        __syncwarp();
        const int nstrips = (nx - 1) / G::OWN + 1;
        const int expected[4] = {(int)gridDim.y, (int)gridDim.y, nstrips, nstrips};
        if (lane == 0) peer_signal(sy, sides, expected);
    }
    if constexpr (RED > 0) {
        rr.commit(red, lane, dmin, fdep);
        // decomposed SPEC run: the last committing warp publishes the tile's
        // CFL bound to every rank's board
        if (RED >= 2 && lane == 0 && sy.nranks > 0)
            board_publish(sy, red.cfl_min, (uint32_t)(((nx - 1) / G::OWN + 1) * gridDim.y));
    }
    return nstages;
}

// One time step: every warp sweeps its (strip, segment) once.
template <class T, bool FAST, int RED, int NW>
__global__ void __launch_bounds__(NW * 32, tma::Blk<T, NW>::template ctas_per_sm<FAST, RED>())
sw_step_tma(const __grid_constant__ CUtensorMap tmH, const __grid_constant__ CUtensorMap tmU,
            const __grid_constant__ CUtensorMap tmV, int nx, int ny, int64_t pitch, const __grid_constant__ SegMap sm,
            int alt,
            T* __restrict__ oH, T* __restrict__ oU, T* __restrict__ oV,
            T dx, T dy, DtSrc dts, T g, const __grid_constant__ BCs bc, RedPtrs red,
            const __grid_constant__ Peers P, const __grid_constant__ SyncArgs sy) {
    extern __shared__ __align__(128) uint8_t smem_raw[];
    const uint32_t sbase = (smem_u32(smem_raw) + 127u) & ~127u;
    tma_sweep<T, FAST, RED, NW, true>(&tmH, &tmU, &tmV, nx, ny, pitch, sm, alt, oH, oU, oV, dx, dy, dts, g, bc, red,
                                      P, sy, sbase, 0u);
}

// ---------------------------------------------------------------------------
// Wavefront launch of the streamed host run (fkc_sw_run_host): one launch
// advances several row bands, each by one step of its own (task k =
// blockIdx.z: band rows [ybase, ybase + nyw), global step parity -> which
// buffer it reads / writes, its step's reduction row).  The host schedules
// tasks of one launch two bands apart per step, so no task reads rows
// another task of the same launch writes.
// ---------------------------------------------------------------------------
constexpr int WAVE_MAX_TASKS = 40;
struct WaveTask {
    int odd;                       // global step parity: 0 reads A writes B, 1 reads B writes A
    int ybase, nyw;
    unsigned long long* red_row;   // 5-word reduction row of the task's step, or null
};
struct WaveArgs {
    WaveTask t[WAVE_MAX_TASKS];
    int ntask, seg;
};

template <class T, bool FAST, int RED, int NW>
__global__ void __launch_bounds__(NW * 32, tma::Blk<T, NW>::template ctas_per_sm<FAST, RED>())
sw_wave_tma(const __grid_constant__ CUtensorMap mA0, const __grid_constant__ CUtensorMap mA1,
            const __grid_constant__ CUtensorMap mA2, const __grid_constant__ CUtensorMap mB0,
            const __grid_constant__ CUtensorMap mB1, const __grid_constant__ CUtensorMap mB2, int nx, int ny,
            int64_t pitch, int alt, const __grid_constant__ LoopBufs bufs, T dx, T dy, T dt, T g,
            const __grid_constant__ BCs bc, const __grid_constant__ WaveArgs w) {
    const WaveTask& tk = w.t[blockIdx.z];
    pdl_launch_dependents();
    if ((int)blockIdx.y * w.seg >= tk.nyw) return;           // this task has fewer segments
    extern __shared__ __align__(128) uint8_t smem_raw[];
    const uint32_t sbase = (smem_u32(smem_raw) + 127u) & ~127u;
    const int warp = warp_index();
    const uint32_t full = sbase + NW * tma::Geo<T>::WARP_RING + warp * tma::S * 8;
    if ((threadIdx.x & 31) == 0) {
        for (int s = 0; s < tma::S; ++s) mbar_init(full + 8 * s, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    const SegMap sm{w.seg, 0, 0, 0, tk.ybase, tk.nyw};
    const bool odd = tk.odd != 0;
    void* const* out = odd ? bufs.a : bufs.b;
    RedPtrs red{nullptr, nullptr, nullptr, nullptr, nullptr};
    if (tk.red_row)
        red = RedPtrs{(double*)tk.red_row, tk.red_row + 1, tk.red_row + 2, nullptr, (uint32_t*)(tk.red_row + 4)};
    const DtSrc dts{(double)dt, nullptr, 1.0};
    pdl_wait();                                   // the previous launch's output is complete
    tma_sweep<T, FAST, RED, NW>(odd ? &mB0 : &mA0, odd ? &mB1 : &mA1, odd ? &mB2 : &mA2, nx, ny, pitch, sm, alt,
                                (T*)out[0], (T*)out[1], (T*)out[2], dx, dy, dts, g, bc, red, c_no_peers, c_no_sync,
                                sbase, 0u);
}

// ---------------------------------------------------------------------------
// Persistent time loop (mid-size grids, fkc_sw_advance_n): the step grid is
// launched ONCE (cooperatively: every warp resident) and each warp sweeps
// the same (strip, segment) step after step.  Between steps a warp waits
// only for its direct neighbours -- left / right strips of its segment,
// segments below / above in its strip, and the periodic wrap partners,
// i.e. every warp whose cells it reads (its loaded columns and halo rows)
// or whose reads of the buffer it is about to overwrite it must not race
// (double buffering: step s+1 overwrites state s-1) -- through per-warp
// step counters in global memory (release / acquire).  Cells of the
// diagonal neighbours that the TMA boxes bring in (ghost lanes of the halo
// rows) feed no stored value.  With a CFL-chosen dt every step ends in a
// grid-wide arrival (two-level counters) so the next dt sees every warp's
// bound.  No launch per step, no tail wave, the state stays in L2.
// ---------------------------------------------------------------------------
// f32 fast mode: the loop's extra live state does not fit the step
// kernel's 168-register budget (12 warps per SM) without spills; the loop
// kernel runs FKC_LOOP_WARPS_FAST warps per SM instead (registers are split
// over the 4 SM sub-partitions: 9-12 warps cap a warp at 168, 8 at 255)
#ifndef FKC_LOOP_WARPS_FAST
#define FKC_LOOP_WARPS_FAST 8
#endif
template <class T, bool FAST, int RED, int NW>
constexpr int loop_ctas_per_sm() {
    return (FAST && sizeof(T) == 4) ? (FKC_LOOP_WARPS_FAST / NW > 0 ? FKC_LOOP_WARPS_FAST / NW : 1)
                                    : tma::Blk<T, NW>::template ctas_per_sm<FAST, RED>();
}
template <class T, bool FAST, int RED, int NW>
__global__ void __launch_bounds__(NW * 32, (loop_ctas_per_sm<T, FAST, RED, NW>()))
sw_loop_tma(const __grid_constant__ CUtensorMap mA0, const __grid_constant__ CUtensorMap mA1,
            const __grid_constant__ CUtensorMap mA2, const __grid_constant__ CUtensorMap mB0,
            const __grid_constant__ CUtensorMap mB1, const __grid_constant__ CUtensorMap mB2, int nx, int ny,
            int64_t pitch, SegMap sm, int alt, const __grid_constant__ LoopBufs bufs, T dx, T dy, T g,
            const __grid_constant__ BCs bc, const __grid_constant__ LoopCtl ctl) {
    extern __shared__ __align__(128) uint8_t smem_raw[];
    const uint32_t sbase = (smem_u32(smem_raw) + 127u) & ~127u;
    const int warp = warp_index();
    const int lane = threadIdx.x & 31;
    const uint32_t full = sbase + NW * tma::Geo<T>::WARP_RING + warp * tma::S * 8;
    const int strip = blockIdx.x * NW + warp;
    if (strip >= ctl.nstrips) return;               // owns nothing (no neighbour waits on it)
    if (lane == 0) {
        for (int s = 0; s < tma::S; ++s) mbar_init(full + 8 * s, 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    const int nseg = (int)gridDim.y, ns = ctl.nstrips;
    const int me = (int)blockIdx.y * ns + strip;
    // grid-wide arrival (CFL mode): warp `me` arrives on sub-counter me % 32
    const int nwarps = nseg * ns;
    const int nsub = nwarps < 32 ? nwarps : 32;
    const uint32_t sub_n = (uint32_t)(nwarps / 32 + ((me % 32) < (nwarps % 32) ? 1 : 0));
    const bool cfl_loop = ctl.dt_from_slots != 0;
    uint32_t kb = 0;
    for (int64_t s = 0; s < ctl.steps; ++s) {
        const int64_t i = ctl.first + s;
        const bool even = (i & 1) == 0;
        const CUtensorMap* m0 = even ? &mA0 : &mB0;
        const CUtensorMap* m1 = even ? &mA1 : &mB1;
        const CUtensorMap* m2 = even ? &mA2 : &mB2;
        void* const* out = even ? bufs.b : bufs.a;
        DtSrc dts{ctl.dt, nullptr, ctl.cfl};
        RedPtrs red{nullptr, nullptr, nullptr, nullptr, nullptr};
        if (ctl.slots) {
            unsigned long long* row = ctl.slots + 5 * (i + 1);
            red = RedPtrs{(double*)row, row + 1, row + 2, ctl.want_cfl ? row + 3 : nullptr, (uint32_t*)(row + 4)};
            if (cfl_loop) dts.bound = ctl.slots + 5 * i + 3;
        }
        const int n = tma_sweep<T, FAST, RED, NW>(m0, m1, m2, nx, ny, pitch, sm, alt, (T*)out[0], (T*)out[1],
                                                  (T*)out[2], dx, dy, dts, g, bc, red, c_no_peers, c_no_sync, sbase, kb,
                                                  (s > 0 && !cfl_loop) ? &ctl : nullptr, (uint32_t)s);
        kb += (uint32_t)n;
        __syncwarp();                                // every lane's stores (and reduction atomics) issued
        if (lane == 0) {
            asm volatile("fence.proxy.async.global;" ::: "memory");   // our stores, read by TMA next
            if (cfl_loop) {
                __threadfence();
                // grid-wide arrival: the last warp of a sub-counter bumps the top
                const uint32_t old = atomicAdd(ctl.bar + (me % 32), 1u);
                if (old + 1u == sub_n * (uint32_t)(s + 1)) {
                    __threadfence();
                    atomicAdd(ctl.bar + 32, 1u);
                }
                spin_until(ctl.bar + 32, (uint32_t)nsub * (uint32_t)(s + 1), red.err);
                asm volatile("fence.proxy.async.global;" ::: "memory");
            } else {
                st_release_gpu(ctl.flags + me, (uint32_t)(s + 1));
            }
        }
        __syncwarp();
    }
}

}  // namespace fkc
