// fkc_sw.cu -- C-ABI entry points (include/fkc_sw.h) over the sm_100a
// kernels in sw_kernels.cuh.  Host code only validates arguments, encodes
// (and caches) the TMA tensor maps and launches; it never synchronises.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <chrono>
#include <mutex>
#include <vector>
#include <string>

#include "../../include/fkc_sw.h"
#include "sw_tma.cuh"
#include "sw_resident.cuh"

#ifndef FKC_GEN_BX
#define FKC_GEN_BX 64              // generic kernel CTA: 64 x 4 cells
#endif
#ifndef FKC_GEN_BY
#define FKC_GEN_BY 4
#endif

using namespace fkc;

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}

int check_launch(const char* what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(FKC_ECUDA, "%s: %s", what, cudaGetErrorString(e));
    return FKC_OK;
}

bool valid_grid(const fkc_grid* g) {
    return g && g->nx >= 1 && g->ny >= 1 && g->pitch >= (int64_t)g->nx + 2 &&
           (g->dtype == FKC_F32 || g->dtype == FKC_F64);
}

bool valid_bc(const int32_t* bc) {
    for (int i = 0; i < 4; ++i)
        if (bc[i] < FKC_BC_REFLECTIVE || bc[i] > FKC_BC_NONE) return false;
    // periodic must be paired on an axis
    if ((bc[0] == FKC_BC_PERIODIC) != (bc[1] == FKC_BC_PERIODIC)) return false;
    if ((bc[2] == FKC_BC_PERIODIC) != (bc[3] == FKC_BC_PERIODIC)) return false;
    return true;
}

BCs to_bcs(const int32_t* bc) {
    BCs b;
    for (int i = 0; i < 4; ++i) b.s[i] = bc[i];
    return b;
}

RedPtrs to_red(const fkc_sw_reduce& r) {
    RedPtrs p;
    p.mass = r.mass;
    p.max_u = (unsigned long long*)r.max_abs_u;
    p.max_v = (unsigned long long*)r.max_abs_v;
    p.cfl_min = (unsigned long long*)r.cfl_min;
    p.err = r.err;
    return p;
}

bool any_red(const RedPtrs& p) { return p.mass || p.max_u || p.max_v || p.cfl_min || p.err; }

Peers to_peers(const fkc_sw_step_args* a) {
    Peers P;
    for (int s = 0; s < 4; ++s) {
        for (int f = 0; f < 3; ++f) P.s[s].p[f] = a->peer[s].p[0] ? a->peer[s].p[f] : nullptr;
        P.s[s].stride = a->peer[s].stride;
    }
    return P;
}

SyncArgs to_sync(const fkc_sw_step_args* a) {
    SyncArgs S;
    for (int s = 0; s < 4; ++s) {
        S.wait[s] = a->sync.wait[s];
        S.signal[s] = a->sync.signal[s];
    }
    S.counter = a->sync.counter;
    S.epoch = a->sync.epoch;
    S.board = (unsigned long long*)a->sync.cfl_board;
    for (int r = 0; r < FKC_MAX_RANKS; ++r) S.peers[r] = (unsigned long long*)a->sync.cfl_peers[r];
    S.ccount = a->sync.cfl_counter;
    S.rank = a->sync.cfl_rank;
    S.nranks = a->sync.cfl_board ? a->sync.cfl_nranks : 0;
    return S;
}

int valid_peers(const fkc_sw_step_args* a) {
    for (int s = 0; s < 4; ++s) {
        const fkc_peer_line& l = a->peer[s];
        if (!l.p[0]) continue;
        if (!l.p[1] || !l.p[2]) return fail(FKC_EUSAGE, "peer line %d: null field pointer", s);
        if (a->bc[s] != FKC_BC_NONE) return fail(FKC_EUSAGE, "peer line %d needs bc NONE on that side", s);
        if (s >= 2 ? l.stride != 1 : l.stride < (int64_t)1) return fail(FKC_EUSAGE, "peer line %d: bad stride", s);
    }
    const fkc_sync& y = a->sync;
    if (y.counter) {
        for (int s = 0; s < 4; ++s)
            if ((y.wait[s] != nullptr) != (y.signal[s] != nullptr))
                return fail(FKC_EUSAGE, "sync side %d: wait and signal must be given together", s);
    }
    if (y.flags & ~FKC_SYNC_PDL) return fail(FKC_EUSAGE, "sync.flags: unknown bits");
    if (y.cfl_board) {
        if (y.cfl_nranks < 1 || y.cfl_nranks > FKC_MAX_RANKS || y.cfl_rank < 0 || y.cfl_rank >= y.cfl_nranks)
            return fail(FKC_EUSAGE, "sync: cfl_nranks must be 1..%d and cfl_rank < cfl_nranks", FKC_MAX_RANKS);
        if (!y.cfl_counter) return fail(FKC_EUSAGE, "sync: cfl_counter missing");
        for (int r = 0; r < y.cfl_nranks; ++r)
            if (!y.cfl_peers[r]) return fail(FKC_EUSAGE, "sync: cfl_peers[%d] missing", r);
    }
    return FKC_OK;
}

int valid_tune(const fkc_sw_tune& t) {
    if (t.seg < 0) return fail(FKC_EUSAGE, "tune.seg must be >= 0");
    if (t.tail_rows < -1) return fail(FKC_EUSAGE, "tune.tail_rows must be >= -1");
    if (t.tail_waves < 0 || t.tail_waves > 64) return fail(FKC_EUSAGE, "tune.tail_waves must be in 0..64");
    if (t.order < 0 || t.order > 2) return fail(FKC_EUSAGE, "tune.order must be 0, 1 or 2");
    if (t.parity != 0 && t.parity != 1) return fail(FKC_EUSAGE, "tune.parity must be 0 or 1");
    if (t.warps != 0 && t.warps != 1 && t.warps != 2 && t.warps != 4)
        return fail(FKC_EUSAGE, "tune.warps must be 0 (auto), 1, 2 or 4");
    if ((t.no_pdl | t.no_alternate) & ~1) return fail(FKC_EUSAGE, "tune.no_pdl / no_alternate must be 0 or 1");
    return FKC_OK;
}

bool peers_tma_ok(const fkc_sw_step_args* a, int es) {
    for (int s = 2; s < 4; ++s)
        for (int f = 0; f < 3; ++f)
            if (a->peer[s].p[0] && (((uintptr_t)a->peer[s].p[f]) + es) % 16 != 0) return false;
    return true;
}

// ---------------------------------------------------------------------------
// TMA tensor maps (driver entry point fetched through the runtime so the
// library does not link libcuda directly)
// ---------------------------------------------------------------------------
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiledFn encode_fn() {
    static EncodeTiledFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (EncodeTiledFn)p;
    });
    return fn;
}

struct MapKey {
    const void* p;
    int nx, ny;
    int64_t pitch;
    int boxw, boxh, esize;
    bool operator==(const MapKey& o) const {
        return p == o.p && nx == o.nx && ny == o.ny && pitch == o.pitch && boxw == o.boxw && boxh == o.boxh &&
               esize == o.esize;
    }
};

struct MapCache {
    static constexpr int N = 64;
    MapKey key[N];
    alignas(64) CUtensorMap map[N];
    int next = 0, used = 0;
    std::mutex mu;
};
MapCache g_maps;

// Map over one field (f32 / f64, element size esize) whose element (0,0) is
// at `p`: tensor column t is full column t - (CPL-1), CPL = 16 / esize, so
// box starts stay 16-B aligned when column 1 is.
int get_map(const void* p, int nx, int ny, int64_t pitch, int boxw, int esize, CUtensorMap* out) {
    MapKey k{p, nx, ny, pitch, boxw, tma::R, esize};
    std::lock_guard<std::mutex> lk(g_maps.mu);
    for (int i = 0; i < g_maps.used; ++i)
        if (g_maps.key[i] == k) { *out = g_maps.map[i]; return FKC_OK; }
    EncodeTiledFn fn = encode_fn();
    if (!fn) return fail(FKC_ECUDA, "cuTensorMapEncodeTiled unavailable");
    alignas(64) CUtensorMap m;
    const int lead = 16 / esize - 1;
    cuuint64_t dims[2] = {(cuuint64_t)nx + 2 + lead, (cuuint64_t)ny + 2};
    cuuint64_t strides[1] = {(cuuint64_t)pitch * esize};
    cuuint32_t box[2] = {(cuuint32_t)boxw, (cuuint32_t)tma::R};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = fn(&m, esize == 4 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2,
                    (void*)((const char*)p - (size_t)lead * esize), dims, strides, box, estr,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                    CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(FKC_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    int slot = g_maps.next;
    g_maps.key[slot] = k;
    g_maps.map[slot] = m;
    g_maps.next = (slot + 1) % MapCache::N;
    if (g_maps.used < MapCache::N) g_maps.used++;
    *out = m;
    return FKC_OK;
}

bool tma_eligible(const fkc_sw_step_args* a) {
    const fkc_grid& g = a->grid;
    const int es = g.dtype == FKC_F32 ? 4 : 8, cpl = 16 / es;
    if ((g.nx % cpl) != 0 || (g.pitch % cpl) != 0) return false;
    const void* ps[6] = {a->H, a->U, a->V, a->oH, a->oU, a->oV};
    for (const void* p : ps)
        if ((((uintptr_t)p) + es) % 16 != 0) return false;
    return peers_tma_ok(a, es);
}

// Launch with programmatic dependent launch (see pdl_wait in sw_kernels.cuh).
// `pdl` false: plain launch -- for grids below ~512^2 (B200, CUDA graphs: the
// programmatic edge costs more than it hides, 256^2 fast 26 -> 20 Gcell/s)
// and with the fused exchange unless every neighbour tile runs on another
// GPU (sync.flags FKC_SYNC_PDL): CTAs parked in griddepcontrol.wait must not
// hold SMs a neighbour tile's kernel on the same GPU needs.
template <class... KArgs, class... Args>
void launch_step(void (*kern)(KArgs...), dim3 grd, dim3 blk, size_t smem, cudaStream_t st, bool pdl, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grd;
    cfg.blockDim = blk;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = pdl ? 1 : 0;
    cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

template <class T>
int launch_generic(const fkc_sw_step_args* a, cudaStream_t st) {
    const fkc_grid& g = a->grid;
    DtSrc dts{a->dt, (const unsigned long long*)a->dt_bound, a->cfl};
    RedPtrs red = to_red(a->red);
    dim3 blk(FKC_GEN_BX, FKC_GEN_BY);
    dim3 grd((g.nx + FKC_GEN_BX - 1) / FKC_GEN_BX, (g.ny + FKC_GEN_BY - 1) / FKC_GEN_BY);
    const bool fast = a->mode == FKC_MODE_FAST;
    const bool r = any_red(red);
    const bool pdl = !a->tune.no_pdl && (int64_t)g.nx * g.ny >= (1 << 18) &&
                     (a->sync.counter == nullptr || (a->sync.flags & FKC_SYNC_PDL));
#define GEN_ARGS g.nx, g.ny, g.pitch, (const T*)a->H, (const T*)a->U, (const T*)a->V, (T*)a->oH, (T*)a->oU, \
                 (T*)a->oV, T(a->dx), T(a->dy), dts, T(a->g), to_bcs(a->bc), red, to_peers(a), to_sync(a)
    if (fast) {
        if (r) launch_step(sw_step_generic<T, DIV_FAST, true>, grd, blk, 0, st, pdl, GEN_ARGS);
        else launch_step(sw_step_generic<T, DIV_FAST, false>, grd, blk, 0, st, pdl, GEN_ARGS);
    } else {
        if (r) launch_step(sw_step_generic<T, DIV_IEEE, true>, grd, blk, 0, st, pdl, GEN_ARGS);
        else launch_step(sw_step_generic<T, DIV_IEEE, false>, grd, blk, 0, st, pdl, GEN_ARGS);
    }
#undef GEN_ARGS
    return check_launch("sw_step_generic");
}

// SMs of the current device (148 on a B200), cached per device
int sm_count() {
    static int cached[64] = {0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
    if (cached[dev] == 0) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev);
        cached[dev] = v > 0 ? v : 148;
    }
    return cached[dev];
}

// SEG_LEAN: an f32 fast-mode step with fused reductions on a grid of <= 2^22 cells.
// Every segment ends in its reduction atomics and starts with the dt bound
// read, so there fewer, longer segments win: >= 1.5 waves instead of 3 and
// no guided tail (scripts/red_cost.py --seg/--warps sweep, CFL step: 1024^2
// 13.6 -> 12.3 us, 2048^2 35.4 -> 32.0; 4096^2 and exact mode keep the
// default schedule, which is best there).
// SEG_LONG: an f32 CFL step (RED 2) on a grid of > 2^26 cells -- its
// per-segment commit and bound read favour long segments even there:
// uniform 46-row segments (16384^2 CFL, 2-warp CTAs: 257.1 -> 260.4 Gcell/s;
// the diagnostics-only and plain steps are best with the default).
// SEG_HBM: the plain f32 fast step (no reductions) on a grid of >= 3*2^25
// cells, launched eagerly: uniform 14-row segments (16 loaded rows = 4 whole
// TMA stages) and no guided tail -- 16384^2 268.5 -> 278.2 Gcell/s, 32768^2
// 273.6 -> 281.8, 11584^2 265 -> 272 (bench.py --seg sweep, round 2; DRAM
// traffic stays 0.995x the algorithmic bytes, ncu); smaller grids, exact
// mode, the reducing steps and captured launches keep their own schedules
// (14-row segments cost them 4-15 %).
// SEG_NOTAIL: f64 on > 2^26 cells -- the default length without the guided
// tail (16384^2 fast 131.6-132.4 -> 133.9, exact 84.6 -> 85.5 Gcell/s).
// SEG_FINE: the f32 exact step on 23*2^20 .. 2^27 cells, launched eagerly:
// uniform segments, the longest of 30/22/18/14/10 rows that still gives
// >= 18 waves of CTAs -- many small CTAs balance the FMA-bound sweeps
// (bench.py --seg sweep: 6144^2 116.6 -> 129.0 (10 rows), 8192^2 134.8 ->
// 142.4 (14 rows), 5000^2 110.7 -> 118.6 (10 rows), 8192^2 diagnostics
// 127.3 -> 132.2, CFL 110.1 -> 111.5;
// 11584^2 and 16384^2 unchanged, 4096^2 best with the default).
// SEG_18: the plain f32 fast step on 2^26 .. 3*2^25 cells (8192^2 class):
// uniform 18-row segments, eager or captured (8192^2 eager 255.5 -> 259.5,
// graph 261.8 -> 266.7 Gcell/s).
// SEG_TINY: the plain f32 exact step below 2^20 cells: uniform 2-row
// segments (one 4-row TMA stage per warp; 512^2 19.6 -> 36.3 Gcell/s on
// the TMA kernel, the default's 6-row segments leave too few warps for the
// FMA-bound engine).
enum SegShape { SEG_DEFAULT = 0, SEG_LEAN = 1, SEG_LONG = 2, SEG_HBM = 3, SEG_NOTAIL = 4, SEG_FINE = 5, SEG_18 = 6,
                SEG_TINY = 7 };
int pick_seg(int nbands, int ny, int ctas_per_sm, const fkc_sw_tune& t, int shape = SEG_DEFAULT) {
    if (t.seg > 0) return t.seg;
    if (shape == SEG_LONG) return 46;
    if (shape == SEG_HBM) return 14;
    if (shape == SEG_18) return 18;
    if (shape == SEG_TINY) return 2;
    if (shape == SEG_FINE) {
        const int64_t want = 18 * (int64_t)sm_count() * ctas_per_sm;
        for (int seg : {30, 22, 18, 14})
            if ((int64_t)nbands * ((ny + seg - 1) / seg) >= want) return seg;
        return 10;
    }
    const bool lean = shape == SEG_LEAN;
    // Rows per CTA segment.  Long segments amortise the 2 halo rows and the
    // pipeline prologue; short ones shrink the tail of the last wave.  A
    // segment loads seg + 2 rows in stages of R = 4, so seg = 4k - 2 wastes
    // no row of its last stage (1024^2: 6 rows 114 vs 8 rows 87 Gcell/s).
    // B200 sweeps (profiles/r01/seg_sweep2.json, seg_sweep3.json): take the
    // longest of 30/22/14/10/6 rows that still gives >= 3 waves of CTAs; on
    // smaller grids the one whose CTAs fill the last wave best.
    const int cands[5] = {30, 22, 14, 10, 6};
    const int64_t slots = (int64_t)sm_count() * ctas_per_sm;
    for (int seg : cands)
        if ((lean ? 2 : 1) * (int64_t)nbands * ((ny + seg - 1) / seg) >= 3 * slots) return seg;
    int best = 6;
    double best_fill = -1.0;
    for (int seg : cands) {
        const int64_t c = (int64_t)nbands * ((ny + seg - 1) / seg);
        const double fill = (double)c / (double)(((c + slots - 1) / slots) * slots);
        if (fill > best_fill + 1e-9) { best_fill = fill; best = seg; }
    }
    return best;
}

// Segment order: alternate per step (tune.parity, the global step index's
// parity in fkc_sw_advance_n), so each step starts with the rows its
// predecessor wrote last (still in L2).  Carried in the argument block, so
// concurrent callers, streams and captured graphs never share state.
int seg_rev(const fkc_sw_tune& t) {
    if (t.order == 1) return 0;
    if (t.order == 2) return 1;
    return t.parity & 1;
}

// Guided segmentation: the last ~tail_waves waves of CTAs get short
// segments of `tail` rows.
SegMap pick_segmap(int nbands, int ny, int ctas_per_sm, const fkc_sw_tune& t, int shape = SEG_DEFAULT) {
    SegMap m{pick_seg(nbands, ny, ctas_per_sm, t, shape), 0, 0, 0, 1, ny};
    if (shape != SEG_DEFAULT && t.tail_rows == 0) return m;
    // auto: about half the segment, again 4k - 2 rows (30 -> 14, 22 -> 10, 14 -> 6, 10 / 6 -> 2)
    const int tail = t.tail_rows == 0 ? ((m.seg / 2 + 2) / 4) * 4 - 2 : t.tail_rows;
    if (tail <= 0 || tail >= m.seg || t.seg > 0) return m;
    const int waves = t.tail_waves > 0 ? t.tail_waves : 1;
    const int64_t slots = (int64_t)sm_count() * ctas_per_sm;
    // tail rows: enough segments to fill `waves` waves of CTAs
    const int64_t tail_segs = (waves * slots + nbands - 1) / nbands;
    const int64_t tail_rows = tail_segs * tail;
    if (tail_rows >= ny / 2) return m;   // small grid: keep it uniform
    m.jt = (int)((ny - tail_rows) / m.seg);
    m.tail = tail;
    return m;
}

// The TMA kernel's launch geometry: bands of NW strips x row segments.
struct TmaPlan {
    int nbands, nseg;
    SegMap sm;
};
// the segment shape of an instantiation on a grid (row window) of `cells`
int seg_shape(bool f32, bool fast, int red, int64_t cells) {
    if (f32 && fast && red == 0 && cells >= (int64_t(3) << 25)) return SEG_HBM;
    if (f32 && fast && red == 0 && cells >= (int64_t(1) << 26)) return SEG_18;
    // (5000^2: uniform 14-row segments 224.6 -> 231.8 Gcell/s; 3584^2 and
    // below keep the default)
    if (f32 && fast && red == 0 && cells >= (int64_t(23) << 20)) return SEG_HBM;
    if (!f32 && cells > (int64_t(1) << 26)) return SEG_NOTAIL;
    if (f32 && !fast && cells >= (int64_t(23) << 20) && cells < (int64_t(1) << 27)) return SEG_FINE;
    if (f32 && !fast && red == 0 && cells < (int64_t(1) << 20)) return SEG_TINY;
    if (!f32 || red == 0) return SEG_DEFAULT;
    if (red == 2 && cells > (int64_t(1) << 26)) return SEG_LONG;   // exact too: 125.9 -> 127.6
    return (fast && cells <= (int64_t(1) << 22)) ? SEG_LEAN : SEG_DEFAULT;
}
TmaPlan plan_tma(int nx, int ny, int own, int nw, int ctas_per_sm, const fkc_sw_tune& t, int shape = SEG_DEFAULT) {
    TmaPlan p;
    const int nstrips = (nx + own - 1) / own;
    p.nbands = (nstrips + nw - 1) / nw;
    p.sm = pick_segmap(p.nbands, ny, ctas_per_sm, t, shape);
    const SegMap& m = p.sm;
    p.nseg = m.tail == 0 ? (ny + m.seg - 1) / m.seg : m.jt + (ny - m.jt * m.seg + m.tail - 1) / m.tail;
    return p;
}

// Row window [ybase, ybase + nyw) of the interior (nyw 0: all rows).
template <class T, bool FAST, int RED, int NW>
int launch_tma_t(const fkc_sw_step_args* a, cudaStream_t st, const CUtensorMap* m, int ybase, int nyw) {
    using G = tma::Geo<T>;
    using B = tma::Blk<T, NW>;
    auto kern = sw_step_tma<T, FAST, RED, NW>;
    static std::once_flag attr_once;   // per instantiation; thread-safe
    static cudaError_t attr_err = cudaSuccess;
    std::call_once(attr_once, [&] {
        attr_err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, B::SMEM_BYTES);
    });
    if (attr_err != cudaSuccess)
        return fail(FKC_ECUDA, "cudaFuncSetAttribute(max dynamic smem): %s", cudaGetErrorString(attr_err));
    const fkc_grid& g = a->grid;
    if (nyw <= 0) { ybase = 1; nyw = g.ny; }
    int shape = seg_shape(sizeof(T) == 4, FAST, RED, (int64_t)g.nx * nyw);
    if (shape == SEG_HBM || shape == SEG_FINE) {
        // inside a CUDA graph the 14-row segments lose 5 % against the
        // default (scripts/seg_probe.py: 16384^2 graph 250 vs 264, eager
        // 276 vs 268 Gcell/s): a captured launch keeps the default schedule
        cudaStreamCaptureStatus cst = cudaStreamCaptureStatusNone;
        if (cudaStreamIsCapturing(st, &cst) != cudaSuccess) {
            cudaGetLastError();               // (non-sticky) -- not this launch's error
            shape = SEG_DEFAULT;
        } else if (cst != cudaStreamCaptureStatusNone) {
            shape = SEG_DEFAULT;
        }
    }
    TmaPlan p = plan_tma(g.nx, nyw, G::OWN, NW, B::template ctas_per_sm<FAST, RED>(), a->tune, shape);
    p.sm.rev = seg_rev(a->tune);
    p.sm.ybase = ybase;
    dim3 grd(p.nbands, p.nseg);
    SegMap sm = p.sm;
    DtSrc dts{a->dt, (const unsigned long long*)a->dt_bound, a->cfl};
    // with the fused exchange only when the caller vouches that no neighbour
    // tile shares this GPU (FKC_SYNC_PDL)
    const bool pdl = !a->tune.no_pdl && (a->sync.counter == nullptr || (a->sync.flags & FKC_SYNC_PDL));
    launch_step(kern, grd, dim3(B::THREADS), B::SMEM_BYTES, st, pdl, m[0], m[1], m[2], g.nx,
                g.ny, g.pitch, sm, a->tune.no_alternate ? 0 : 1, (T*)a->oH, (T*)a->oU, (T*)a->oV, (T)a->dx, (T)a->dy, dts, (T)a->g,
                to_bcs(a->bc), to_red(a->red), to_peers(a), to_sync(a));
    return check_launch("sw_step_tma");
}

// Warps per CTA (B200 sweeps, profiles/r01/cta_warps.json): f32 fast
// without reductions 1 below 3*2^23 cells (2048^2: 186 vs 151 Gcell/s with
// 4), 4 above (16384^2: 269 vs 262 with 1); f32 fast with fused reductions 1
// (16384^2 diagnostics 244 -> 266, CFL 232 -> 252); f32 exact 1 below 2^26
// cells, 2 above (16384^2 153 vs 150); f64 1 (fast 16384^2 116 -> 131).
template <class T>
int pick_warps(const fkc_grid& g, bool fast, int red, const fkc_sw_tune& t) {
    if (t.warps) return t.warps;
    if (sizeof(T) == 8) return 1;
    const int64_t cells = (int64_t)g.nx * g.ny;
    // fast with fused reductions: 1-warp CTAs, 2-warp ones above 2^26 cells
    // (round 2, reduction atomics fire-and-forget: 16384^2 CFL 252.7 -> 257.1,
    // diagnostics 266.9 -> 268.0 Gcell/s; 8192^2 equal)
    if (fast) return red > 0 ? (cells > (1LL << 26) ? 2 : 1) : (cells < (3LL << 23) ? 1 : 4);
    return cells < (1LL << 26) ? 1 : 2;
}

template <class T, bool FAST, int RED>
int launch_tma_nw(const fkc_sw_step_args* a, cudaStream_t st, const CUtensorMap* m, int ybase, int nyw) {
    switch (pick_warps<T>(a->grid, FAST, RED, a->tune)) {
        case 1: return launch_tma_t<T, FAST, RED, 1>(a, st, m, ybase, nyw);
        case 2: return launch_tma_t<T, FAST, RED, 2>(a, st, m, ybase, nyw);
        default: return launch_tma_t<T, FAST, RED, 4>(a, st, m, ybase, nyw);
    }
}

template <class T>
int launch_tma_typed(const fkc_sw_step_args* a, cudaStream_t st, int ybase, int nyw) {
    CUtensorMap m[3];  // H, U, V
    const fkc_grid& g = a->grid;
    const void* ps[3] = {a->H, a->U, a->V};
    int rc;
    for (int f = 0; f < 3; ++f)
        if ((rc = get_map(ps[f], g.nx, g.ny, g.pitch, tma::Geo<T>::BOXW, (int)sizeof(T), &m[f]))) return rc;
    const bool fast = a->mode == FKC_MODE_FAST;
    // reduction level: 0 none, 1 mass / maxima / error word, 2 + CFL bound
    const RedPtrs rp = to_red(a->red);
    const int lvl = rp.cfl_min ? 2 : (any_red(rp) ? 1 : 0);
    if (fast) {
        if (lvl == 2) return launch_tma_nw<T, true, 2>(a, st, m, ybase, nyw);
        return lvl ? launch_tma_nw<T, true, 1>(a, st, m, ybase, nyw) : launch_tma_nw<T, true, 0>(a, st, m, ybase, nyw);
    }
    if (lvl == 2) return launch_tma_nw<T, false, 2>(a, st, m, ybase, nyw);
    return lvl ? launch_tma_nw<T, false, 1>(a, st, m, ybase, nyw) : launch_tma_nw<T, false, 0>(a, st, m, ybase, nyw);
}

int launch_tma(const fkc_sw_step_args* a, cudaStream_t st, int ybase = 1, int nyw = 0) {
    return a->grid.dtype == FKC_F32 ? launch_tma_typed<float>(a, st, ybase, nyw)
                                    : launch_tma_typed<double>(a, st, ybase, nyw);
}

// ---------------------------------------------------------------------------
// resident time loop (sw_resident.cuh): the whole loop of a small grid in one
// cluster launch
// ---------------------------------------------------------------------------
// AUTO picks the resident loop for time loops (eager or captured in a
// graph) of grids up to these sizes that fit one cluster's shared memory.
// B200 (profiles/r02/resident_sweep.json, us / step, resident vs the best
// per-step kernel replayed from a CUDA graph): f32 fast 64^2 1.16 vs 2.34,
// 128^2 1.92 vs 2.64, 224^2 2.64 vs 2.76, 256^2 4.29 vs 2.77 (three strips
// of 8 warps); f32 exact 128^2 3.16 vs 3.86, 224^2 4.71 vs 5.52, 256^2 6.37
// vs 5.45; f64 exact 160^2 5.40 vs 6.80; f64 fast 96^2 1.93 vs 2.84, 128^2
// 2.88 vs 2.88.  The SPEC run (CFL dt + diagnostics, eager): 128^2 3.29 vs
// 6.15 (fast), 4.86 vs 6.72 (exact).
#ifndef FKC_RESIDENT_MAX_CELLS_F32
#define FKC_RESIDENT_MAX_CELLS_F32 (224 * 224)
#endif
#ifndef FKC_RESIDENT_MAX_CELLS_F64_FAST
#define FKC_RESIDENT_MAX_CELLS_F64_FAST (112 * 112)
#endif
#ifndef FKC_RESIDENT_MAX_CELLS_F64_EXACT
#define FKC_RESIDENT_MAX_CELLS_F64_EXACT (160 * 160)
#endif

int smem_optin() {
    static int cached[64] = {0};
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 227 * 1024;
    if (cached[dev] == 0) {
        int v = 0;
        cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
        cached[dev] = v > 0 ? v : 227 * 1024;
    }
    return cached[dev];
}

// cluster size, warps and dynamic shared memory of the resident kernel for
// a grid (nb = 0: does not fit one cluster's shared memory)
struct ResPlan {
    int nb, groups, warps;
    size_t smem;
};
template <class T>
ResPlan plan_resident_t(const fkc_grid& g, bool fast) {
    const size_t budget = (size_t)smem_optin() - 1024;   // static shared memory of the kernel
    // as many CTAs (SMs) as the rows allow: a step's arithmetic is spread
    // over the whole cluster (the cluster barrier costs the same)
    const int nb = g.ny < RES_MAX_CLUSTER ? g.ny : RES_MAX_CLUSTER;
    const int R = (g.ny + nb - 1) / nb;
    const ResGeo<T> geo(g.nx, R);
    if (geo.bytes() > budget) return {0, 0, 0, 0};
    // row groups: ~FKC_RES_GROUP_ROWS_* rows per warp's sweep (2 halo rows of
    // overhead each), at most res_warps() warps per CTA
    const int grows = fast ? FKC_RES_GROUP_ROWS_FAST : FKC_RES_GROUP_ROWS_EXACT;
    int groups = (R + grows - 1) / grows;
    const int gmax = (fast ? res_warps<T, true>() : res_warps<T, false>()) / geo.ns;
    if (gmax < 1) return {0, 0, 0, 0};
    if (groups > gmax) groups = gmax;
    if (groups < 1) groups = 1;
    return {nb, groups, groups * geo.ns, geo.bytes()};
}
ResPlan plan_resident(const fkc_grid& g, bool fast) {
    return g.dtype == FKC_F32 ? plan_resident_t<float>(g, fast) : plan_resident_t<double>(g, fast);
}

template <class T, bool FAST, int RED>
int launch_resident_t(const fkc_sw_loop_args* L, const ResPlan& rp, cudaStream_t st) {
    auto kern = sw_resident<T, FAST, RED>;
    static std::once_flag once;
    static cudaError_t attr_err = cudaSuccess;
    std::call_once(once, [&] {
        attr_err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_optin() - 1024);
        if (attr_err == cudaSuccess) attr_err = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    });
    if (attr_err != cudaSuccess) return fail(FKC_ECUDA, "resident kernel attributes: %s", cudaGetErrorString(attr_err));
    const fkc_sw_step_args& s = L->step;
    ResArgs ra;
    ra.nx = s.grid.nx; ra.ny = s.grid.ny; ra.pitch = s.grid.pitch;
    const void* A[3] = {s.H, s.U, s.V};
    void* B[3] = {s.oH, s.oU, s.oV};
    const bool in_a = (L->first_step & 1) == 0;
    const bool out_b = ((L->first_step + L->steps - 1) & 1) == 0;
    for (int f = 0; f < 3; ++f) {
        ra.in[f] = in_a ? A[f] : B[f];
        ra.out[f] = out_b ? B[f] : (void*)A[f];
    }
    ra.dx = s.dx; ra.dy = s.dy; ra.g = s.g; ra.dt = s.dt; ra.cfl = s.cfl;
    ra.dt_from_slots = L->dt_from_slots; ra.want_cfl = L->slots && L->want_cfl;
    ra.bc = to_bcs(s.bc);
    ra.first = L->first_step; ra.steps = L->steps;
    ra.slots = (unsigned long long*)L->slots;
    ra.groups = rp.groups;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(rp.nb);
    cfg.blockDim = dim3(rp.warps * 32);
    cfg.dynamicSmemBytes = rp.smem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = rp.nb;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, ra);
    if (e != cudaSuccess) return fail(FKC_ECUDA, "sw_resident launch: %s", cudaGetErrorString(e));
    if (L->slots && L->host_slots) {
        e = cudaMemcpyAsync(L->host_slots + 5 * (L->first_step + 1), L->slots + 5 * (L->first_step + 1),
                            5 * sizeof(uint64_t) * (size_t)L->steps, cudaMemcpyDeviceToHost, st);
        if (e != cudaSuccess) return fail(FKC_ECUDA, "cudaMemcpyAsync (diagnostics rows): %s", cudaGetErrorString(e));
    }
    // row halos and corners of the final state (== apply_boundary of it, as the step kernels' fused epilogue)
    return fkc_sw_apply_boundary(&s.grid, ra.out[0], ra.out[1], ra.out[2], s.bc, st);
}

template <class T, bool FAST>
int launch_resident_red(const fkc_sw_loop_args* L, const ResPlan& rp, cudaStream_t st) {
    if (!L->slots) return launch_resident_t<T, FAST, 0>(L, rp, st);
    if (L->want_cfl || L->dt_from_slots) return launch_resident_t<T, FAST, 2>(L, rp, st);
    return launch_resident_t<T, FAST, 1>(L, rp, st);
}

// resident loop if asked for (variant RESIDENT) or, with AUTO, for small
// grids that fit: returns -1 when the loop should take the per-step path
int try_resident(const fkc_sw_loop_args* L, cudaStream_t st) {
    const fkc_sw_step_args& s = L->step;
    if (s.variant != FKC_VARIANT_RESIDENT && s.variant != FKC_VARIANT_AUTO) return -1;
    const bool forced = s.variant == FKC_VARIANT_RESIDENT;
    auto no = [&](const char* why) { return forced ? fail(FKC_EUSAGE, "resident variant: %s", why) : -1; };
    if (!valid_grid(&s.grid)) return no("invalid grid");
    const int64_t max_cells = s.grid.dtype == FKC_F32 ? FKC_RESIDENT_MAX_CELLS_F32
                              : (s.mode == FKC_MODE_FAST ? FKC_RESIDENT_MAX_CELLS_F64_FAST
                                                         : FKC_RESIDENT_MAX_CELLS_F64_EXACT);
    if (!forced && (int64_t)s.grid.nx * s.grid.ny > max_cells) return -1;
    for (int i = 0; i < 4; ++i)
        if (s.bc[i] != FKC_BC_REFLECTIVE && s.bc[i] != FKC_BC_PERIODIC) return no("reflective / periodic sides only");
    if (!valid_bc(s.bc)) return no("invalid boundary spec");
    if (s.mode != FKC_MODE_EXACT && s.mode != FKC_MODE_FAST) return no("invalid mode");
    if (s.red.mass || s.red.max_abs_u || s.red.max_abs_v || s.red.cfl_min || s.red.err || s.dt_bound)
        return no("per-call reductions / dt_bound: use slots");
    if (!s.H || !s.U || !s.V || !s.oH || !s.oU || !s.oV) return no("null field pointer");
    if (s.H == s.oH || s.U == s.oU || s.V == s.oV) return no("outputs alias inputs");
    if (!(s.dx > 0) || !(s.dy > 0)) return no("dx, dy must be > 0");
    const int cpl = s.grid.dtype == FKC_F32 ? 4 : 2;
    if (s.grid.nx % cpl != 0) return no("nx must be a multiple of 16 / element size (the row engines' lane vectors)");
    const ResPlan rp = plan_resident(s.grid, s.mode == FKC_MODE_FAST);
    if (!rp.nb) return no("state does not fit in one cluster's shared memory");
    const bool fast = s.mode == FKC_MODE_FAST;
    if (s.grid.dtype == FKC_F32)
        return fast ? launch_resident_red<float, true>(L, rp, st) : launch_resident_red<float, false>(L, rp, st);
    return fast ? launch_resident_red<double, true>(L, rp, st) : launch_resident_red<double, false>(L, rp, st);
}

// ---------------------------------------------------------------------------
// persistent TMA time loop (sw_loop_tma): mid-size grids, one cooperative
// launch for the whole loop
// ---------------------------------------------------------------------------
// Opt-in (variant LOOP); AUTO does not take it.  Measured on B200
// (profiles/r02/loop_sweep.json, fast mode, fixed dt): 512^2 10.1 vs 4.3,
// 1024^2 14.4 vs 9.9, 2048^2 38.5 vs 25.3 us / step against the per-step
// kernels replayed from a CUDA graph -- even with the neighbour waits
// compiled out (racy, timing only) a 1024^2 loop step takes 11.1 us: at
// these sizes a warp's 12-row sweep at 8 resident warps per SM is latency
// bound, and a per-step launch re-spreads the same work over 12-warp SMs
// with short segments; from 4096^2 up the long per-warp sweeps also lose
// DRAM efficiency (123 vs 73 us).  Kept as a correct, tested alternative
// schedule (and for the CFL run without a host launch per step).
// rows per warp segment of the persistent grid: every warp must be resident,
// so the (bands x segments) CTAs fit in SMs x CTAs-per-SM; among the 4k-2
// lengths (no wasted row in the last stage) the shortest that fits -- the
// most warps sharing each step
int loop_seg(int nbands, int ny, int64_t cap, const fkc_sw_tune& t) {
    if (t.seg > 0) return t.seg;
    for (int seg = 2; seg < ny + 4; seg += 4)
        if ((int64_t)nbands * ((ny + seg - 1) / seg) <= cap) return seg;
    return 0;
}

template <class T, bool FAST, int RED, int NW>
int launch_loop_t(const fkc_sw_loop_args* L, cudaStream_t st, bool forced) {
    using G = tma::Geo<T>;
    using B = tma::Blk<T, NW>;
    auto kern = sw_loop_tma<T, FAST, RED, NW>;
    static std::once_flag once;
    static cudaError_t attr_err = cudaSuccess;
    static int occ = 0;
    std::call_once(once, [&] {
        attr_err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, B::SMEM_BYTES);
        if (attr_err == cudaSuccess)
            attr_err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, B::THREADS, B::SMEM_BYTES);
    });
    if (attr_err != cudaSuccess) return fail(FKC_ECUDA, "loop kernel attributes: %s", cudaGetErrorString(attr_err));
    const fkc_sw_step_args& s = L->step;
    const fkc_grid& g = s.grid;
    const int nstrips = (g.nx + G::OWN - 1) / G::OWN;
    const int nbands = (nstrips + NW - 1) / NW;
    const int64_t cap = (int64_t)sm_count() * occ;
    const int seg = loop_seg(nbands, g.ny, cap, s.tune);
    const int nseg = seg > 0 ? (g.ny + seg - 1) / seg : 0;
    if (seg <= 0 || (int64_t)nbands * nseg > cap) {
        if (!forced) return -1;
        return fail(FKC_EUSAGE, "loop variant: %d x %d warps do not fit on the GPU at once (%lld CTAs)", nstrips,
                    nseg, (long long)cap);
    }
    CUtensorMap m[6];
    const void* ps[6] = {s.H, s.U, s.V, s.oH, s.oU, s.oV};
    for (int f = 0; f < 6; ++f)
        if (int rc = get_map(ps[f], g.nx, g.ny, g.pitch, G::BOXW, (int)sizeof(T), &m[f])) return rc;
    const size_t nflags = (size_t)nseg * nstrips + 33;
    uint32_t* ws = nullptr;
    cudaError_t e = cudaMallocAsync((void**)&ws, nflags * sizeof(uint32_t), st);
    if (e != cudaSuccess) return fail(FKC_ECUDA, "cudaMallocAsync (loop flags): %s", cudaGetErrorString(e));
    e = cudaMemsetAsync(ws, 0, nflags * sizeof(uint32_t), st);
    if (e != cudaSuccess) return fail(FKC_ECUDA, "cudaMemsetAsync (loop flags): %s", cudaGetErrorString(e));
    LoopBufs bufs{{(void*)s.H, (void*)s.U, (void*)s.V}, {s.oH, s.oU, s.oV}};
    LoopCtl ctl;
    ctl.first = L->first_step;
    ctl.steps = L->steps;
    ctl.slots = (unsigned long long*)L->slots;
    ctl.dt_from_slots = L->dt_from_slots;
    ctl.want_cfl = L->slots && L->want_cfl;
    ctl.flags = ws;
    ctl.bar = ws + (size_t)nseg * nstrips;
    ctl.nstrips = nstrips;
    ctl.per_lr = s.bc[0] == FKC_BC_PERIODIC;
    ctl.per_du = s.bc[2] == FKC_BC_PERIODIC;
    ctl.dt = s.dt;
    ctl.cfl = s.cfl;
    SegMap sm{seg, 0, 0, 0, 1, g.ny};
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(nbands, nseg);
    cfg.blockDim = dim3(B::THREADS);
    cfg.dynamicSmemBytes = B::SMEM_BYTES;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;   // every warp resident, or the launch fails
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    e = cudaLaunchKernelEx(&cfg, kern, m[0], m[1], m[2], m[3], m[4], m[5], g.nx, g.ny, g.pitch, sm,
                           s.tune.no_alternate ? 0 : 1, bufs, (T)s.dx, (T)s.dy, (T)s.g, to_bcs(s.bc), ctl);
    if (e != cudaSuccess) {
        cudaFreeAsync(ws, st);
        return fail(FKC_ECUDA, "sw_loop_tma launch: %s", cudaGetErrorString(e));
    }
    e = cudaFreeAsync(ws, st);
    if (e != cudaSuccess) return fail(FKC_ECUDA, "cudaFreeAsync (loop flags): %s", cudaGetErrorString(e));
    if (L->slots && L->host_slots) {
        e = cudaMemcpyAsync(L->host_slots + 5 * (L->first_step + 1), L->slots + 5 * (L->first_step + 1),
                            5 * sizeof(uint64_t) * (size_t)L->steps, cudaMemcpyDeviceToHost, st);
        if (e != cudaSuccess) return fail(FKC_ECUDA, "cudaMemcpyAsync (diagnostics rows): %s", cudaGetErrorString(e));
    }
    return FKC_OK;
}

template <class T, bool FAST, int RED>
int launch_loop_nw(const fkc_sw_loop_args* L, cudaStream_t st, bool forced) {
    if (L->step.tune.warps > 1) return fail(FKC_EUSAGE, "loop variant: one warp per CTA (tune.warps 0 or 1)");
    return launch_loop_t<T, FAST, RED, 1>(L, st, forced);
}

template <class T>
int launch_loop_typed(const fkc_sw_loop_args* L, cudaStream_t st, bool forced) {
    const bool fast = L->step.mode == FKC_MODE_FAST;
    const int lvl = L->slots ? (L->want_cfl ? 2 : 1) : 0;
    if (fast) {
        if (lvl == 2) return launch_loop_nw<T, true, 2>(L, st, forced);
        return lvl ? launch_loop_nw<T, true, 1>(L, st, forced) : launch_loop_nw<T, true, 0>(L, st, forced);
    }
    if (lvl == 2) return launch_loop_nw<T, false, 2>(L, st, forced);
    return lvl ? launch_loop_nw<T, false, 1>(L, st, forced) : launch_loop_nw<T, false, 0>(L, st, forced);
}

// persistent loop if asked for (variant LOOP) or, with AUTO, for mid-size
// grids: returns -1 when the loop should take another path
int try_loop(const fkc_sw_loop_args* L, cudaStream_t st) {
    const fkc_sw_step_args& s = L->step;
    if (s.variant != FKC_VARIANT_LOOP && s.variant != FKC_VARIANT_AUTO) return -1;
    const bool forced = s.variant == FKC_VARIANT_LOOP;
    auto no = [&](const char* why) { return forced ? fail(FKC_EUSAGE, "loop variant: %s", why) : -1; };
    if (!valid_grid(&s.grid)) return no("invalid grid");
    if (!forced) return -1;
    if (!valid_bc(s.bc)) return no("invalid boundary spec");
    if (s.mode != FKC_MODE_EXACT && s.mode != FKC_MODE_FAST) return no("invalid mode");
    if (s.red.mass || s.red.max_abs_u || s.red.max_abs_v || s.red.cfl_min || s.red.err || s.dt_bound)
        return no("per-call reductions / dt_bound: use slots");
    if (!s.H || !s.U || !s.V || !s.oH || !s.oU || !s.oV) return no("null field pointer");
    if (s.H == s.oH || s.U == s.oU || s.V == s.oV) return no("outputs alias inputs");
    if (!(s.dx > 0) || !(s.dy > 0)) return no("dx, dy must be > 0");
    if (int rc = valid_tune(s.tune)) return rc;
    if (!tma_eligible(&s)) return no("needs the TMA layout (nx, pitch multiples of 16 / element size, aligned fields)");
    return s.grid.dtype == FKC_F32 ? launch_loop_typed<float>(L, st, forced) : launch_loop_typed<double>(L, st, forced);
}

}  // namespace

// ===========================================================================
// C-ABI
// ===========================================================================
extern "C" {

const char* fkc_last_error(void) { return g_err.c_str(); }
int fkc_abi_version(void) { return FKC_ABI_VERSION; }

// The TMA kernel's schedule for a grid (no device work; CPU-testable):
// out[0..6] = warps per CTA, bands, row segments (grid.y), segment rows,
// tail segment rows (0 = uniform), first tail segment, CTAs per SM.
int fkc_tma_plan(const fkc_grid* g, int mode, int red_level, const fkc_sw_tune* tune, int* out) {
    if (!g || !out || g->nx <= 0 || g->ny <= 0 || (g->dtype != FKC_F32 && g->dtype != FKC_F64) ||
        (mode != FKC_MODE_EXACT && mode != FKC_MODE_FAST) || red_level < 0 || red_level > 2)
        return fail(FKC_EUSAGE, "fkc_tma_plan: bad arguments");
    const fkc_sw_tune t = tune ? *tune : fkc_sw_tune{};
    if (int rc = valid_tune(t)) return rc;
    const bool f32 = g->dtype == FKC_F32, fast = mode == FKC_MODE_FAST;
    const int nw = f32 ? pick_warps<float>(*g, fast, red_level, t) : pick_warps<double>(*g, fast, red_level, t);
    int wps;   // resident warps per SM of that instantiation
    if (f32) wps = fast ? (red_level ? tma::Geo<float>::warps_per_sm<true, 1>() : tma::Geo<float>::warps_per_sm<true, 0>())
                        : tma::Geo<float>::warps_per_sm<false, 0>();
    else wps = tma::Geo<double>::warps_per_sm<true, 0>();
    const int own = f32 ? tma::Geo<float>::OWN : tma::Geo<double>::OWN;
    const TmaPlan p = plan_tma(g->nx, g->ny, own, nw, wps / nw, t,
                               seg_shape(f32, fast, red_level, (int64_t)g->nx * g->ny));
    out[0] = nw; out[1] = p.nbands; out[2] = p.nseg; out[3] = p.sm.seg; out[4] = p.sm.tail; out[5] = p.sm.jt;
    out[6] = wps / nw;
    return FKC_OK;
}

int fkc_test_div_f64(const double* a, const double* b, double* q, double* qref, int64_t n, void* stream) {
    if (!a || !b || !q || !qref || n < 0) return fail(FKC_EUSAGE, "bad arguments");
    test_div64_kernel<<<148 * 8, 256, 0, (cudaStream_t)stream>>>(a, b, q, qref, n);
    return check_launch("test_div64_kernel");
}

int fkc_test_sqrt2_f32(const float* x, float* s, float* sref, int64_t n, void* stream) {
    if (!x || !s || !sref || n < 0 || (n & 1)) return fail(FKC_EUSAGE, "bad arguments (n must be even)");
    test_sqrt2_kernel<<<148 * 8, 256, 0, (cudaStream_t)stream>>>(x, s, sref, n);
    return check_launch("test_sqrt2_kernel");
}

int fkc_test_div_f32(const float* a, const float* b, float* q, float* qref, int64_t n, void* stream) {
    if (!a || !b || !q || !qref || n < 0) return fail(FKC_EUSAGE, "bad arguments");
    test_div_kernel<<<148 * 8, 256, 0, (cudaStream_t)stream>>>(a, b, q, qref, n);
    return check_launch("test_div_kernel");
}

int fkc_sw_step(const fkc_sw_step_args* a, void* stream) {
    if (!a) return fail(FKC_EUSAGE, "null args");
    if (!valid_grid(&a->grid)) return fail(FKC_EUSAGE, "invalid grid (nx=%d ny=%d pitch=%lld dtype=%d)",
                                           a ? a->grid.nx : 0, a ? a->grid.ny : 0,
                                           (long long)(a ? a->grid.pitch : 0), a ? a->grid.dtype : -1);
    if (!a->H || !a->U || !a->V || !a->oH || !a->oU || !a->oV) return fail(FKC_EUSAGE, "null field pointer");
    if (a->H == a->oH || a->U == a->oU || a->V == a->oV)
        return fail(FKC_EUSAGE, "outputs must not alias inputs (double buffering, PAPER.md:488-493)");
    if (!valid_bc(a->bc)) return fail(FKC_EUSAGE, "invalid boundary spec");
    if (a->mode != FKC_MODE_EXACT && a->mode != FKC_MODE_FAST) return fail(FKC_EUSAGE, "invalid mode");
    if (!(a->dx > 0) || !(a->dy > 0)) return fail(FKC_EUSAGE, "dx, dy must be > 0");
    if (int rc = valid_peers(a)) return rc;
    if (int rc = valid_tune(a->tune)) return rc;
    cudaStream_t st = (cudaStream_t)stream;
    int variant = a->variant;
    // AUTO: the TMA sweep for grids of >= 640 Ki cells; below that (L2-
    // resident, launch-bound) the generic kernel's one-thread-per-cell
    // parallelism wins -- B200 sweep (profiles/r01/variant_crossover.json):
    // 768^2 generic 85 / 43 vs TMA 43 (exact), 896^2 generic 92 / 45 vs TMA
    // 96 / 60, 1024^2 generic 98 / 46 vs TMA 112 / 71 Gcell/s (fast / exact)
    //
    // Round 2: the plain exact step takes the TMA kernel from 2^18 cells
    // (f32, with 2-row segments below 2^20, SEG_TINY: 512^2 34.9 -> 37.0,
    // 640^2 39.3 -> 45.6, 768^2 42.2 -> 53.5 Gcell/s) / 3*2^17 cells (f64:
    // 640^2 19.5 -> 33.7, 768^2 20.9 -> 35.8), graph replays.
    if (variant == FKC_VARIANT_AUTO) {
        const int64_t cells = (int64_t)a->grid.nx * a->grid.ny;
        const bool plain_exact = a->mode == FKC_MODE_EXACT && !any_red(to_red(a->red)) && a->dt_bound == nullptr;
        const int64_t exact_min = a->grid.dtype == FKC_F32 ? (int64_t(1) << 18) : (int64_t(3) << 17);
        variant = tma_eligible(a) && (cells >= (int64_t(5) << 17) || (plain_exact && cells >= exact_min))
                      ? FKC_VARIANT_TMA
                      : FKC_VARIANT_GENERIC;
    }
    if (variant == FKC_VARIANT_TMA) {
        if (!tma_eligible(a))
            return fail(FKC_EUSAGE, "TMA variant needs nx and pitch multiples of 16/elem_size and (ptr+1 elem) "
                                    "16-B aligned (fields and row peer lines)");
        return launch_tma(a, st);
    }
    if (variant == FKC_VARIANT_RESIDENT || variant == FKC_VARIANT_LOOP)
        return fail(FKC_EUSAGE, "the resident / loop variants run whole time loops (fkc_sw_advance_n)");
    if (variant != FKC_VARIANT_GENERIC) return fail(FKC_EUSAGE, "invalid variant");
    return a->grid.dtype == FKC_F32 ? launch_generic<float>(a, st) : launch_generic<double>(a, st);
}

// ---------------------------------------------------------------------------
// native time loop (+ cached CUDA graphs)
// ---------------------------------------------------------------------------
// row_words: the slot row stride (5 = the caller's layout; the chunk ring
// uses RING_ROW)
static int enqueue_loop(const fkc_sw_loop_args* L, cudaStream_t st, int row_words = 5) {
    fkc_sw_step_args a = L->step;
    const void* A[3] = {L->step.H, L->step.U, L->step.V};
    void* B[3] = {L->step.oH, L->step.oU, L->step.oV};
    for (int64_t k = 0; k < L->steps; ++k) {
        const int64_t i = L->first_step + k;
        const bool even = (i & 1) == 0;
        a.H = even ? A[0] : B[0]; a.U = even ? A[1] : B[1]; a.V = even ? A[2] : B[2];
        a.oH = even ? B[0] : (void*)A[0]; a.oU = even ? B[1] : (void*)A[1]; a.oV = even ? B[2] : (void*)A[2];
        if (L->slots) {
            uint64_t* in = L->slots + row_words * i;
            uint64_t* out = L->slots + row_words * (i + 1);
            a.red.mass = (double*)out;
            a.red.max_abs_u = out + 1;
            a.red.max_abs_v = out + 2;
            a.red.cfl_min = L->want_cfl ? out + 3 : nullptr;
            a.red.err = (uint32_t*)(out + 4);
            a.dt_bound = L->dt_from_slots ? in + 3 : nullptr;
        }
        a.tune.parity = (int32_t)(i & 1);
        if (int rc = fkc_sw_step(&a, st)) return rc;
        if (L->slots && L->host_slots) {
            cudaError_t e = cudaMemcpyAsync(L->host_slots + 5 * (i + 1), L->slots + 5 * (i + 1), 5 * sizeof(uint64_t),
                                            cudaMemcpyDeviceToHost, st);
            if (e != cudaSuccess) return fail(FKC_ECUDA, "cudaMemcpyAsync (diagnostics row): %s", cudaGetErrorString(e));
        }
    }
    return FKC_OK;
}

struct GraphEntry {
    std::vector<unsigned char> key;
    cudaGraphExec_t exec;
};
std::mutex g_graph_mu;
std::vector<GraphEntry> g_graphs;

// Chunked replay of an eager time loop (the SPEC run: per-step reductions,
// CFL dt from the device slots; or plain fixed-dt steps): the loop's
// launch-per-step host cost (~3-6 us, more than a small grid's step) goes
// away by replaying ONE captured graph of FKC_CHUNK_STEPS steps.  The graph
// is position independent: its steps reduce into a private ring of rows
// that a small kernel appends to the caller's slots at a device step
// counter, so every chunk of the run (and later runs on the same buffers)
// replays the same graph.
#ifndef FKC_CHUNK_STEPS
#define FKC_CHUNK_STEPS 32
#endif
#ifndef FKC_CHUNK_MAX_CELLS
#define FKC_CHUNK_MAX_CELLS (int64_t(1) << 24)   // above: the launch is noise, and eager launches take SEG_HBM
#endif
struct ChunkGraph {
    std::vector<unsigned char> key;
    cudaGraphExec_t exec;
    unsigned long long* ring;
    long long* counter;
};
std::mutex g_chunk_mu;
std::vector<ChunkGraph> g_chunks;

static int enqueue_loop(const fkc_sw_loop_args* L, cudaStream_t st, int row_words);

static int run_chunked(const fkc_sw_loop_args* L0, cudaStream_t st) {
    fkc_sw_loop_args L = *L0;
    const int K = FKC_CHUNK_STEPS;
    if (L.first_step & 1) {                 // chunks start on an even step (A -> B)
        fkc_sw_loop_args one = L;
        one.steps = 1;
        if (int rc = enqueue_loop(&one, st)) return rc;
        L.first_step += 1;
        L.steps -= 1;
    }
    const int64_t nchunks = L.steps / K, rem = L.steps % K;
    if (nchunks > 0) {
        // key: the argument block with the position fields cleared
        fkc_sw_loop_args kb = L;
        kb.first_step = 0;
        kb.steps = 0;
        kb.host_slots = nullptr;
        std::vector<unsigned char> key((const unsigned char*)&kb, (const unsigned char*)&kb + sizeof(kb));
        std::lock_guard<std::mutex> lk(g_chunk_mu);
        ChunkGraph* cg = nullptr;
        for (auto& e : g_chunks)
            if (e.key == key) cg = &e;
        if (!cg) {
            // with reduction slots: a ring of K+1 rows and the step counter
            ChunkGraph ng{key, nullptr, nullptr, nullptr};
            auto release = [&ng]() {
                if (ng.ring) cudaFree(ng.ring);
                if (ng.counter) cudaFree(ng.counter);
            };
            if (L.slots && (cudaMalloc((void**)&ng.ring, RING_ROW * sizeof(uint64_t) * (K + 1)) != cudaSuccess ||
                            cudaMalloc((void**)&ng.counter, sizeof(long long)) != cudaSuccess)) {
                release();
                return fail(FKC_ECUDA, "cudaMalloc (chunk ring)");
            }
            fkc_sw_loop_args lc = L;        // the chunk: K steps from an even step (into the ring)
            lc.first_step = 0;
            lc.steps = K;
            lc.slots = (uint64_t*)ng.ring;
            lc.host_slots = nullptr;
            // captured on a private stream (the caller's may be the legacy
            // default stream, which cannot capture); replayed on the caller's
            int dev = 0;
            cudaGetDevice(&dev);
            static cudaStream_t cap[64] = {};
            if (dev < 0 || dev >= 64) {
                release();
                return fail(FKC_EUSAGE, "device index %d", dev);
            }
            if (!cap[dev] && cudaStreamCreateWithFlags(&cap[dev], cudaStreamNonBlocking) != cudaSuccess) {
                release();
                return fail(FKC_ECUDA, "cudaStreamCreate (chunk capture)");
            }
            cudaStream_t cs = cap[dev];
            cudaError_t err = cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal);
            if (err != cudaSuccess) {
                release();
                return fail(FKC_ECUDA, "cudaStreamBeginCapture: %s", cudaGetErrorString(err));
            }
            if (L.slots) ring_reset_kernel<<<1, 64, 0, cs>>>(ng.ring, K);
            const int rc = enqueue_loop(&lc, cs, RING_ROW);
            if (L.slots) ring_append_kernel<<<1, 256, 0, cs>>>(ng.ring, K, (unsigned long long*)L.slots, ng.counter);
            cudaGraph_t graph = nullptr;
            err = cudaStreamEndCapture(cs, &graph);
            if (rc || err != cudaSuccess) {
                if (graph) cudaGraphDestroy(graph);
                release();
                return rc ? rc : fail(FKC_ECUDA, "cudaStreamEndCapture: %s", cudaGetErrorString(err));
            }
            err = cudaGraphInstantiate(&ng.exec, graph, 0);
            cudaGraphDestroy(graph);
            if (err != cudaSuccess) {
                release();
                return fail(FKC_ECUDA, "cudaGraphInstantiate: %s", cudaGetErrorString(err));
            }
            if (g_chunks.size() >= 8) {
                // the evicted graph may still run on another stream
                cudaDeviceSynchronize();
                cudaGraphExecDestroy(g_chunks.front().exec);
                if (g_chunks.front().ring) cudaFree(g_chunks.front().ring);
                if (g_chunks.front().counter) cudaFree(g_chunks.front().counter);
                g_chunks.erase(g_chunks.begin());
            }
            g_chunks.push_back(ng);
            cg = &g_chunks.back();
        }
        if (L.slots) {
            // the run's position: the input bound row and the step counter
            cudaMemcpyAsync(cg->ring, L.slots + 5 * L.first_step, 5 * sizeof(uint64_t), cudaMemcpyDeviceToDevice,
                            st);
            set_counter_kernel<<<1, 1, 0, st>>>(cg->counter, (long long)L.first_step);
        }
        for (int64_t c = 0; c < nchunks; ++c) {
            cudaError_t err = cudaGraphLaunch(cg->exec, st);
            if (err != cudaSuccess) return fail(FKC_ECUDA, "cudaGraphLaunch: %s", cudaGetErrorString(err));
            if (L.slots && L.host_slots) {  // the host follows the run chunk by chunk
                const int64_t r = L.first_step + 1 + c * K;
                cudaMemcpyAsync(L.host_slots + 5 * r, L.slots + 5 * r, 5 * sizeof(uint64_t) * K,
                                cudaMemcpyDeviceToHost, st);
            }
        }
    }
    if (rem > 0) {
        fkc_sw_loop_args tail = L;
        tail.first_step = L.first_step + nchunks * K;
        tail.steps = rem;
        return enqueue_loop(&tail, st);
    }
    return check_launch("chunked time loop");
}

int fkc_sw_advance_n(const fkc_sw_loop_args* L, void* stream) {
    if (!L) return fail(FKC_EUSAGE, "null args");
    if (L->steps < 0 || L->first_step < 0) return fail(FKC_EUSAGE, "steps and first_step must be >= 0");
    if (L->step.sync.counter || L->step.peer[0].p[0] || L->step.peer[1].p[0] || L->step.peer[2].p[0] ||
        L->step.peer[3].p[0])
        return fail(FKC_EUSAGE, "fkc_sw_advance_n: peer lines / sync are per-step (use fkc_sw_step)");
    if (L->dt_from_slots && !L->slots) return fail(FKC_EUSAGE, "dt_from_slots needs slots");
    if (L->steps == 0) return FKC_OK;
    cudaStream_t st = (cudaStream_t)stream;
    {
        const int rc = try_resident(L, st);
        if (rc >= 0) return rc;
    }
    {
        const int rc = try_loop(L, st);
        if (rc >= 0) return rc;
    }
    // eager loops (the SPEC run with per-step reductions, or plain fixed-dt
    // steps) on grids where the launch per step costs about as much as the
    // step: replay a chunk graph
    if (!L->use_graph && L->steps >= 4 * FKC_CHUNK_STEPS && !getenv("FKC_NO_CHUNK") &&
        (int64_t)L->step.grid.nx * L->step.grid.ny <= FKC_CHUNK_MAX_CELLS) {
        cudaStreamCaptureStatus cst = cudaStreamCaptureStatusNone;
        if (cudaStreamIsCapturing(st, &cst) == cudaSuccess && cst == cudaStreamCaptureStatusNone)
            return run_chunked(L, st);
    }
    if (!L->use_graph) return enqueue_loop(L, st);
    // graph path: key = the whole argument block (pointers, dt, steps, parity...)
    std::vector<unsigned char> key((const unsigned char*)L, (const unsigned char*)L + sizeof(*L));
    std::lock_guard<std::mutex> lk(g_graph_mu);
    for (auto& e : g_graphs)
        if (e.key == key) {
            cudaError_t err = cudaGraphLaunch(e.exec, st);
            if (err != cudaSuccess) return fail(FKC_ECUDA, "cudaGraphLaunch: %s", cudaGetErrorString(err));
            return FKC_OK;
        }
    cudaError_t err = cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
    if (err != cudaSuccess) return fail(FKC_ECUDA, "cudaStreamBeginCapture: %s", cudaGetErrorString(err));
    const int rc = enqueue_loop(L, st);
    cudaGraph_t graph = nullptr;
    err = cudaStreamEndCapture(st, &graph);
    if (rc) {
        if (graph) cudaGraphDestroy(graph);
        return rc;
    }
    if (err != cudaSuccess) return fail(FKC_ECUDA, "cudaStreamEndCapture: %s", cudaGetErrorString(err));
    cudaGraphExec_t exec = nullptr;
    err = cudaGraphInstantiate(&exec, graph, 0);
    cudaGraphDestroy(graph);
    if (err != cudaSuccess) return fail(FKC_ECUDA, "cudaGraphInstantiate: %s", cudaGetErrorString(err));
    if (g_graphs.size() >= 16) {
        cudaGraphExecDestroy(g_graphs.front().exec);
        g_graphs.erase(g_graphs.begin());
    }
    g_graphs.push_back({key, exec});
    err = cudaGraphLaunch(exec, st);
    if (err != cudaSuccess) return fail(FKC_ECUDA, "cudaGraphLaunch: %s", cudaGetErrorString(err));
    return FKC_OK;
}

extern "C++" {
// one wavefront launch (sw_wave_tma): tasks of one band and step each
template <class T, bool FAST, int RED, int NW>
int launch_wave_t(const fkc_sw_step_args* a, const WaveArgs& w, int band_rows, cudaStream_t st) {
    using G = tma::Geo<T>;
    using B = tma::Blk<T, NW>;
    auto kern = sw_wave_tma<T, FAST, RED, NW>;
    static std::once_flag once;
    static cudaError_t attr_err = cudaSuccess;
    std::call_once(once, [&] {
        attr_err = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, B::SMEM_BYTES);
    });
    if (attr_err != cudaSuccess) return fail(FKC_ECUDA, "wave kernel attributes: %s", cudaGetErrorString(attr_err));
    const fkc_grid& g = a->grid;
    CUtensorMap m[6];
    const void* ps[6] = {a->H, a->U, a->V, a->oH, a->oU, a->oV};
    for (int f = 0; f < 6; ++f)
        if (int rc = get_map(ps[f], g.nx, g.ny, g.pitch, G::BOXW, (int)sizeof(T), &m[f])) return rc;
    const int nstrips = (g.nx + G::OWN - 1) / G::OWN;
    const int nbands = (nstrips + NW - 1) / NW;
    dim3 grd(nbands, (band_rows + w.seg - 1) / w.seg, w.ntask);
    LoopBufs bufs{{(void*)a->H, (void*)a->U, (void*)a->V}, {a->oH, a->oU, a->oV}};
    launch_step(kern, grd, dim3(B::THREADS), B::SMEM_BYTES, st, !a->tune.no_pdl, m[0], m[1], m[2], m[3], m[4], m[5],
                g.nx, g.ny, g.pitch, a->tune.no_alternate ? 0 : 1, bufs, (T)a->dx, (T)a->dy, (T)a->dt, (T)a->g,
                to_bcs(a->bc), w);
    return check_launch("sw_wave_tma");
}

// the wave kernel's schedule: warps per CTA and rows per segment for a launch
// of ntask bands of band_rows rows (a grid of nx x ntask*band_rows cells)
template <class T>
void wave_plan(const fkc_sw_step_args* a, int band_rows, int ntask, bool fast, int red, int& nw, int& seg) {
    fkc_grid eq = a->grid;
    eq.ny = band_rows * ntask;
    nw = pick_warps<T>(eq, fast, red, a->tune);
    const int wps = sizeof(T) == 8 ? tma::Geo<T>::template warps_per_sm<true, 0>()
                                   : (fast ? tma::Geo<T>::template warps_per_sm<true, 0>()
                                           : tma::Geo<T>::template warps_per_sm<false, 0>());
    const int nstrips = (a->grid.nx + tma::Geo<T>::OWN - 1) / tma::Geo<T>::OWN;
    (void)nstrips; (void)wps;
    // a band splits into m = ceil(band / 30) segments of equal length, rounded
    // up to 4k - 2 rows (no wasted row in a segment's last stage): 64-row
    // bands take 22 + 22 + 20 instead of 30 + 30 + 4
    if (a->tune.seg > 0) {
        seg = a->tune.seg;
        return;
    }
    const int m = (band_rows + 29) / 30;
    const int even = (band_rows + m - 1) / m;
    seg = ((even + 2 + 3) / 4) * 4 - 2;
}

template <class T>
int launch_wave(const fkc_sw_step_args* a, const WaveArgs& w0, int band_rows, cudaStream_t st) {
    const bool fast = a->mode == FKC_MODE_FAST;
    const int red = w0.t[0].red_row ? 1 : 0;
    int nw, seg;
    wave_plan<T>(a, band_rows, w0.ntask, fast, red, nw, seg);
    WaveArgs w = w0;
    w.seg = seg;
#define WAVE_NW(F, R) \
    (nw == 1 ? launch_wave_t<T, F, R, 1>(a, w, band_rows, st) \
             : nw == 2 ? launch_wave_t<T, F, R, 2>(a, w, band_rows, st) : launch_wave_t<T, F, R, 4>(a, w, band_rows, st))
    if (fast) return red ? WAVE_NW(true, 1) : WAVE_NW(true, 0);
    return red ? WAVE_NW(false, 1) : WAVE_NW(false, 0);
#undef WAVE_NW
}

}  // extern "C++"

#ifndef FKC_STREAM_COPY_ROWS
#define FKC_STREAM_COPY_ROWS 512    // rows per host<->device copy of the streamed host run (256: 1.5 % slower)
#endif
// ---------------------------------------------------------------------------
// streamed host run (fkc_sw_run_host): upload, steps and download overlapped
// ---------------------------------------------------------------------------
int fkc_sw_reduce_state(const fkc_grid* g, const void* H, const void* U, const void* V, double dx, double dy,
                        double gravity, const fkc_sw_reduce* red, void* stream);
int fkc_region_cpy(int32_t dtype, const void* src, int32_t nx_full, int32_t ny_full, int64_t src_pitch,
                   const int32_t halo[4], void* dst, int64_t dst_pitch, void* stream);
namespace {
// step args of global step i (buffers by parity, reduction row i+1)
fkc_sw_step_args step_of(const fkc_sw_loop_args* L, int64_t i) {
    fkc_sw_step_args a = L->step;
    const bool even = (i & 1) == 0;
    a.H = even ? L->step.H : L->step.oH;
    a.U = even ? L->step.U : L->step.oU;
    a.V = even ? L->step.V : L->step.oV;
    a.oH = even ? L->step.oH : (void*)L->step.H;
    a.oU = even ? L->step.oU : (void*)L->step.U;
    a.oV = even ? L->step.oV : (void*)L->step.V;
    if (L->slots) {
        uint64_t* out = L->slots + 5 * (i + 1);
        a.red.mass = (double*)out;
        a.red.max_abs_u = out + 1;
        a.red.max_abs_v = out + 2;
        a.red.cfl_min = L->want_cfl ? out + 3 : nullptr;
        a.red.err = (uint32_t*)(out + 4);
    }
    a.dt_bound = nullptr;
    a.tune.parity = (int32_t)(i & 1);
    return a;
}

struct CopyStreams {
    cudaStream_t up = nullptr, down = nullptr, red = nullptr, pack = nullptr;
    std::vector<cudaEvent_t> ev;
    cudaEvent_t last = nullptr;      // end of the previous call (calls share the streams and the staging)
    char* stage = nullptr;           // staging slots, grow-only
    size_t stage_bytes = 0;
};
std::mutex g_cs_mu;
CopyStreams g_cs[64];

int copy_streams(CopyStreams** out, size_t nev) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return fail(FKC_ECUDA, "cudaGetDevice");
    CopyStreams& c = g_cs[dev];
    if (!c.up) {
        if (cudaStreamCreateWithFlags(&c.up, cudaStreamNonBlocking) != cudaSuccess ||
            cudaStreamCreateWithFlags(&c.down, cudaStreamNonBlocking) != cudaSuccess ||
            cudaStreamCreateWithFlags(&c.red, cudaStreamNonBlocking) != cudaSuccess ||
            cudaStreamCreateWithFlags(&c.pack, cudaStreamNonBlocking) != cudaSuccess)
            return fail(FKC_ECUDA, "cudaStreamCreate (copy streams)");
    }
    if (!c.last && cudaEventCreateWithFlags(&c.last, cudaEventDisableTiming) != cudaSuccess)
        return fail(FKC_ECUDA, "cudaEventCreate");
    while (c.ev.size() < nev) {
        cudaEvent_t e;
        // timing-enabled under FKC_STREAM_TRACE (the trace below reads them)
        const unsigned fl = getenv("FKC_STREAM_TRACE") ? cudaEventDefault : cudaEventDisableTiming;
        if (cudaEventCreateWithFlags(&e, fl) != cudaSuccess) return fail(FKC_ECUDA, "cudaEventCreate");
        c.ev.push_back(e);
    }
    *out = &c;
    return FKC_OK;
}
}  // namespace

int fkc_sw_run_host(const fkc_sw_loop_args* L, const void* const host_in[3], void* const host_out[3],
                    int64_t host_pitch_bytes, int32_t band_rows, void* stream) {
    if (!L || !host_in || !host_out) return fail(FKC_EUSAGE, "null args");
    const fkc_sw_step_args& s0 = L->step;
    const fkc_grid& g = s0.grid;
    if (!valid_grid(&g)) return fail(FKC_EUSAGE, "invalid grid");
    for (int f = 0; f < 3; ++f)
        if (!host_in[f] || !host_out[f]) return fail(FKC_EUSAGE, "null host field");
    const int es = g.dtype == FKC_F32 ? 4 : 8;
    if (host_pitch_bytes < (int64_t)(g.nx + 2) * es || host_pitch_bytes % es)
        return fail(FKC_EUSAGE, "host pitch below a full row or not a multiple of the element size");
    if (L->steps < 0 || L->first_step < 0 || band_rows < 0) return fail(FKC_EUSAGE, "negative steps / band_rows");
    if (L->dt_from_slots) return fail(FKC_EUSAGE, "fkc_sw_run_host: fixed dt only (a CFL dt needs every band of a step)");
    if (s0.bc[2] == FKC_BC_PERIODIC) return fail(FKC_EUSAGE, "fkc_sw_run_host: periodic rows wrap around the wavefront");
    if (s0.sync.counter || s0.peer[0].p[0] || s0.peer[1].p[0] || s0.peer[2].p[0] || s0.peer[3].p[0])
        return fail(FKC_EUSAGE, "fkc_sw_run_host: no peer lines");
    if (!tma_eligible(&s0)) return fail(FKC_EUSAGE, "fkc_sw_run_host: needs the TMA layout (nx, pitch, alignment)");
    cudaStream_t st = (cudaStream_t)stream;
    std::lock_guard<std::mutex> lk(g_cs_mu);     // the copy streams and events are per device, shared
    // bands of ~band_rows interior rows (auto: 512 bands, >= 16 rows): the
    // wavefront's lag is 2 bands per step, so thin bands shorten the head
    // (upload only) and the tail (download only); the copies move several
    // bands at once (B200, 16384^2 x 20 steps, profiles/r02/stream_timing.txt:
    // 32 / 64 / 128-row bands 88.6 / 89.8 / 95.7 ms, the copies alone 81 ms)
    // A run of at most 32 steps is one wavefront (upload and download):
    // 1024 bands halve its lag (16384^2 x 20 steps: 82.2 -> 81.2 ms); longer
    // runs keep 512 (their wavefront phases run faster on 32-row bands)
    const int nbands_auto = L->steps <= 32 ? 1024 : 512;
    int br = band_rows > 0 ? band_rows : (g.ny + nbands_auto - 1) / nbands_auto;
    if (br < 16) br = 16;
    if (br > g.ny) br = g.ny;
    const int nb = (g.ny + br - 1) / br;
    // copies move chunks of cb bands (~FKC_STREAM_COPY_ROWS rows): the copy
    // engines reach both directions' full rate only with large transfers
    int cb = FKC_STREAM_COPY_ROWS / br;
    if (cb < 1) cb = 1;
    if (cb > nb) cb = nb;
    const int nc = (nb + cb - 1) / cb;
    auto chunk_of = [&](int i) { return i / cb; };
    CopyStreams* cs = nullptr;
    if (int rc = copy_streams(&cs, (size_t)6 * nc + 3)) return rc;
    cudaEvent_t* ev_up = cs->ev.data();            // [nc]   chunk c in its upload staging slot
    cudaEvent_t* ev_rep = cs->ev.data() + nc;      // [nc]   chunk c unpacked into the field (slot free)
    cudaEvent_t* ev_done = cs->ev.data() + 2 * nc; // [nc]   chunk c final (its last step done)
    cudaEvent_t* ev_dl = cs->ev.data() + 3 * nc;   // [nc]   chunk c downloaded (slot free)
    cudaEvent_t* ev_red = cs->ev.data() + 4 * nc;  // [nc]   chunk c of the uploaded state reduced
    cudaEvent_t* ev_pk = cs->ev.data() + 5 * nc;   // [nc]   chunk c packed into its download slot
    cudaEvent_t ev_start = cs->ev[6 * nc], ev_end = cs->ev[6 * nc + 1], ev_rows = cs->ev[6 * nc + 2];
    const int64_t S = L->steps, f0 = L->first_step;
    const int64_t dpitch = g.pitch * es, row_b = (int64_t)(g.nx + 2) * es;
    const bool in_a = (f0 & 1) == 0, out_a = ((f0 + S) & 1) == 0;
    const void* A[3] = {s0.H, s0.U, s0.V};
    const void* Bf[3] = {s0.oH, s0.oU, s0.oV};
    // full rows of copy chunk c: [r_lo, r_hi] (the halo rows travel with the
    // first / last chunk)
    auto chunk = [&](int c, int& r_lo, int& r_hi) {
        r_lo = c == 0 ? 0 : 1 + c * cb * br;
        r_hi = c == nc - 1 ? g.ny + 1 : (c + 1) * cb * br;
    };
    auto band = [&](int i, int& lo, int& n) {
        lo = 1 + i * br;
        n = (i == nb - 1 ? g.ny : (i + 1) * br) - lo + 1;
    };
    cudaError_t e;
    // The copies are 1-D (the host rows of a chunk are one contiguous block):
    // PCIe runs both directions at full rate only for linear copies (B200:
    // 55 + 55 GB/s at once vs 74 GB/s in total for pitched 2-D ones).  A
    // chunk lands in a device staging slot with the host row pitch and is
    // unpacked into the padded field by a copy kernel (and the other way
    // round for downloads); NS slots per direction, reused behind events.
    constexpr int NS = 16;
    const int64_t hp_el = host_pitch_bytes / es;
    const int64_t slot_field = (int64_t)(cb * br + 2) * host_pitch_bytes;
    const int64_t slot_bytes = 3 * slot_field;
    // the previous call may still use the staging slots
    cudaStreamWaitEvent(st, cs->last, 0);
    if (cs->stage_bytes < (size_t)(2 * NS * slot_bytes)) {
        if (cs->stage) {
            cudaDeviceSynchronize();
            cudaFree(cs->stage);
            cs->stage = nullptr;
            cs->stage_bytes = 0;
        }
        e = cudaMalloc((void**)&cs->stage, (size_t)(2 * NS * slot_bytes));
        if (e != cudaSuccess) return fail(FKC_ECUDA, "cudaMalloc (staging, %lld bytes): %s",
                                          (long long)(2 * NS * slot_bytes), cudaGetErrorString(e));
        cs->stage_bytes = (size_t)(2 * NS * slot_bytes);
    }
    char* stage = cs->stage;
    char* stage_up = stage;
    char* stage_dn = stage + NS * slot_bytes;
    const int32_t no_halo[4] = {0, 0, 0, 0};
    auto host_block = [&](int r_lo, int r_hi) { return (int64_t)(r_hi - r_lo) * host_pitch_bytes + row_b; };
    // upload chunk i: H2D into slot i % NS (after the slot's previous chunk was
    // unpacked), then unpack it into the input buffer on the compute stream
    auto upload_ = [&](int i) -> int {
        int r_lo, r_hi;
        chunk(i, r_lo, r_hi);
        char* slot = stage_up + (int64_t)(i % NS) * slot_bytes;
        if (i >= NS) cudaStreamWaitEvent(cs->up, ev_rep[i - NS], 0);
        for (int f = 0; f < 3; ++f) {
            e = cudaMemcpyAsync(slot + f * slot_field, (const char*)host_in[f] + (int64_t)r_lo * host_pitch_bytes,
                                (size_t)host_block(r_lo, r_hi), cudaMemcpyHostToDevice, cs->up);
            if (e != cudaSuccess) return fail(FKC_ECUDA, "cudaMemcpyAsync (upload %d): %s", i, cudaGetErrorString(e));
        }
        cudaEventRecord(ev_up[i], cs->up);
        cudaStreamWaitEvent(st, ev_up[i], 0);
        for (int f = 0; f < 3; ++f) {
            char* dev = (char*)(in_a ? A[f] : Bf[f]) + (int64_t)r_lo * dpitch;
            if (int rc = fkc_region_cpy(g.dtype, slot + f * slot_field, g.nx + 2, r_hi - r_lo + 1, hp_el, no_halo, dev,
                                        g.pitch, st))
                return rc;
        }
        cudaEventRecord(ev_rep[i], st);
        return FKC_OK;
    };
    // download chunk i once its rows are final (compute-stream order): pack
    // into slot i % NS on the pack stream (after the slot's previous chunk
    // left), D2H on the download stream.  The compute stream never waits for
    // the downloads (a backlog would stall the last wavefront steps), and the
    // packs run ahead of the D2H copies (no bubble between them).  The rows
    // of a final chunk are only read from then on (later tasks write their
    // own bands).
    auto download_ = [&](int i) -> int {
        int r_lo, r_hi;
        chunk(i, r_lo, r_hi);
        char* slot = stage_dn + (int64_t)(i % NS) * slot_bytes;
        cudaEventRecord(ev_done[i], st);
        cudaStreamWaitEvent(cs->pack, ev_done[i], 0);
        if (i >= NS) cudaStreamWaitEvent(cs->pack, ev_dl[i - NS], 0);
        for (int f = 0; f < 3; ++f) {
            const char* dev = (const char*)(out_a ? A[f] : Bf[f]) + (int64_t)r_lo * dpitch;
            if (int rc = fkc_region_cpy(g.dtype, dev, g.nx + 2, r_hi - r_lo + 1, g.pitch, no_halo, slot + f * slot_field,
                                        hp_el, cs->pack))
                return rc;
        }
        cudaEventRecord(ev_pk[i], cs->pack);
        cudaStreamWaitEvent(cs->down, ev_pk[i], 0);
        for (int f = 0; f < 3; ++f) {
            char* dst = (char*)host_out[f] + (int64_t)r_lo * host_pitch_bytes;
            // rows padded beyond the row length: a pitched copy, so the
            // caller's padding is never written
            e = host_pitch_bytes == row_b
                    ? cudaMemcpyAsync(dst, slot + f * slot_field, (size_t)host_block(r_lo, r_hi),
                                      cudaMemcpyDeviceToHost, cs->down)
                    : cudaMemcpy2DAsync(dst, host_pitch_bytes, slot + f * slot_field, host_pitch_bytes, row_b,
                                        r_hi - r_lo + 1, cudaMemcpyDeviceToHost, cs->down);
            if (e != cudaSuccess) return fail(FKC_ECUDA, "device-to-host copy (chunk %d): %s", i, cudaGetErrorString(e));
        }
        cudaEventRecord(ev_dl[i], cs->down);
        return FKC_OK;
    };
    auto row_back = [&](int64_t sidx) -> int {
        if (!L->slots || !L->host_slots) return FKC_OK;
        const int64_t r = f0 + sidx + 1;
        e = cudaMemcpyAsync(L->host_slots + 5 * r, L->slots + 5 * r, 5 * sizeof(uint64_t), cudaMemcpyDeviceToHost, st);
        return e == cudaSuccess ? FKC_OK : fail(FKC_ECUDA, "cudaMemcpyAsync (diagnostics row): %s", cudaGetErrorString(e));
    };
    // diagnostics row of the uploaded state (row first_step), band by band as
    // the bands arrive, on a side stream (the step that overwrites band i of
    // the input buffer -- the run's second -- waits for it)
    auto reduce_initial = [&](int c) -> int {
        if (!L->slots) return FKC_OK;
        cudaStreamWaitEvent(cs->red, ev_rep[c], 0);
        const int lo = 1 + c * cb * br, hi = c == nc - 1 ? g.ny : (c + 1) * cb * br;
        fkc_grid sub = g;
        sub.ny = hi - lo + 1;
        const int64_t off = (int64_t)(lo - 1) * dpitch;
        fkc_sw_reduce red{};
        uint64_t* row = L->slots + 5 * f0;
        red.mass = (double*)row;
        red.max_abs_u = row + 1;
        red.max_abs_v = row + 2;
        red.cfl_min = row + 3;
        red.err = (uint32_t*)(row + 4);
        const char* base[3] = {(const char*)(in_a ? A[0] : Bf[0]), (const char*)(in_a ? A[1] : Bf[1]),
                               (const char*)(in_a ? A[2] : Bf[2])};
        if (int rc = fkc_sw_reduce_state(&sub, base[0] + off, base[1] + off, base[2] + off, s0.dx, s0.dy, s0.g, &red,
                                         cs->red))
            return rc;
        cudaEventRecord(ev_red[c], cs->red);
        return FKC_OK;
    };
    // the copy streams start after the caller's prior work
    cudaEventRecord(ev_start, st);
    cudaStreamWaitEvent(cs->up, ev_start, 0);
    cudaStreamWaitEvent(cs->down, ev_start, 0);
    cudaStreamWaitEvent(cs->red, ev_start, 0);
    cudaStreamWaitEvent(cs->pack, ev_start, 0);
    // Phases: (1) the first P steps band by band as a wavefront behind the
    // upload (step s of band i after step s-1 of bands i-1 .. i+1 -- which also
    // covers the double buffer's write-after-read -- and after the upload of
    // band i+1); (2) whole-grid steps;
    // (3) the last P steps as a wavefront, each band downloaded as soon as
    // its last step is done.  With S <= 2P there is no phase 2.
    const int64_t P = 32;
    const int64_t s1 = S < P ? S : P;                        // steps of phase 1
    const int64_t s3 = (S - s1) < P ? (S - s1) : P;          // steps of phase 3
    const int64_t s2 = S - s1 - s3;
    // Iteration t launches ONE wave kernel with the tasks (step sa+k, band
    // t-2k-lag), k = 0 .. : step s of band i follows step s-1 of bands
    // i-1 .. i+1 (earlier iterations) -- which also covers the double
    // buffer's write-after-read -- and the upload of band i+lag; tasks of
    // one launch are two bands apart, so none reads rows another writes.
    const bool trace = getenv("FKC_STREAM_TRACE") != nullptr;
    std::vector<cudaEvent_t> trace_ev;               // [launch start, launch end] pairs (trace mode)
    std::vector<double> trace_host;                  // host time of each traced launch's enqueue (ms)
    const auto host_t0 = std::chrono::steady_clock::now();
    fkc_sw_step_args a0 = s0;                       // H,U,V = buffer A, oH,oU,oV = buffer B
    a0.red = fkc_sw_reduce{};                       // per task (WaveTask::red_row)
    a0.dt_bound = nullptr;
    auto wavefront = [&](int64_t sa, int64_t sb, bool upload, bool download) -> int {
        const int lag = upload ? 1 : 0;
        const int64_t tmax = (int64_t)nb + 2 * (sb - sa) + 2;
        for (int64_t t = 0; t < tmax; ++t) {
            // the first step of band t-1 needs band t: its chunk arrives now
            if (upload && t < nb && t % cb == 0) {
                if (int rc = upload_((int)(t / cb))) return rc;
                if (int rc = reduce_initial((int)(t / cb))) return rc;
            }
            WaveArgs w{};
            for (int64_t sidx = sa; sidx < sb && w.ntask < WAVE_MAX_TASKS; ++sidx) {
                const int64_t i = t - 2 * (sidx - sa) - lag;
                if (i < 0 || i >= nb) continue;
                int lo, n;
                band((int)i, lo, n);
                const int64_t gi = f0 + sidx;
                WaveTask& tk = w.t[w.ntask];
                tk.odd = (int)(gi & 1);
                tk.ybase = lo;
                tk.nyw = n;
                tk.red_row = L->slots ? (unsigned long long*)(L->slots + 5 * (gi + 1)) : nullptr;
                ++w.ntask;
                if (sidx == 1 && L->slots) cudaStreamWaitEvent(st, ev_red[chunk_of((int)i)], 0);   // overwrites band i
            }
            if (w.ntask == 0) continue;
            if (trace) {
                cudaEvent_t e0;
                cudaEventCreate(&e0);
                cudaEventRecord(e0, st);
                trace_ev.push_back(e0);
                trace_host.push_back(
                    std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - host_t0).count());
            }
            const int rc = g.dtype == FKC_F32 ? launch_wave<float>(&a0, w, br, st) : launch_wave<double>(&a0, w, br, st);
            if (rc) return rc;
            if (trace) {
                cudaEvent_t e1;
                cudaEventCreate(&e1);
                cudaEventRecord(e1, st);
                trace_ev.push_back(e1);
            }
            // (the wavefront's diagnostics rows go back in one copy at its
            // end: a 40-byte D2H per step on the compute stream queued behind
            // the chunk downloads on the copy engine and stalled the steps --
            // 2 ms each in the last wavefront)
            if (download) {
                // the band whose last step ran in this launch: i = t - 2(sb-1-sa) - lag;
                // its chunk leaves once its last band is final
                const int64_t i = t - 2 * (sb - 1 - sa) - lag;
                if (i >= 0 && i < nb && (i == nb - 1 || (i + 1) % cb == 0))
                    if (int rc2 = download_(chunk_of((int)i))) return rc2;
            }
        }
        if (L->slots && L->host_slots && sb > sa) {
            // rows of steps sa .. sb-1, on the download stream after the last task
            cudaEventRecord(ev_rows, st);
            cudaStreamWaitEvent(cs->down, ev_rows, 0);
            const int64_t r = f0 + sa + 1;
            e = cudaMemcpyAsync(L->host_slots + 5 * r, L->slots + 5 * r, (size_t)(5 * sizeof(uint64_t) * (sb - sa)),
                                cudaMemcpyDeviceToHost, cs->down);
            if (e != cudaSuccess)
                return fail(FKC_ECUDA, "cudaMemcpyAsync (diagnostics rows): %s", cudaGetErrorString(e));
        }
        return FKC_OK;
    };
    if (S == 0) {
        for (int c = 0; c < nc; ++c) {
            if (int rc = upload_(c)) return rc;
            if (int rc = reduce_initial(c)) return rc;
            if (int rc = download_(c)) return rc;
        }
    } else {
        if (int rc = wavefront(0, s1, true, s2 == 0 && s3 == 0)) return rc;
        for (int64_t sidx = s1; sidx < s1 + s2; ++sidx) {
            fkc_sw_step_args a = step_of(L, f0 + sidx);
            if (int rc = launch_tma(&a, st)) return rc;
            if (int rc = row_back(sidx)) return rc;
        }
        if (s3 > 0)
            if (int rc = wavefront(s1 + s2, S, false, true)) return rc;
    }
    // the caller's stream continues after the last download and reduction
    cudaEventRecord(ev_end, cs->red);
    cudaStreamWaitEvent(st, ev_end, 0);
    cudaEventRecord(ev_end, cs->down);
    cudaStreamWaitEvent(st, ev_end, 0);
    cudaEventRecord(cs->last, st);
    if (getenv("FKC_STREAM_TRACE")) {
        // diagnostics: when each band's upload and last step completed (ms
        // after the start), and the end -- synchronises the device
        cudaEventSynchronize(ev_end);
        float te = 0.f;
        cudaEventElapsedTime(&te, ev_start, ev_end);
        fprintf(stderr, "fkc_sw_run_host trace: %d bands of %d rows, copies of %d bands, %lld steps, end %.3f ms\n", nb,
                br, cb, (long long)S, te);
        for (int c = 0; c < nc; c += (nc > 16 ? nc / 16 : 1)) {
            float tu = -1.f, td = -1.f, tl = -1.f;
            if (cudaEventQuery(ev_up[c]) == cudaSuccess) cudaEventElapsedTime(&tu, ev_start, ev_up[c]);
            if (S > 0 && cudaEventQuery(ev_done[c]) == cudaSuccess) cudaEventElapsedTime(&td, ev_start, ev_done[c]);
            if (cudaEventQuery(ev_dl[c]) == cudaSuccess) cudaEventElapsedTime(&tl, ev_start, ev_dl[c]);
            fprintf(stderr, "  chunk %4d: uploaded %8.3f ms, last step done %8.3f ms, downloaded %8.3f ms\n", c, tu,
                    td, tl);
        }
        cudaDeviceSynchronize();
        for (size_t k = 0; k + 1 < trace_ev.size(); k += 2) {
            if (k / 2 % 16 != 0 && k / 2 + 60 < trace_ev.size() / 2) continue;
            float a = 0.f, b = 0.f;
            cudaEventElapsedTime(&a, ev_start, trace_ev[k]);
            cudaEventElapsedTime(&b, trace_ev[k], trace_ev[k + 1]);
            fprintf(stderr, "  wave launch %4zu: starts %8.3f ms, runs %7.3f ms, enqueued %8.3f ms (host)\n", k / 2, a,
                    b, trace_host[k / 2]);
        }
        for (auto e : trace_ev) cudaEventDestroy(e);
    }
    return check_launch("fkc_sw_run_host");
}

int fkc_sw_apply_boundary(const fkc_grid* g, void* H, void* U, void* V, const int32_t bc[4], void* stream) {
    if (!valid_grid(g)) return fail(FKC_EUSAGE, "invalid grid");
    if (!H || !U || !V) return fail(FKC_EUSAGE, "null field pointer");
    if (!bc || !valid_bc(bc)) return fail(FKC_EUSAGE, "invalid boundary spec");
    cudaStream_t st = (cudaStream_t)stream;
    const int t = 256;
    for (int phase = 0; phase < 2; ++phase) {
        const int n = phase == 0 ? g->ny : g->nx + 2;
        if (g->dtype == FKC_F32)
            sw_bc_kernel<float><<<(n + t - 1) / t, t, 0, st>>>(g->nx, g->ny, g->pitch, (float*)H, (float*)U,
                                                               (float*)V, to_bcs(bc), phase);
        else
            sw_bc_kernel<double><<<(n + t - 1) / t, t, 0, st>>>(g->nx, g->ny, g->pitch, (double*)H, (double*)U,
                                                                (double*)V, to_bcs(bc), phase);
    }
    return check_launch("sw_bc_kernel");
}

int fkc_copy2d(void* dst, int64_t dst_pitch_bytes, const void* src, int64_t src_pitch_bytes,
               int64_t width_bytes, int64_t height, void* stream) {
    if (!dst || !src || width_bytes < 0 || height < 0 || dst_pitch_bytes < width_bytes ||
        src_pitch_bytes < width_bytes)
        return fail(FKC_EUSAGE, "bad 2-D copy arguments");
    cudaError_t e = cudaMemcpy2DAsync(dst, (size_t)dst_pitch_bytes, src, (size_t)src_pitch_bytes,
                                      (size_t)width_bytes, (size_t)height, cudaMemcpyDefault,
                                      (cudaStream_t)stream);
    if (e != cudaSuccess) return fail(FKC_ECUDA, "cudaMemcpy2DAsync: %s", cudaGetErrorString(e));
    return FKC_OK;
}

int fkc_sw_reduce_reset(const fkc_sw_reduce* red, void* stream) {
    if (!red) return fail(FKC_EUSAGE, "null reduce");
    reduce_reset_kernel<<<1, 32, 0, (cudaStream_t)stream>>>(to_red(*red));
    return check_launch("reduce_reset_kernel");
}

int fkc_sw_reduce_state(const fkc_grid* g, const void* H, const void* U, const void* V, double dx, double dy,
                        double gravity, const fkc_sw_reduce* red, void* stream) {
    if (!valid_grid(g)) return fail(FKC_EUSAGE, "invalid grid");
    if (!H || !U || !V || !red) return fail(FKC_EUSAGE, "null pointer");
    cudaStream_t st = (cudaStream_t)stream;
    const double dmin = dx < dy ? dx : dy;
    int blocks = (g->ny + 7) / 8;                 // 8 warps (rows in flight) per block
    if (blocks > 148 * 8) blocks = 148 * 8;
    if (g->dtype == FKC_F32)
        sw_reduce_kernel<float><<<blocks, 256, 0, st>>>(g->nx, g->ny, g->pitch, (const float*)H, (const float*)U,
                                                        (const float*)V, (float)gravity, (float)dmin, to_red(*red));
    else
        sw_reduce_kernel<double><<<blocks, 256, 0, st>>>(g->nx, g->ny, g->pitch, (const double*)H,
                                                         (const double*)U, (const double*)V, gravity, dmin,
                                                         to_red(*red));
    return check_launch("sw_reduce_kernel");
}

int fkc_region_cpy(int32_t dtype, const void* src, int32_t nx_full, int32_t ny_full, int64_t src_pitch,
                   const int32_t halo[4], void* dst, int64_t dst_pitch, void* stream) {
    if (!src || !dst || !halo) return fail(FKC_EUSAGE, "null pointer");
    for (int i = 0; i < 4; ++i)
        if (halo[i] < 0) return fail(FKC_EUSAGE, "halo components must be >= 0");
    const int mx = nx_full - halo[0] - halo[1], my = ny_full - halo[2] - halo[3];
    if (mx < 1 || my < 1) return fail(FKC_EDOMAIN, "HaloTooLarge: halo leaves no interior");
    if (src_pitch < nx_full || dst_pitch < mx) return fail(FKC_EUSAGE, "bad pitch");
    dim3 b(64, 4), gr((mx + 63) / 64, (my + 3) / 4);
    cudaStream_t st = (cudaStream_t)stream;
    if (dtype == FKC_F32)
        region_cpy_kernel<float><<<gr, b, 0, st>>>((const float*)src, src_pitch, halo[0], halo[2], mx, my,
                                                   (float*)dst, dst_pitch);
    else if (dtype == FKC_F64)
        region_cpy_kernel<double><<<gr, b, 0, st>>>((const double*)src, src_pitch, halo[0], halo[2], mx, my,
                                                    (double*)dst, dst_pitch);
    else
        return fail(FKC_EUSAGE, "bad dtype");
    return check_launch("region_cpy_kernel");
}

int fkc_cshift(int32_t dtype, const void* src, int32_t nx, int32_t ny, int64_t src_pitch, int32_t dim,
               int64_t offset, void* dst, int64_t dst_pitch, void* stream) {
    if (!src || !dst) return fail(FKC_EUSAGE, "null pointer");
    if (nx < 1 || ny < 1 || src_pitch < nx || dst_pitch < nx) return fail(FKC_EUSAGE, "bad extent");
    if (dim != 1 && dim != 2) return fail(FKC_EUSAGE, "dim must be 1 or 2");
    if (src == dst) return fail(FKC_EUSAGE, "cshift is out-of-place");
    dim3 b(64, 4), gr((nx + 63) / 64, (ny + 3) / 4);
    cudaStream_t st = (cudaStream_t)stream;
    if (dtype == FKC_F32)
        cshift_kernel<float><<<gr, b, 0, st>>>((const float*)src, src_pitch, nx, ny, dim, offset, (float*)dst,
                                               dst_pitch);
    else if (dtype == FKC_F64)
        cshift_kernel<double><<<gr, b, 0, st>>>((const double*)src, src_pitch, nx, ny, dim, offset, (double*)dst,
                                                dst_pitch);
    else
        return fail(FKC_EUSAGE, "bad dtype");
    return check_launch("cshift_kernel");
}

static int halo_common(const fkc_grid* g, int side, bool unpack, const void* H, const void* U, const void* V,
                       void* buf, void* oH, void* oU, void* oV, const void* ibuf, void* stream) {
    if (!valid_grid(g)) return fail(FKC_EUSAGE, "invalid grid");
    if (side < 0 || side > 3) return fail(FKC_EUSAGE, "side must be 0..3");
    const int len = side < 2 ? g->ny : g->nx;
    const int t = 256;
    cudaStream_t st = (cudaStream_t)stream;
    if (g->dtype == FKC_F32)
        halo_pack_kernel<float><<<(len + t - 1) / t, t, 0, st>>>(g->nx, g->ny, g->pitch, (const float*)H,
                                                                 (const float*)U, (const float*)V, side, (float*)buf,
                                                                 unpack, (float*)oH, (float*)oU, (float*)oV,
                                                                 (const float*)ibuf);
    else
        halo_pack_kernel<double><<<(len + t - 1) / t, t, 0, st>>>(g->nx, g->ny, g->pitch, (const double*)H,
                                                                  (const double*)U, (const double*)V, side,
                                                                  (double*)buf, unpack, (double*)oH, (double*)oU,
                                                                  (double*)oV, (const double*)ibuf);
    return check_launch("halo_pack_kernel");
}

int fkc_halo_pack(const fkc_grid* g, const void* H, const void* U, const void* V, int32_t side, void* buf,
                  void* stream) {
    if (!H || !U || !V || !buf) return fail(FKC_EUSAGE, "null pointer");
    return halo_common(g, side, false, H, U, V, buf, nullptr, nullptr, nullptr, nullptr, stream);
}

int fkc_ipc_export(const void* ptr, uint8_t handle[64], int64_t* offset) {
    if (!ptr || !handle || !offset) return fail(FKC_EUSAGE, "null pointer");
    typedef CUresult (*RangeFn)(CUdeviceptr*, size_t*, CUdeviceptr);
    static RangeFn range = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            range = (RangeFn)p;
    });
    if (!range) return fail(FKC_ECUDA, "cuMemGetAddressRange unavailable");
    CUdeviceptr base = 0;
    size_t size = 0;
    if (range(&base, &size, (CUdeviceptr)ptr) != CUDA_SUCCESS) return fail(FKC_EUSAGE, "not a device allocation");
    cudaIpcMemHandle_t h;
    cudaError_t e = cudaIpcGetMemHandle(&h, (void*)base);
    if (e != cudaSuccess) return fail(FKC_ECUDA, "cudaIpcGetMemHandle: %s", cudaGetErrorString(e));
    static_assert(sizeof(h) == 64, "cudaIpcMemHandle_t is 64 bytes");
    memcpy(handle, &h, 64);
    *offset = (int64_t)((CUdeviceptr)ptr - base);
    return FKC_OK;
}

int fkc_ipc_open(const uint8_t handle[64], void** base) {
    if (!handle || !base) return fail(FKC_EUSAGE, "null pointer");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, 64);
    cudaError_t e = cudaIpcOpenMemHandle(base, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return fail(FKC_ECUDA, "cudaIpcOpenMemHandle: %s", cudaGetErrorString(e));
    return FKC_OK;
}

int fkc_ipc_close(void* base) {
    if (!base) return fail(FKC_EUSAGE, "null pointer");
    cudaError_t e = cudaIpcCloseMemHandle(base);
    if (e != cudaSuccess) return fail(FKC_ECUDA, "cudaIpcCloseMemHandle: %s", cudaGetErrorString(e));
    return FKC_OK;
}

int fkc_halo_unpack(const fkc_grid* g, void* H, void* U, void* V, int32_t side, const void* buf, void* stream) {
    if (!H || !U || !V || !buf) return fail(FKC_EUSAGE, "null pointer");
    return halo_common(g, side, true, nullptr, nullptr, nullptr, nullptr, H, U, V, buf, stream);
}

}  // extern "C"
