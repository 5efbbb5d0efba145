// sw_pair.cuh -- row engines of the TMA kernel.
//
// An engine holds the register window of the y-sweep (the previous row's
// cell quantities, its x-face fluxes, the y-face below it) and offers
//   row<DM>(h, u, v, have_prev, want_x, c, ok)  -- faces of a freshly loaded row
//   update<DM>(c, oh, ou, ov)                    -- full step of the previous row
//   shift()                                      -- the new row becomes the previous one
//
// ScalarEngine: one scalar op per cell (any T; exact mode's bit-exact order).
// PairEngine  : f32 fast mode on sm_100a's packed FP32 pipe.  A lane's four
//   cells c0..c3 form the register pairs P0 = (c0, c1), P1 = (c2, c3) (as
//   ld.shared.v4 delivers them) and every cell-wise or column-aligned
//   operation -- the cell quantities, the y-faces between two rows, the
//   full-step update -- is one FADD2 / FMUL2 / FFMA2 per pair, i.e. half the
//   issue slots.  The x-faces pair cells that straddle the pairs (c1|c2,
//   c3|lane+1), so they stay scalar and are stored directly as the per-cell
//   differences F_left - F_right the update consumes.
#pragma once
#include "sw_kernels.cuh"

namespace fkc {

// one lane's 16-byte vector of a row: 4 floats or 2 doubles
template <class T> struct VecF {
    T v[16 / sizeof(T)];
};

template <class T, int CPL> struct ScalarEngine {
    CellQ<T> pc[CPL];                  // previous row's cells
    FaceF<T> pxl, pxr[CPL];            // previous row's x-face fluxes
    FaceF<T> ydn[CPL];                 // y-face below the previous row
    CellQ<T> nc[CPL];                  // new row
    FaceF<T> yup[CPL], nxl, nxr[CPL];

    // benign window (a lake at rest) so a branch-free first row computes
    // finite, discarded faces
    __device__ __forceinline__ void init(const Coef<T>&) {
#pragma unroll
        for (int i = 0; i < CPL; ++i) {
            pc[i] = CellQ<T>{T(1), T(0), T(0), T(0), T(0), T(0)};
            ydn[i] = pxr[i] = FaceF<T>{T(0), T(0), T(0), T(1)};
        }
        pxl = FaceF<T>{T(0), T(0), T(0), T(1)};
    }

    template <int DM>
    __device__ __forceinline__ void row(const VecF<T>& h, const VecF<T>& u, const VecF<T>& v, bool have_prev,
                                        bool want_x, const Coef<T>& c, bool& ok) {
#pragma unroll
        for (int i = 0; i < CPL; ++i) nc[i] = cell_q<T, DM>(h.v[i], u.v[i], v.v[i], c, ok);
        if (have_prev) {
#pragma unroll
            for (int i = 0; i < CPL; ++i) yup[i] = y_face<T, DM>(pc[i], nc[i], c, ok);
        }
        if (want_x) {
            CellQ<T> nb;  // first cell of lane+1
            nb.h = __shfl_down_sync(0xffffffffu, nc[0].h, 1);
            nb.u = __shfl_down_sync(0xffffffffu, nc[0].u, 1);
            nb.v = __shfl_down_sync(0xffffffffu, nc[0].v, 1);
            nb.fu = __shfl_down_sync(0xffffffffu, nc[0].fu, 1);
            nb.cr = __shfl_down_sync(0xffffffffu, nc[0].cr, 1);
            nb.fv = T(0);
#pragma unroll
            for (int i = 0; i < CPL - 1; ++i) nxr[i] = x_face<T, DM>(nc[i], nc[i + 1], c, ok);
            nxr[CPL - 1] = x_face<T, DM>(nc[CPL - 1], nb, c, ok);
            nxl.fh = __shfl_up_sync(0xffffffffu, nxr[CPL - 1].fh, 1);
            nxl.fu = __shfl_up_sync(0xffffffffu, nxr[CPL - 1].fu, 1);
            nxl.fv = __shfl_up_sync(0xffffffffu, nxr[CPL - 1].fv, 1);
        }
    }
    template <int DM>
    __device__ __forceinline__ void update(const Coef<T>& c, T (&oh)[CPL], T (&ou)[CPL], T (&ov)[CPL]) const {
#pragma unroll
        for (int i = 0; i < CPL; ++i)
            update_cell<T, DM>(pc[i].h, pc[i].u, pc[i].v, i == 0 ? pxl : pxr[i - 1], pxr[i], ydn[i], yup[i], c,
                               oh[i], ou[i], ov[i]);
    }
    __device__ __forceinline__ void shift() {
#pragma unroll
        for (int i = 0; i < CPL; ++i) { pc[i] = nc[i]; ydn[i] = yup[i]; pxr[i] = nxr[i]; }
        pxl = nxl;
    }
    // min face depth of the row just computed (fused NonPositiveDepth check):
    // xall = every x-face right of this lane's cells, xlast = only the last
    // one (ghost lane 0: the face left of lane 1), y = the y-faces below them
    __device__ __forceinline__ void track(T& m, bool xall, bool xlast, bool y) const {
        const T inf = T(INFINITY);
#pragma unroll
        for (int i = 0; i < CPL; ++i) {
            m = fmin(m, (xall || (xlast && i == CPL - 1)) ? nxr[i].hd : inf);
            m = fmin(m, y ? yup[i].hd : inf);
        }
    }
};

// ---------------------------------------------------------------------------
// packed-pair arithmetic (fast mode: contraction into FFMA2 is intended)
// ---------------------------------------------------------------------------
__device__ __forceinline__ float2 bc2(float a) { return make_float2(a, a); }
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 sub2(float2 a, float2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 rcp2(float2 a) { return make_float2(rcp_approx(a.x), rcp_approx(a.y)); }

struct CellQ2 {
    float2 h, u, v, fu, fv, cr;
    __device__ __forceinline__ CellQ<float> lo() const { return {h.x, u.x, v.x, fu.x, fv.x, cr.x}; }
    __device__ __forceinline__ CellQ<float> hi() const { return {h.y, u.y, v.y, fu.y, fv.y, cr.y}; }
};
struct FaceF2 {
    float2 fh, fu, fv, hd;   // hd: face depths (see FaceF)
};
struct Coef2 {
    float2 half, cx2, cy2, cx, cy, g2;
    bool absorb;   // g/2 >= 1/4: tiny fxu quotients are absorbed (ExactPairEngine)
};

// fxu(h,u) = u*u/h + g2*h*h, fxu(h,v), cross = u*v/h with one reciprocal
__device__ __forceinline__ CellQ2 cell_q2(float2 h, float2 u, float2 v, const Coef2& c) {
    CellQ2 q;
    q.h = h; q.u = u; q.v = v;
    const float2 r = rcp2(h);
    const float2 uq = mul2(u, r), vq = mul2(v, r);
    const float2 gh2 = mul2(mul2(c.g2, h), h);
    q.fu = fma2(u, uq, gh2);
    q.fv = fma2(v, vq, gh2);
    q.cr = mul2(uq, v);
    return q;
}

// y-faces between row cells D (below) and U (above), statements Hy, Uy, Vy
__device__ __forceinline__ FaceF2 y_face2(const CellQ2& D, const CellQ2& U, const Coef2& c) {
    const float2 Hy = fma2(c.cy2, sub2(D.v, U.v), mul2(c.half, add2(D.h, U.h)));
    const float2 Uy = fma2(c.cy2, sub2(D.cr, U.cr), mul2(c.half, add2(D.u, U.u)));
    const float2 Vy = fma2(c.cy2, sub2(D.fv, U.fv), mul2(c.half, add2(D.v, U.v)));
    const float2 t = mul2(Vy, rcp2(Hy));
    FaceF2 f;
    f.fh = Vy;
    f.fu = mul2(Uy, t);
    f.fv = fma2(Vy, t, mul2(mul2(c.g2, Hy), Hy));
    f.hd = Hy;
    return f;
}

struct PairEngine {
    static constexpr int CPL = 4;
    CellQ2 pc[2];       // previous row: pairs (c0,c1), (c2,c3)
    FaceF2 pdx[2];      // previous row: F_left - F_right of its x-faces, per cell
    FaceF2 ydn[2];      // y-face below the previous row
    CellQ2 nc[2];
    FaceF2 ndx[2], yup[2];
    float2 nhx[2];      // depths of the new row's x-faces (f01, f12), (f23, f34) -- track() only
    Coef2 c2;

    __device__ __forceinline__ void init(const Coef<float>& c) {
        c2.half = bc2(c.half); c2.cx2 = bc2(c.cx2); c2.cy2 = bc2(c.cy2);
        c2.cx = bc2(c.cx); c2.cy = bc2(c.cy); c2.g2 = bc2(c.g2);
        c2.absorb = false;
        // benign window (a lake at rest): a branch-free first row computes
        // finite, discarded faces
        const float2 one = bc2(1.f), zero = bc2(0.f);
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            pc[j] = CellQ2{one, zero, zero, zero, zero, zero};
            pdx[j] = ydn[j] = FaceF2{zero, zero, zero, one};
        }
    }

    template <int DM>
    __device__ __forceinline__ void row(const VecF<float>& h, const VecF<float>& u, const VecF<float>& v,
                                        bool have_prev, bool want_x, const Coef<float>& c, bool& ok) {
        nc[0] = cell_q2(make_float2(h.v[0], h.v[1]), make_float2(u.v[0], u.v[1]), make_float2(v.v[0], v.v[1]), c2);
        nc[1] = cell_q2(make_float2(h.v[2], h.v[3]), make_float2(u.v[2], u.v[3]), make_float2(v.v[2], v.v[3]), c2);
        if (have_prev) {
            yup[0] = y_face2(pc[0], nc[0], c2);
            yup[1] = y_face2(pc[1], nc[1], c2);
        }
        if (want_x) {
            CellQ<float> nb;  // first cell of lane+1
            nb.h = __shfl_down_sync(0xffffffffu, nc[0].h.x, 1);
            nb.u = __shfl_down_sync(0xffffffffu, nc[0].u.x, 1);
            nb.v = __shfl_down_sync(0xffffffffu, nc[0].v.x, 1);
            nb.fu = __shfl_down_sync(0xffffffffu, nc[0].fu.x, 1);
            nb.cr = __shfl_down_sync(0xffffffffu, nc[0].cr.x, 1);
            nb.fv = 0.f;
            const FaceF<float> f01 = x_face<float, DIV_FAST>(nc[0].lo(), nc[0].hi(), c, ok);
            const FaceF<float> f12 = x_face<float, DIV_FAST>(nc[0].hi(), nc[1].lo(), c, ok);
            const FaceF<float> f23 = x_face<float, DIV_FAST>(nc[1].lo(), nc[1].hi(), c, ok);
            const FaceF<float> f34 = x_face<float, DIV_FAST>(nc[1].hi(), nb, c, ok);
            FaceF<float> fl;  // face left of c0 = lane-1's f34
            fl.fh = __shfl_up_sync(0xffffffffu, f34.fh, 1);
            fl.fu = __shfl_up_sync(0xffffffffu, f34.fu, 1);
            fl.fv = __shfl_up_sync(0xffffffffu, f34.fv, 1);
            ndx[0].fh = make_float2(fl.fh - f01.fh, f01.fh - f12.fh);
            ndx[0].fu = make_float2(fl.fu - f01.fu, f01.fu - f12.fu);
            ndx[0].fv = make_float2(fl.fv - f01.fv, f01.fv - f12.fv);
            ndx[1].fh = make_float2(f12.fh - f23.fh, f23.fh - f34.fh);
            ndx[1].fu = make_float2(f12.fu - f23.fu, f23.fu - f34.fu);
            ndx[1].fv = make_float2(f12.fv - f23.fv, f23.fv - f34.fv);
            nhx[0] = make_float2(f01.hd, f12.hd);
            nhx[1] = make_float2(f23.hd, f34.hd);
        }
    }
    __device__ __forceinline__ void track(float& m, bool xall, bool xlast, bool y) const {
        const float inf = INFINITY;
        m = fminf(m, xall ? fminf(fminf(nhx[0].x, nhx[0].y), nhx[1].x) : inf);
        m = fminf(m, (xall || xlast) ? nhx[1].y : inf);
        m = fminf(m, y ? fminf(fminf(yup[0].hd.x, yup[0].hd.y), fminf(yup[1].hd.x, yup[1].hd.y)) : inf);
    }
    // q' = (q + cx*(F_left - F_right)) + cy*(G_down - G_up)
    template <int DM>
    __device__ __forceinline__ void update(const Coef<float>&, float (&oh)[4], float (&ou)[4], float (&ov)[4]) const {
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const float2 h = fma2(c2.cy, sub2(ydn[j].fh, yup[j].fh), fma2(c2.cx, pdx[j].fh, pc[j].h));
            const float2 u = fma2(c2.cy, sub2(ydn[j].fu, yup[j].fu), fma2(c2.cx, pdx[j].fu, pc[j].u));
            const float2 v = fma2(c2.cy, sub2(ydn[j].fv, yup[j].fv), fma2(c2.cx, pdx[j].fv, pc[j].v));
            oh[2 * j] = h.x; oh[2 * j + 1] = h.y;
            ou[2 * j] = u.x; ou[2 * j + 1] = u.y;
            ov[2 * j] = v.x; ov[2 * j + 1] = v.y;
        }
    }
    __device__ __forceinline__ void shift() {
#pragma unroll
        for (int j = 0; j < 2; ++j) { pc[j] = nc[j]; ydn[j] = yup[j]; pdx[j] = ndx[j]; }
    }
};

// ---------------------------------------------------------------------------
// ExactPairEngine: f32 exact mode with the MULTIPLIES (and the FMAs of the
// exact division) on the packed pipe.  The additions stay scalar __fadd_rn:
// ptxas 12.9 contracts an f32x2 multiply feeding an f32x2 add into FFMA2 even
// with explicit .rn and -fmad=false, which would break the node-by-node
// order; an FMUL2 feeding scalar adds is left alone.  Every node is still
// one IEEE RN operation in the wave_advance.fk order (sw_math.cuh cell_q /
// y_face / update_cell), so the results are bit-identical (tested).
// ---------------------------------------------------------------------------
__device__ __forceinline__ float2 sadd2(float2 a, float2 b) {
    return make_float2(__fadd_rn(a.x, b.x), __fadd_rn(a.y, b.y));
}
__device__ __forceinline__ float2 ssub2(float2 a, float2 b) {
    return make_float2(__fsub_rn(a.x, b.x), __fsub_rn(a.y, b.y));
}
__device__ __forceinline__ float2 pmul2(float2 a, float2 b) { return __fmul2_rn(a, b); }

// RN(a / b) per element for the numerators over one denominator pair b, in
// two classes (sequences and fallbacks of sw_math.cuh div_group):
//  * af: fxu numerators (q^2, the quotient is added to g/2 h^2).  With
//    `absorb` (g/2 >= 1/4) a tiny |a| < 2^-100 needs no exactness: for
//    b >= 2^-24 the quotient is < 2^-76 while half an ulp of g/2 b^2 >=
//    2^-50 is >= 2^-74, so RN(q + g/2 b^2) = g/2 b^2 for the oracle's q and
//    ours alike -- the lean sequence suffices.
//  * ac: cross numerators (u v, added to values of their own magnitude).
//    Always scaled by 2^64 (exact), divided in the normal range and scaled
//    back (exact whenever the quotient is normal); so tiny-but-normal
//    quotients -- the far field of a wave -- need no fixup, and a subnormal
//    quotient is redone for that element alone in closed form
//    (fdiv_subnormal_rn).
// DIV_GUARD clears ok when an operand is outside that (b outside
// [2^-24, 2^24], |a| too large, inf / nan);
// DIV_FIXUP is the scalar never-failing path for such rows.
// RN(a / b) for a subnormal quotient, from the correctly rounded SCALED
// quotient qs = RN24(a 2^64 / b) (|qs| < 2^-62, qs != 0, b > 0 in range):
// T = |qs| 2^85 is exactly RN24(t) with t = |a| 2^149 / b < 2^23, so the
// closed form of sw_math.cuh fdiv_subnormal_rn applies without redoing the
// division -- RN_int(T) unless T is a half-integer, where the sign of the
// exact residual fma(-b, T, |a| 2^149) decides.
__device__ __forceinline__ float subnormal_from_scaled(float a, float b, float qs) {
    const float T = fabsf(qs) * 0x1p85f;
    const float fl = floorf(T);
    float k = rintf(T);
    if (T - fl == 0.5f) {
        const float e = __fmaf_rn(-b, T, (fabsf(a) * 0x1p100f) * 0x1p49f);
        k = e > 0.0f ? fl + 1.0f : (e < 0.0f ? fl : k);
    }
    return __uint_as_float((__float_as_uint(a) & 0x80000000u) | (uint32_t)k);
}

template <int DM, int NF, int NC>
__device__ __forceinline__ void div2(float2 b, const float2 (&af)[NF], const float2 (&ac)[NC], float2 (&qf)[NF],
                                     float2 (&qc)[NC], bool absorb, bool& ok) {
    if constexpr (DM == DIV_GUARD) {
        const float2 r0 = rcp2(b);
        const float2 r = __ffma2_rn(r0, __ffma2_rn(make_float2(-b.x, -b.y), r0, bc2(1.0f)), r0);
        const float2 nr = make_float2(-r.x, -r.y);
        bool g = (b.x >= 0x1p-24f) & (b.x <= 0x1p+24f) & (b.y >= 0x1p-24f) & (b.y <= 0x1p+24f);
#pragma unroll
        for (int i = 0; i < NF; ++i) {
            const float2 qi = pmul2(af[i], r);
            const float2 res = __ffma2_rn(b, qi, make_float2(-af[i].x, -af[i].y));
            qf[i] = __ffma2_rn(nr, res, qi);
            const float ax = fabsf(af[i].x), ay = fabsf(af[i].y);
            g = g & (ax <= 0x1p+100f) & (ay <= 0x1p+100f);
            if (!absorb)   // warp-uniform
                g = g & ((ax >= 0x1p-100f) | (af[i].x == 0.0f)) & ((ay >= 0x1p-100f) | (af[i].y == 0.0f));
        }
#pragma unroll
        for (int i = 0; i < NC; ++i) {
            const float2 as = pmul2(ac[i], bc2(0x1p64f));
            const float2 qi = pmul2(as, r);
            const float2 res = __ffma2_rn(b, qi, make_float2(-as.x, -as.y));
            const float2 qs = __ffma2_rn(nr, res, qi);
            qc[i] = pmul2(qs, bc2(0x1p-64f));
            // a subnormal quotient (|qs| < 2^-62): that element alone takes the
            // closed-form exact path (divergent, sparse) instead of failing the row
            const bool subx = (fabsf(qs.x) < 0x1p-62f) & (qs.x != 0.0f);
            const bool suby = (fabsf(qs.y) < 0x1p-62f) & (qs.y != 0.0f);
            if (subx | suby) {
                if (subx) qc[i].x = subnormal_from_scaled(ac[i].x, b.x, qs.x);
                if (suby) qc[i].y = subnormal_from_scaled(ac[i].y, b.y, qs.y);
            }
            g = g & (fabsf(ac[i].x) <= 0x1p+36f) & (fabsf(ac[i].y) <= 0x1p+36f);
        }
        ok = ok & g;
    } else {
#pragma unroll
        for (int i = 0; i < NF; ++i) {
            const float ax[1] = {af[i].x}, ay[1] = {af[i].y};
            float qx[1], qy[1];
            div_group<float, DM, 1>(b.x, ax, qx, ok);
            div_group<float, DM, 1>(b.y, ay, qy, ok);
            qf[i] = make_float2(qx[0], qy[0]);
        }
#pragma unroll
        for (int i = 0; i < NC; ++i) {
            const float ax[1] = {ac[i].x}, ay[1] = {ac[i].y};
            float qx[1], qy[1];
            div_group<float, DM, 1>(b.x, ax, qx, ok);
            div_group<float, DM, 1>(b.y, ay, qy, ok);
            qc[i] = make_float2(qx[0], qy[0]);
        }
    }
}

template <int DM>
__device__ __forceinline__ CellQ2 cell_q2_exact(float2 h, float2 u, float2 v, const Coef2& c, bool& ok) {
    CellQ2 q;
    q.h = h; q.u = u; q.v = v;
    const float2 nf[2] = {pmul2(u, u), pmul2(v, v)}, nc[1] = {pmul2(u, v)};
    float2 qf[2], qc[1];
    div2<DM, 2, 1>(h, nf, nc, qf, qc, c.absorb, ok);
    const float2 gh2 = pmul2(pmul2(c.g2, h), h);
    q.fu = sadd2(qf[0], gh2);
    q.fv = sadd2(qf[1], gh2);
    q.cr = qc[0];
    return q;
}

template <int DM>
__device__ __forceinline__ FaceF2 y_face2_exact(const CellQ2& D, const CellQ2& U, const Coef2& c, bool& ok) {
    const float2 Hy = sadd2(pmul2(c.half, sadd2(D.h, U.h)), pmul2(c.cy2, ssub2(D.v, U.v)));
    const float2 Uy = sadd2(pmul2(c.half, sadd2(D.u, U.u)), pmul2(c.cy2, ssub2(D.cr, U.cr)));
    const float2 Vy = sadd2(pmul2(c.half, sadd2(D.v, U.v)), pmul2(c.cy2, ssub2(D.fv, U.fv)));
    const float2 nf[1] = {pmul2(Vy, Vy)}, nc[1] = {pmul2(Uy, Vy)};
    float2 qf[1], qc[1];
    div2<DM, 1, 1>(Hy, nf, nc, qf, qc, c.absorb, ok);
    FaceF2 f;
    f.fh = Vy;
    f.fu = qc[0];
    f.fv = sadd2(qf[0], pmul2(pmul2(c.g2, Hy), Hy));
    f.hd = Hy;
    return f;
}

// x-faces between the cells of L and R (two faces at once; statements Hx,
// Ux, Vx).  The cell quantities only enter through scalar sums / differences,
// so the pairs L and R never have to exist as register pairs.
template <int DM>
__device__ __forceinline__ FaceF2 x_face2_exact(const CellQ2& L, const CellQ2& R, const Coef2& c, bool& ok) {
    const float2 Hx = sadd2(pmul2(c.half, sadd2(L.h, R.h)), pmul2(c.cx2, ssub2(L.u, R.u)));
    const float2 Ux = sadd2(pmul2(c.half, sadd2(L.u, R.u)), pmul2(c.cx2, ssub2(L.fu, R.fu)));
    const float2 Vx = sadd2(pmul2(c.half, sadd2(L.v, R.v)), pmul2(c.cx2, ssub2(L.cr, R.cr)));
    const float2 nf[1] = {pmul2(Ux, Ux)}, nc[1] = {pmul2(Ux, Vx)};
    float2 qf[1], qc[1];
    div2<DM, 1, 1>(Hx, nf, nc, qf, qc, c.absorb, ok);
    FaceF2 f;
    f.fh = Ux;
    f.fu = sadd2(qf[0], pmul2(pmul2(c.g2, Hx), Hx));
    f.fv = qc[0];
    f.hd = Hx;
    return f;
}

__device__ __forceinline__ CellQ2 cells2(const CellQ2& a, bool ahi, const CellQ2& b, bool bhi) {
    auto pick = [](float2 p, bool hi) { return hi ? p.y : p.x; };
    CellQ2 q;
    q.h = make_float2(pick(a.h, ahi), pick(b.h, bhi));
    q.u = make_float2(pick(a.u, ahi), pick(b.u, bhi));
    q.v = make_float2(pick(a.v, ahi), pick(b.v, bhi));
    q.fu = make_float2(pick(a.fu, ahi), pick(b.fu, bhi));
    q.fv = make_float2(pick(a.fv, ahi), pick(b.fv, bhi));
    q.cr = make_float2(pick(a.cr, ahi), pick(b.cr, bhi));
    return q;
}

struct ExactPairEngine {
    static constexpr int CPL = 4;
    CellQ2 pc[2];
    FaceF2 pdx[2], ydn[2];
    CellQ2 nc[2];
    FaceF2 ndx[2], yup[2];
    float2 nhx[2];      // depths of the new row's x-faces (f01, f23), (f12, f34) -- track() only
    Coef2 c2;

    __device__ __forceinline__ void init(const Coef<float>& c) {
        c2.half = bc2(c.half); c2.cx2 = bc2(c.cx2); c2.cy2 = bc2(c.cy2);
        c2.cx = bc2(c.cx); c2.cy = bc2(c.cy); c2.g2 = bc2(c.g2);
        c2.absorb = c.g2 >= 0.25f;
        const float2 one = bc2(1.f), zero = bc2(0.f);
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            pc[j] = CellQ2{one, zero, zero, zero, zero, zero};
            pdx[j] = ydn[j] = FaceF2{zero, zero, zero, one};
        }
    }

    template <int DM>
    __device__ __forceinline__ void row(const VecF<float>& h, const VecF<float>& u, const VecF<float>& v,
                                        bool have_prev, bool want_x, const Coef<float>& c, bool& ok) {
        nc[0] = cell_q2_exact<DM>(make_float2(h.v[0], h.v[1]), make_float2(u.v[0], u.v[1]),
                                  make_float2(v.v[0], v.v[1]), c2, ok);
        nc[1] = cell_q2_exact<DM>(make_float2(h.v[2], h.v[3]), make_float2(u.v[2], u.v[3]),
                                  make_float2(v.v[2], v.v[3]), c2, ok);
        if (have_prev) {
            yup[0] = y_face2_exact<DM>(pc[0], nc[0], c2, ok);
            yup[1] = y_face2_exact<DM>(pc[1], nc[1], c2, ok);
        }
        if (want_x) {
            CellQ<float> nb;  // first cell of lane+1
            nb.h = __shfl_down_sync(0xffffffffu, nc[0].h.x, 1);
            nb.u = __shfl_down_sync(0xffffffffu, nc[0].u.x, 1);
            nb.v = __shfl_down_sync(0xffffffffu, nc[0].v.x, 1);
            nb.fu = __shfl_down_sync(0xffffffffu, nc[0].fu.x, 1);
            nb.cr = __shfl_down_sync(0xffffffffu, nc[0].cr.x, 1);
            nb.fv = 0.f;
            CellQ2 nbq;
            nbq.h = bc2(nb.h); nbq.u = bc2(nb.u); nbq.v = bc2(nb.v); nbq.fu = bc2(nb.fu); nbq.fv = bc2(0.f);
            nbq.cr = bc2(nb.cr);
            // faces (f01, f23) = x_face((c0, c2), (c1, c3)); (f12, f34) = x_face((c1, c3), (c2, c4))
            const FaceF2 F0 = x_face2_exact<DM>(cells2(nc[0], false, nc[1], false), cells2(nc[0], true, nc[1], true),
                                                c2, ok);
            const FaceF2 F1 = x_face2_exact<DM>(cells2(nc[0], true, nc[1], true), cells2(nc[1], false, nbq, false),
                                                c2, ok);
            FaceF<float> fl;  // face left of c0 = lane-1's f34
            fl.fh = __shfl_up_sync(0xffffffffu, F1.fh.y, 1);
            fl.fu = __shfl_up_sync(0xffffffffu, F1.fu.y, 1);
            fl.fv = __shfl_up_sync(0xffffffffu, F1.fv.y, 1);
            ndx[0].fh = make_float2(__fsub_rn(fl.fh, F0.fh.x), __fsub_rn(F0.fh.x, F1.fh.x));
            ndx[0].fu = make_float2(__fsub_rn(fl.fu, F0.fu.x), __fsub_rn(F0.fu.x, F1.fu.x));
            ndx[0].fv = make_float2(__fsub_rn(fl.fv, F0.fv.x), __fsub_rn(F0.fv.x, F1.fv.x));
            ndx[1].fh = make_float2(__fsub_rn(F1.fh.x, F0.fh.y), __fsub_rn(F0.fh.y, F1.fh.y));
            ndx[1].fu = make_float2(__fsub_rn(F1.fu.x, F0.fu.y), __fsub_rn(F0.fu.y, F1.fu.y));
            ndx[1].fv = make_float2(__fsub_rn(F1.fv.x, F0.fv.y), __fsub_rn(F0.fv.y, F1.fv.y));
            nhx[0] = F0.hd;
            nhx[1] = F1.hd;
        }
    }
    __device__ __forceinline__ void track(float& m, bool xall, bool xlast, bool y) const {
        const float inf = INFINITY;
        m = fminf(m, xall ? fminf(fminf(nhx[0].x, nhx[0].y), nhx[1].x) : inf);
        m = fminf(m, (xall || xlast) ? nhx[1].y : inf);
        m = fminf(m, y ? fminf(fminf(yup[0].hd.x, yup[0].hd.y), fminf(yup[1].hd.x, yup[1].hd.y)) : inf);
    }
    // q' = (q + cx*(F_left - F_right)) + cy*(G_down - G_up), RN per node
    template <int DM>
    __device__ __forceinline__ void update(const Coef<float>&, float (&oh)[4], float (&ou)[4], float (&ov)[4]) const {
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const float2 h = sadd2(sadd2(pc[j].h, pmul2(c2.cx, pdx[j].fh)), pmul2(c2.cy, ssub2(ydn[j].fh, yup[j].fh)));
            const float2 u = sadd2(sadd2(pc[j].u, pmul2(c2.cx, pdx[j].fu)), pmul2(c2.cy, ssub2(ydn[j].fu, yup[j].fu)));
            const float2 v = sadd2(sadd2(pc[j].v, pmul2(c2.cx, pdx[j].fv)), pmul2(c2.cy, ssub2(ydn[j].fv, yup[j].fv)));
            oh[2 * j] = h.x; oh[2 * j + 1] = h.y;
            ou[2 * j] = u.x; ou[2 * j + 1] = u.y;
            ov[2 * j] = v.x; ov[2 * j + 1] = v.y;
        }
    }
    __device__ __forceinline__ void shift() {
#pragma unroll
        for (int j = 0; j < 2; ++j) { pc[j] = nc[j]; ydn[j] = yup[j]; pdx[j] = ndx[j]; }
    }
};

// ---------------------------------------------------------------------------
// ExactPairEngine2: f32 exact mode with EVERY operation on the packed FP32
// pipe (FADD2 / FFMA2 / FMUL2), range guards reduced per ROW, and the pairs
// laid out so the x-faces need few register moves.
//
//  * Contraction.  ptxas fuses an f32x2 multiply feeding an f32x2 add into
//    FFMA2 even with explicit .rn (which would round once instead of twice).
//    A product that feeds an add is therefore formed as FFMA2(a, b, nz) with
//    nz an opaque -0.0 (derived from a runtime parameter, so ptxas cannot
//    see it): RN(a*b + -0) == RN(a*b) for every a, b (a +0 product stays
//    +0), and an FMA feeding an add is not fusable.  So every parse-tree node
//    of wave_advance.fk is still exactly one IEEE RN operation.
//  * Guards.  The shared-reciprocal division (sw_math.cuh DIV_GUARD) is
//    exact for b in [2^-24, 2^24], fxu numerators <= 2^100 (tiny ones are
//    absorbed, g/2 >= 1/4) and cross numerators <= 2^36 (scaled by 2^64).
//    Instead of comparing every operand, each lane keeps the row's min / max
//    denominator and max numerators with 3-input FMNMX3 (NaN operands are
//    skipped -- NaN in gives NaN out on either path), and the row is checked
//    once; if any lane fails, the row is recomputed with DIV_FIXUP as before.
//  * Subnormal cross quotients (common in the far field of a wave) need no
//    branch: with qs = RN(a 2^64 / b) correctly rounded, qc = RN(qs 2^-64) is
//    the correctly rounded quotient unless qs 2^-64 lies exactly on a
//    midpoint of the subnormal grid (then the first rounding may have moved
//    it onto the tie; sw_math.cuh fdiv_subnormal_rn).  The down-scaling
//    error d = qc 2^64 - qs is exact, |d| < 2^-86 off a tie and == 2^-86 on
//    one, so each lane keeps max |d| over the row (FMNMX3) and a tie -- rare --
//    fails the row guard like an out-of-range operand (redone exactly with
//    DIV_FIXUP).
//  * Layout.  A lane's cells form the pairs P0 = (c0, c1), P1 = (c2, c3)
//    (as ld.shared.v4 delivers and st.global.v4 wants them); the x-faces are
//    computed as (f01, f12) = x(P0, (c1, c2)) and (f23, f34) = x(P1, (c3, c4)),
//    so only the right-hand cells (c1, c2) / (c3, c4) are assembled.
// ---------------------------------------------------------------------------
__device__ __forceinline__ float fmin3f(float a, float b, float c) {
    float r;
    asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}
__device__ __forceinline__ float fmax3f(float a, float b, float c) {
    float r;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}

struct XCoef2 {
    float2 half, cx2, cy2, cx, cy, g2;
    float2 nz;      // opaque -0.0 pair (see above)
};

struct RowGuard {
    float bmin, bmax, af, ac;   // denominators min / max, max fxu numerator, max |cross numerator|
    float tie;                  // max |qc 2^64 - qs| of the cross quotients (2^-86 = a subnormal tie)
    __device__ __forceinline__ void reset() { bmin = INFINITY; bmax = 0.f; af = 0.f; ac = 0.f; tie = 0.f; }
    __device__ __forceinline__ bool ok() const {
        return (bmin >= 0x1p-24f) & (bmax <= 0x1p+24f) & (af <= 0x1p+100f) & (ac <= 0x1p+36f) &
               (tie < 0x1p-86f);
    }
};

__device__ __forceinline__ float2 xmul(float2 a, float2 b, const XCoef2& c) { return __ffma2_rn(a, b, c.nz); }
__device__ __forceinline__ float2 xadd(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 xsub(float2 a, float2 b) { return __fadd2_rn(a, make_float2(-b.x, -b.y)); }

// RN(a / b) per element of the pair for the fxu numerators af and cross
// numerators ac over one denominator pair b.  DIV_GUARD: packed shared-
// reciprocal sequence + row guard; DIV_FIXUP: the never-failing scalar path.
template <int DM, int NF, int NC>
__device__ __forceinline__ void xdiv2(float2 b, const float2 (&af)[NF], const float2 (&ac)[NC], float2 (&qf)[NF],
                                      float2 (&qc)[NC], const XCoef2& c, RowGuard& gd) {
    if constexpr (DM == DIV_GUARD) {
        const float2 r0 = rcp2(b);
        const float2 r = __ffma2_rn(r0, __ffma2_rn(make_float2(-b.x, -b.y), r0, bc2(1.0f)), r0);
        const float2 nr = make_float2(-r.x, -r.y);
        gd.bmin = fmin3f(gd.bmin, b.x, b.y);
        gd.bmax = fmax3f(gd.bmax, b.x, b.y);
#pragma unroll
        for (int i = 0; i < NF; ++i) {
            const float2 qi = pmul2(af[i], r);
            const float2 res = __ffma2_rn(b, qi, make_float2(-af[i].x, -af[i].y));
            qf[i] = __ffma2_rn(nr, res, qi);
            gd.af = fmax3f(gd.af, af[i].x, af[i].y);       // squares: >= 0
        }
#pragma unroll
        for (int i = 0; i < NC; ++i) {
            const float2 as = pmul2(ac[i], bc2(0x1p64f));
            const float2 qi = pmul2(as, r);
            const float2 res = __ffma2_rn(b, qi, make_float2(-as.x, -as.y));
            const float2 qs = __ffma2_rn(nr, res, qi);
            qc[i] = xmul(qs, bc2(0x1p-64f), c);
            gd.ac = fmax3f(gd.ac, fabsf(ac[i].x), fabsf(ac[i].y));
            // exact down-scaling error: 0 for a normal quotient, |d| <= 2^-86 for a
            // subnormal one, == 2^-86 only on a tie of the second rounding
            const float2 d = __ffma2_rn(qc[i], bc2(0x1p64f), make_float2(-qs.x, -qs.y));
            gd.tie = fmax3f(gd.tie, fabsf(d.x), fabsf(d.y));
        }
    } else {
        bool ok = true;
#pragma unroll
        for (int i = 0; i < NF; ++i) {
            const float ax[1] = {af[i].x}, ay[1] = {af[i].y};
            float qx[1], qy[1];
            div_group<float, DM, 1>(b.x, ax, qx, ok);
            div_group<float, DM, 1>(b.y, ay, qy, ok);
            qf[i] = make_float2(qx[0], qy[0]);
        }
#pragma unroll
        for (int i = 0; i < NC; ++i) {
            const float ax[1] = {ac[i].x}, ay[1] = {ac[i].y};
            float qx[1], qy[1];
            div_group<float, DM, 1>(b.x, ax, qx, ok);
            div_group<float, DM, 1>(b.y, ay, qy, ok);
            qc[i] = make_float2(qx[0], qy[0]);
        }
    }
}

// cell quantities: fu = (u*u)/h + (g2*h)*h, fv = (v*v)/h + (g2*h)*h, cr = (u*v)/h
template <int DM>
__device__ __forceinline__ CellQ2 xcell(float2 h, float2 u, float2 v, const XCoef2& c, RowGuard& gd) {
    CellQ2 q;
    q.h = h; q.u = u; q.v = v;
    const float2 nf[2] = {pmul2(u, u), pmul2(v, v)}, nc[1] = {pmul2(u, v)};
    float2 qf[2], qc[1];
    xdiv2<DM, 2, 1>(h, nf, nc, qf, qc, c, gd);
    const float2 gh2 = xmul(pmul2(c.g2, h), h, c);
    q.fu = xadd(qf[0], gh2);
    q.fv = xadd(qf[1], gh2);
    q.cr = qc[0];
    return q;
}

// one face pair between cells A (left / down) and B (right / up): statements
// Hx, Ux, Vx (Y = false, coefficient cx2) or Hy, Uy, Vy (Y = true, cy2)
template <int DM, bool Y>
__device__ __forceinline__ FaceF2 xface(const CellQ2& A, const CellQ2& B, const XCoef2& c, RowGuard& gd) {
    const float2 k = Y ? c.cy2 : c.cx2;
    // normal momentum n (hu for x, hv for y), its flux fn, the tangential
    // momentum t and the cross flux
    const float2 Hf = xadd(xmul(c.half, xadd(A.h, B.h), c), xmul(k, xsub(Y ? A.v : A.u, Y ? B.v : B.u), c));
    const float2 Nf = xadd(xmul(c.half, xadd(Y ? A.v : A.u, Y ? B.v : B.u), c),
                           xmul(k, xsub(Y ? A.fv : A.fu, Y ? B.fv : B.fu), c));
    const float2 Tf = xadd(xmul(c.half, xadd(Y ? A.u : A.v, Y ? B.u : B.v), c), xmul(k, xsub(A.cr, B.cr), c));
    // x: Ux*Ux, Ux*Vx; y: Vy*Vy, Uy*Vy (operand order of the reference)
    const float2 nf[1] = {pmul2(Nf, Nf)}, nc[1] = {Y ? pmul2(Tf, Nf) : pmul2(Nf, Tf)};
    float2 qf[1], qc[1];
    xdiv2<DM, 1, 1>(Hf, nf, nc, qf, qc, c, gd);
    const float2 fn = xadd(qf[0], xmul(pmul2(c.g2, Hf), Hf, c));
    FaceF2 f;
    f.fh = Nf;
    f.fu = Y ? qc[0] : fn;
    f.fv = Y ? fn : qc[0];
    f.hd = Hf;
    return f;
}

__device__ __forceinline__ CellQ2 pair_of(const CellQ2& a, bool ahi, const CellQ2& b, bool bhi) {
    auto pick = [](float2 p, bool hi) { return hi ? p.y : p.x; };
    CellQ2 q;
    q.h = make_float2(pick(a.h, ahi), pick(b.h, bhi));
    q.u = make_float2(pick(a.u, ahi), pick(b.u, bhi));
    q.v = make_float2(pick(a.v, ahi), pick(b.v, bhi));
    q.fu = make_float2(pick(a.fu, ahi), pick(b.fu, bhi));
    q.fv = make_float2(0.f, 0.f);   // unused by x-faces
    q.cr = make_float2(pick(a.cr, ahi), pick(b.cr, bhi));
    return q;
}

struct ExactPairEngine2 {
    static constexpr int CPL = 4;
    CellQ2 pc[2];
    FaceF2 pdx[2], ydn[2];
    CellQ2 nc[2];
    FaceF2 ndx[2], yup[2];
    float2 nhx[2];      // depths of the new row's x-faces (f01, f12), (f23, f34) -- track() only
    XCoef2 c2;
    bool absorb;        // g/2 >= 1/4 (warp-uniform): else every row takes DIV_FIXUP

    __device__ __forceinline__ void init(const Coef<float>& c) {
        c2.half = bc2(c.half); c2.cx2 = bc2(c.cx2); c2.cy2 = bc2(c.cy2);
        c2.cx = bc2(c.cx); c2.cy = bc2(c.cy); c2.g2 = bc2(c.g2);
        // -0.0 from the sign of cx = dt/dx (> 0, rejected otherwise on the
        // host): a value ptxas cannot constant-fold
        const float nz = __uint_as_float((~__float_as_uint(c.cx)) & 0x80000000u);
        c2.nz = bc2(nz);
        absorb = c.g2 >= 0.25f;
        const float2 one = bc2(1.f), zero = bc2(0.f);
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            pc[j] = CellQ2{one, zero, zero, zero, zero, zero};
            pdx[j] = ydn[j] = FaceF2{zero, zero, zero, one};
        }
    }

    // The row in two guarded phases (the kernel redoes a failed phase with
    // DIV_FIXUP): (1) cell quantities + the y-faces below the row, after
    // which the previous row can be updated and its window dies; (2) the
    // x-faces.  Keeps the register peak low enough for a 2-row unroll.
    template <int DM>
    __device__ __forceinline__ void cells_y(const VecF<float>& h, const VecF<float>& u, const VecF<float>& v,
                                            bool have_prev, bool& ok) {
        RowGuard gd;
        gd.reset();
        nc[0] = xcell<DM>(make_float2(h.v[0], h.v[1]), make_float2(u.v[0], u.v[1]), make_float2(v.v[0], v.v[1]),
                          c2, gd);
        nc[1] = xcell<DM>(make_float2(h.v[2], h.v[3]), make_float2(u.v[2], u.v[3]), make_float2(v.v[2], v.v[3]),
                          c2, gd);
        if (have_prev) {
            yup[0] = xface<DM, true>(pc[0], nc[0], c2, gd);
            yup[1] = xface<DM, true>(pc[1], nc[1], c2, gd);
        }
        if constexpr (DM == DIV_GUARD) ok = ok & gd.ok() & absorb;
    }
    template <int DM>
    __device__ __forceinline__ void xfaces(bool want_x, bool& ok) {
        RowGuard gd;
        gd.reset();
        if (want_x) {
            CellQ2 nb;  // (c3, first cell of lane+1)
            nb.h = make_float2(nc[1].h.y, __shfl_down_sync(0xffffffffu, nc[0].h.x, 1));
            nb.u = make_float2(nc[1].u.y, __shfl_down_sync(0xffffffffu, nc[0].u.x, 1));
            nb.v = make_float2(nc[1].v.y, __shfl_down_sync(0xffffffffu, nc[0].v.x, 1));
            nb.fu = make_float2(nc[1].fu.y, __shfl_down_sync(0xffffffffu, nc[0].fu.x, 1));
            nb.cr = make_float2(nc[1].cr.y, __shfl_down_sync(0xffffffffu, nc[0].cr.x, 1));
            nb.fv = bc2(0.f);
            // (f01, f12) = x((c0, c1), (c1, c2)); (f23, f34) = x((c2, c3), (c3, c4))
            const FaceF2 F0 = xface<DM, false>(nc[0], pair_of(nc[0], true, nc[1], false), c2, gd);
            const FaceF2 F1 = xface<DM, false>(nc[1], nb, c2, gd);
            FaceF<float> fl;  // face left of c0 = lane-1's f34
            fl.fh = __shfl_up_sync(0xffffffffu, F1.fh.y, 1);
            fl.fu = __shfl_up_sync(0xffffffffu, F1.fu.y, 1);
            fl.fv = __shfl_up_sync(0xffffffffu, F1.fv.y, 1);
            // F_left - F_right per cell: (c0, c1) = (fl, f01) - (f01, f12); (c2, c3) = (f12, f23) - (f23, f34)
            ndx[0].fh = xsub(make_float2(fl.fh, F0.fh.x), F0.fh);
            ndx[0].fu = xsub(make_float2(fl.fu, F0.fu.x), F0.fu);
            ndx[0].fv = xsub(make_float2(fl.fv, F0.fv.x), F0.fv);
            ndx[1].fh = xsub(make_float2(F0.fh.y, F1.fh.x), F1.fh);
            ndx[1].fu = xsub(make_float2(F0.fu.y, F1.fu.x), F1.fu);
            ndx[1].fv = xsub(make_float2(F0.fv.y, F1.fv.x), F1.fv);
            nhx[0] = F0.hd;
            nhx[1] = F1.hd;
        }
        if constexpr (DM == DIV_GUARD) ok = ok & gd.ok() & absorb;
    }
    template <int DM>
    __device__ __forceinline__ void row(const VecF<float>& h, const VecF<float>& u, const VecF<float>& v,
                                        bool have_prev, bool want_x, const Coef<float>&, bool& ok) {
        cells_y<DM>(h, u, v, have_prev, ok);
        xfaces<DM>(want_x, ok);
    }
    // q' = (q + cx*(F_left - F_right)) + cy*(G_down - G_up), RN per node
    template <int DM>
    __device__ __forceinline__ void update(const Coef<float>&, float (&oh)[4], float (&ou)[4], float (&ov)[4]) const {
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            const float2 h = xadd(xadd(pc[j].h, xmul(c2.cx, pdx[j].fh, c2)), xmul(c2.cy, xsub(ydn[j].fh, yup[j].fh), c2));
            const float2 u = xadd(xadd(pc[j].u, xmul(c2.cx, pdx[j].fu, c2)), xmul(c2.cy, xsub(ydn[j].fu, yup[j].fu), c2));
            const float2 v = xadd(xadd(pc[j].v, xmul(c2.cx, pdx[j].fv, c2)), xmul(c2.cy, xsub(ydn[j].fv, yup[j].fv), c2));
            oh[2 * j] = h.x; oh[2 * j + 1] = h.y;
            ou[2 * j] = u.x; ou[2 * j + 1] = u.y;
            ov[2 * j] = v.x; ov[2 * j + 1] = v.y;
        }
    }
    __device__ __forceinline__ void shift() {
#pragma unroll
        for (int j = 0; j < 2; ++j) { pc[j] = nc[j]; ydn[j] = yup[j]; pdx[j] = ndx[j]; }
    }
    __device__ __forceinline__ void track(float& m, bool xall, bool xlast, bool y) const {
        const float inf = INFINITY;
        m = fminf(m, xall ? fminf(fminf(nhx[0].x, nhx[0].y), nhx[1].x) : inf);
        m = fminf(m, (xall || xlast) ? nhx[1].y : inf);
        m = fminf(m, y ? fminf(fminf(yup[0].hd.x, yup[0].hd.y), fminf(yup[1].hd.x, yup[1].hd.y)) : inf);
    }
};

}  // namespace fkc
