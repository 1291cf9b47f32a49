// Production stage-sweep kernels: the MB4 step as column-band marches; vertical
// neighbours in registers / own-column smem history, horizontal neighbours through
// shared-memory rows.  Default schedule (launch_split): two launches per (sub)step,
//   PH 1  the first sweep (MarchFirst2: depth-6 J-chain, Chebyshev-placed, fused energy
//         monitor; 2 CTAs/SM, bound by the shared-memory data pipe), then
//   PH 2  a persistent cooperative launch for the later sweeps (March3: grid barrier
//         between sweeps, in-kernel convergence test, speculative U3-only final sweep;
//         3 CTAs/SM at depth 1, bound by the FP64 pipe).
// PH 0 runs both in one launch (shallow first sweeps); PH 3 is the first sweep as a
// one-sweep launch with its status (sub-domain sweeps of the multi-GPU path).
//
// Same algorithm as sweep_march.cu and sweep_tiled.cu (Phi -> T^-1 -> M-term
// Neumann (I - h lam_k J)^-1 -> T -> update -> ||r||_inf; site_math.cuh) and
// the same band / work split.  Organised around the measured limits of the
// earlier versions (profiles/r01_*): shared-memory wavefronts, FP64 latency
// and integer overhead.
//  - Each thread keeps a 3-row register window of its own column of
//    z = (u0, U1..U3).  z rows arrive by cp.async in a 6-row ring (each thread fills
//    its own column); only the centre row's left/right neighbours are read from it
//    after the row barrier.
//  - Neumann level n works on row i - n at iteration i.  Every level publishes
//    its row into a double-buffered smem row; the neighbours read it one
//    iteration later, and the publishing thread reads its own column two rows
//    back from the same buffers, so one __syncthreads per row suffices.
//  - The Jacobian diagonal is recomputed from u0 where it is needed.
//  - Isotropic lattices (cx == cy, all BASELINE configs) evaluate the unit
//    stencil and fold c into pre-scaled coefficients (SweepConsts::Es, gs, hls);
//    the default scheme's tables are compile-time immediates (defscheme.inc).
//  - The first sweep of a step (U = (u0,u0,u0)) uses the closed form
//    Phi_i = -h c_i f(u0), c_i = sum_j E[i][j].
//  - The later-sweep loop is unrolled by 3 so register-window slots are static (z rows
//    and, at depth 1, the own-column Phi rows); the deep first sweep's loop by 6 (its
//    (P, Q, R) pipeline, u0 / V window and g_1..g_3 history rings rotate by static indices).
//  - Depth-1 later sweeps evaluate Phi in one FMA chain per stage and component
//    (MB4_PHI_FUSED), correct in stage space (r = Phi + hA J Phi), keep no halo columns
//    in the z rings (MB4_NOHALO) and take their band-rows in guided chunks from a device
//    counter (MB4_DYN_SPLIT: the CTAs sharing an SM advance at unequal rates).
// HBM traffic per sweep: 120 B/site (72 B/site for the first sweep, 88 for a
// U3-only final sweep).
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <atomic>
#include <cstdlib>

#include "async_copy.cuh"
#include "mb4cu_internal.hpp"
#include "site_math.cuh"

#ifndef MB4_CONSTS_IN_SMEM
#define MB4_CONSTS_IN_SMEM 1
#endif
#ifndef MB4_MINB_M1
#define MB4_MINB_M1 2
#endif
#ifndef MB4_UNROLL3
#define MB4_UNROLL3 1
#endif
// threads (= columns) per CTA of the production kernel: one band per CTA
#ifndef MB4_NT
#define MB4_NT 128
#endif
// Split step launches for deep first sweeps (mf >= 4): the first sweep in its own
// launch (its shared-memory rings allow 2 CTAs/SM), the later sweeps in a second,
// persistent launch at MB4_MINB_LATER CTAs/SM (depth-1 sweeps fit 3: <= 168
// registers, 70 KB shared memory) -- more warps to hide the FP64 latency.
#ifndef MB4_SPLIT
#define MB4_SPLIT 1
#endif
// first sweeps of depth 3..7: MarchFirst2 (power-of-two rings) instead of MarchFirst
#ifndef MB4_FIRST_V2
#define MB4_FIRST_V2 1
#endif
#ifndef MB4_FIRST_REGZ
#define MB4_FIRST_REGZ 1
#endif
// z rows of u0 / U (double2) arrive by bulk copies (TMA engine, one thread, mbarrier per
// ring slot) instead of per-thread cp.async; V stays on cp.async (8-byte elements).
// Measured (r02, cfg5): slower -- first sweep 1.34 -> 1.50 ms, later sweeps 1.60 -> 1.97 ms
// (threads spin on the ring mbarriers; the rows land later than the cp.async rows).
#ifndef MB4_BULK
#define MB4_BULK 0
#endif
// later sweeps: u0 / U ring rows placed so that every shared address has the alignment of
// its global source modulo 128 B (one cp.async wavefront per 128-byte line instead of two:
// the 16-byte cp.async of a misaligned row cost 9.2 wavefronts per warp instead of ~5)
#ifndef MB4_ALIGN_RING
#define MB4_ALIGN_RING 1
#endif
// later sweeps: the Neumann levels apply J through (P, Q, R) as well
#ifndef MB4_LATER_PQR
#define MB4_LATER_PQR 1
#endif
// later sweeps at depth 1 in stage space: r = Phi + hA (J Phi), hA = T diag(h lam) T^-1
// (no T^-1 / T transforms: 24 fewer FP64 operations per site; same operator, the
// correction rounds differently at the 1e-16 level)
#ifndef MB4_LATER_DIRECT
#define MB4_LATER_DIRECT 1
#endif
// first sweep: J applied through per-site coefficients (P, Q, R) formed once per site
#ifndef MB4_FIRST_PQR
#define MB4_FIRST_PQR 1
#endif
#ifndef MB4_MINB_LATER
#define MB4_MINB_LATER 3
#endif
// threads per CTA of the later-sweep launch (the band width; MINB scales with 128 / NT)
#ifndef MB4_NT_LATER
#define MB4_NT_LATER 128
#endif
// threads per CTA of the first-sweep launch
#ifndef MB4_NT_FIRST
#define MB4_NT_FIRST 128
#endif
// band-rows per CTA at least (small lattices): 1 = no idle CTAs; larger values trade CTAs
// for rows marched in sequence (measured slower at 32: the row march is latency-bound)
#ifndef MB4_MIN_ROWS_PER_CTA
#define MB4_MIN_ROWS_PER_CTA 1
#endif
// later sweeps: the own-column cubic term of a row before the row barrier (measured
// equal or slower: the later sweeps are FP64-bound, not barrier-bound)
#ifndef MB4_CUBIC_EARLY
#define MB4_CUBIC_EARLY 0
#endif
// later sweeps: Phi_k accumulated in ONE FMA chain per stage and component -- from
// z_k - z_0 through the six cubic node terms (weights h gamma WA) and the four stencil
// terms (weights h E) -- instead of separate cubic / stencil combinations joined by two
// more FMAs; with the default scheme the node values at twice their scale, the even part
// of the collocation polynomial from s12 + c_q (s03 - s12) (18 fewer FP64 operations per
// site; the own-column d = 4 + V/c window saves one more).  1: depth-1 later sweeps.
#ifndef MB4_PHI_FUSED
#define MB4_PHI_FUSED 1
#endif
// Later sweeps of a split step: the band-rows are handed out in chunks from a device
// counter (guided: the first round of chunks covers half of the rows, every further round
// half of the rest, down to MB4_DYN_SMIN rows) instead of one fixed share per CTA.  The
// CTAs that share an SM do not advance at the same rate (the warp schedulers favour one of
// them: with fixed shares the three CTAs of an SM finished at 0.87 / 1.13 / 1.39 ms at
// cfg5 and the SM ran its last third with one warp per scheduler); with chunks every CTA
// works until the rows run out.  Which CTA computes a row does not change its arithmetic.
#ifndef MB4_DYN_SPLIT
#define MB4_DYN_SPLIT 1
#endif
#ifndef MB4_DYN_SMIN
#define MB4_DYN_SMIN 32
#endif
// rows of a first-round chunk = (rows per CTA) * MB4_DYN_NUM / 8
#ifndef MB4_DYN_NUM
#define MB4_DYN_NUM 4
#endif
// the first sweep of a split step in chunks as well (its two CTAs per SM finish 6 % apart
// with fixed shares); every chunk stores its own energy partial sums, so the energy record
// does not depend on which CTA took which chunk.  Measured slower (cfg5 1.40 -> 1.49 ms):
// every chunk restarts the 2 MF + 2 = 14 warm-up rows of the depth-6 chain.  Off.
#ifndef MB4_DYN_FIRST
#define MB4_DYN_FIRST 0
#endif
// depth-1 later sweeps: no halo columns in the z rings.  Every thread fills its own column
// only; the band is one more column wider than its output on either side (TX = NT - 4), and
// lanes 0 / NT - 1 read an unfilled neighbour column, which only reaches masked lanes.  The
// halo fill was a divergent second copy pass (address arithmetic + 5 copies for 2 lanes)
// that warp 0 of every CTA ran on every row before the row's barrier partners could go on.
#ifndef MB4_NOHALO
#define MB4_NOHALO 1
#endif
// depth-1 later sweeps: the own-column Phi of the last two rows in a register window (slot =
// row mod 3, static after the unroll by 3) instead of re-read from the published rows
// (6 LDS.128 = 24 of ~128 shared-memory wavefronts per warp-row)
#ifndef MB4_PHI_REGS
#define MB4_PHI_REGS 1
#endif
// first sweep at depth 6: the row loop unrolled by 6, so the register pipelines of the site
// coefficients (6 rows of P, Q, R) and the u0 / V window (3 rows) rotate by static indices
// instead of ~60 register moves per row (20 % of the row's instructions)
#ifndef MB4_FIRST_UNROLL6
#define MB4_FIRST_UNROLL6 1
#endif
// ... and with static slots the own-column history of g_3 (a ring of 3 iterations) and g_2
// (of 6) holds the value the output row needs: two fewer history reads from shared memory
// (8 of ~119 wavefronts per warp-row).  0: off, 1: g_3, 2: g_3 and g_2, 3: and g_1.
#ifndef MB4_FIRST_GREG
#define MB4_FIRST_GREG 3
#endif
// first sweep: the neighbour values of level N + 1 are loaded before level N's arithmetic
// (they were published an iteration ago, so they do not depend on it), one level ahead
#ifndef MB4_FIRST_PREFETCH
#define MB4_FIRST_PREFETCH 1
#endif
// default-scheme later sweeps: the GL-6 nodes in symmetric pairs (experiment knob)
#ifndef MB4_SYM_PAIRS
#define MB4_SYM_PAIRS 1
#endif

namespace cg = cooperative_groups;

#ifdef MB4_CTA_TIMES
// profiling builds: per-CTA (start, end of its last sweep, SM id) of the latest step launch
// of each phase (tools/cta_times.py)
__device__ unsigned long long g_cta_times[4][2048][4];
// [0][1][k]: start of the last two first-sweep launches (k = launch parity), [0][2][0]: a counter
extern "C" int mb4cu_debug_cta_times(unsigned long long* out) {
    return static_cast<int>(cudaMemcpyFromSymbol(out, g_cta_times, sizeof(g_cta_times)));
}
#endif

namespace mb4cu {
namespace {

template <int M, int NT>
struct Geom3 {
    static_assert(M >= 0 && M <= 2, "march v3 supports Neumann depth 0..2");
    static constexpr int SH = MB4_NOHALO && M == 1 ? 1 : 0;  // unfilled ring columns per side
    static constexpr int TX = NT - 2 * (M + SH);  // output columns per band
    static constexpr int ZW = NT + 2;       // columns per smem row (1-site pad each side)
    static constexpr int S = 6;             // z ring rows (divisible by the unroll of 3)
    static constexpr int BACK = M == 2 ? 3 : 1;  // oldest z row still read: j - BACK
    static constexpr int P = S - 1 - BACK;  // rows in flight
    // row stride of the u0 / U rings: a multiple of 128 B with room for a shift of up to
    // 7 columns (MB4_ALIGN_RING)
    static constexpr int ZWP = MB4_ALIGN_RING ? ((ZW + 7 + 7) / 8) * 8 : ZW;
    static constexpr size_t zu0_bytes = sizeof(double2) * S * ZWP;
    static constexpr size_t zv_bytes = ((sizeof(double) * S * ZW + 15) / 16) * 16;
    static constexpr size_t zU_bytes = sizeof(double2) * S * 3 * ZWP;
    static constexpr size_t pub_bytes = sizeof(double2) * 2 * 3 * ZW;  // one level, 2 parities
    static constexpr size_t bytes = zu0_bytes + zv_bytes + zU_bytes + M * pub_bytes;
    // CTAs per SM: M <= 1 fits 3 (<= 168 registers, ~70 KB smem), M = 2 fits 2
    static constexpr int MINB = NT >= 256 ? 1 : (M == 2 ? 2 : MB4_MINB_M1);
};

// The default scheme's tables (alpha1 = -712.5, nodes 1/3, 2/3, 1) as compile-time
// constants, generated at build time from the library's scheme routine
// (gen_default_scheme.cpp).  Kernels specialised on them (DEF) fold the ~80 table
// entries into FFMA immediates instead of constant-bank loads and uniform-register
// shuffling (measured +4 % at cfg4 / cfg5, profiles/).
namespace defscheme {
#define MB4_DS_QUAL __device__ constexpr
#include "defscheme.inc"
#undef MB4_DS_QUAL
}  // namespace defscheme
// The same tables in the constant bank (c[0x3], values opaque to the compiler): sm_100a
// FP64 instructions take no constant-bank operand, so every table entry reaches a DFMA
// through a uniform register -- LDCU.128 moves two entries per instruction, while a
// compile-time immediate costs two UMOVs per entry (13 % of the later sweep's
// instructions with the constexpr tables).  Measured (r02): the later sweep spills at
// the 168-register bound and runs 1.6 -> 3.1 ms at cfg5, so the immediates stay.
namespace defscheme_cb {
#define MB4_DS_QUAL __constant__
#include "defscheme.inc"
#undef MB4_DS_QUAL
}  // namespace defscheme_cb
#ifndef MB4_DEF_CBANK
#define MB4_DEF_CBANK 0
#endif
#if MB4_DEF_CBANK
namespace dsv = defscheme_cb;
#else
namespace dsv = defscheme;
#endif

// Coefficient views: isotropic (unit stencil, pre-scaled constants) or general;
// DEF: scheme tables from defscheme (only with ISO, see dispatch3).
template <bool ISO, bool DEF = false>
struct Coef {
    const SweepConsts& c;
    __device__ __forceinline__ double Lq(int q, int b) const { return DEF ? dsv::L[q][b] : c.L[q][b]; }
    __device__ __forceinline__ double WAk(int k, int q) const { return DEF ? dsv::WA[k][q] : c.WA[k][q]; }
    // level-0 residual Phi_k = dz_k - hr * (E0 w ...) with w = (K+V) z (/ c if ISO):
    // ISO without DEF uses the pre-scaled Es = c E and the true gamma, h; ISO with
    // DEF the unscaled E and gamma / c, c h (the same product, one rounding apart).
    __device__ __forceinline__ double E0(int i, int j) const {
        return DEF ? dsv::E[i][j] : (ISO ? c.Es[i][j] : c.E[i][j]);
    }
    // fused Phi chains: h E (isotropic: c h E) and h gamma WA (/ 8 for node values at twice
    // their scale)
    __device__ __forceinline__ double hE(int k, int b) const { return ISO ? c.hEs[k][b] : c.hE[k][b]; }
    __device__ __forceinline__ double hgW(int k, int q) const { return c.hgW[k][q]; }
    __device__ __forceinline__ double hgW8(int k, int q) const { return c.hgW8[k][q]; }
    __device__ __forceinline__ double g0() const { return DEF && ISO ? c.gs : c.gamma; }
    __device__ __forceinline__ double h0() const { return DEF && ISO ? c.hs : c.h; }
    // phibar = T^-1 phi, r = T rbar
    __device__ __forceinline__ void to_eigen(const double2 phi[3], double2 out[3]) const {
#pragma unroll
        for (int k = 0; k < 3; ++k) {
            out[k].x = fma(Ti(k, 0), phi[0].x, fma(Ti(k, 1), phi[1].x, Ti(k, 2) * phi[2].x));
            out[k].y = fma(Ti(k, 0), phi[0].y, fma(Ti(k, 1), phi[1].y, Ti(k, 2) * phi[2].y));
        }
    }
    __device__ __forceinline__ void from_eigen(const double2 rb[3], double2 out[3]) const {
#pragma unroll
        for (int i = 0; i < 3; ++i) {
            out[i].x = fma(Tm(i, 0), rb[0].x, fma(Tm(i, 1), rb[1].x, Tm(i, 2) * rb[2].x));
            out[i].y = fma(Tm(i, 0), rb[0].y, fma(Tm(i, 1), rb[1].y, Tm(i, 2) * rb[2].y));
        }
    }
    __device__ __forceinline__ double Tm(int i, int k) const { return DEF ? dsv::T[i][k] : c.T[i][k]; }
    __device__ __forceinline__ double Ti(int k, int i) const { return DEF ? dsv::Tinv[k][i] : c.Tinv[k][i]; }
    __device__ __forceinline__ double g() const { return ISO ? c.gs : c.gamma; }
    __device__ __forceinline__ double hl(int k) const { return ISO ? c.hls[k] : c.hlam[k]; }
    __device__ __forceinline__ double hl2(int k) const { return ISO ? c.hls2[k] : c.hlam2[k]; }
    __device__ __forceinline__ double hA(int q, int k) const { return ISO ? c.hAs[q][k] : c.hA[q][k]; }
    __device__ __forceinline__ double fs(int k) const { return ISO ? c.first_ss[k] : c.first_s[k]; }
    __device__ __forceinline__ double fc(int k) const { return ISO ? c.first_cs[k] : c.first_c[k]; }
    // stencil diagonal incl. potential
    __device__ __forceinline__ double dv(double v) const { return ISO ? fma(v, c.inv_c, 4.0) : c.diag + v; }
    // (K+V) x (general) or (K+V) x / c (isotropic)
    __device__ __forceinline__ double2 kv(double d, double2 x, double2 l, double2 r, double2 dn,
                                          double2 up) const {
        double2 y;
        if (ISO) {
            y.x = fma(d, x.x, -((l.x + r.x) + (dn.x + up.x)));
            y.y = fma(d, x.y, -((l.y + r.y) + (dn.y + up.y)));
        } else {
            y.x = fma(d, x.x, -(c.cx * (l.x + r.x) + c.cy * (dn.x + up.x)));
            y.y = fma(d, x.y, -(c.cx * (l.y + r.y) + c.cy * (dn.y + up.y)));
        }
        return y;
    }
    // b = base + h lam_k J t, with a = kv(...) of t and the J diagonal of u0
    // (LEV 2: the second Horner level of a depth-2 sweep, multiplier hl2)
    template <int LEV = 1>
    __device__ __forceinline__ double2 horner(int k, double2 base, double2 t, double2 a, double2 u0) const {
        const double pp = u0.x * u0.x, qq = u0.y * u0.y;
        const double al = fma(3.0, pp, qq), be = 2.0 * u0.x * u0.y, de = fma(3.0, qq, pp);
        const double nlx = fma(al, t.x, be * t.y);
        const double nly = fma(be, t.x, de * t.y);
        const double jx = fma(-g(), nly, a.y);
        const double jy = fma(g(), nlx, -a.x);
        const double m = LEV == 2 ? hl2(k) : hl(k);
        return make_double2(fma(m, jx, base.x), fma(m, jy, base.y));
    }
    // Per-site coefficients of J (isotropic: J / c) in the form
    //   (J t).x = P t.y - (Q t.x + N.y),   (J t).y = R t.x + (Q t.y + N.x)
    // with N = the neighbour sum of t (cx (l + r) + cy (dn + up)) and, from u0 and the
    // stencil diagonal d = dv(v):  P = d - g (p^2 + 3 q^2),  Q = 2 g p q,
    // R = g (3 p^2 + q^2) - d  -- the same operator as jt(), 10 instead of 21 FP64
    // operations per application once P, Q, R are formed (once per site).
    struct PQR {
        double p, q, r;
    };
    __device__ __forceinline__ PQR pqr(double d, double2 u0) const {
        const double pp = u0.x * u0.x, qq = u0.y * u0.y;
        const double al = fma(3.0, pp, qq), de = fma(3.0, qq, pp);
        const double gg = g();
        return PQR{fma(-gg, de, d), 2.0 * gg * (u0.x * u0.y), fma(gg, al, -d)};
    }
    __device__ __forceinline__ double2 nsum(double2 l, double2 r, double2 dn, double2 up) const {
        if (ISO) return make_double2((l.x + r.x) + (dn.x + up.x), (l.y + r.y) + (dn.y + up.y));
        return make_double2(fma(c.cx, l.x + r.x, c.cy * (dn.x + up.x)), fma(c.cx, l.y + r.y, c.cy * (dn.y + up.y)));
    }
    __device__ __forceinline__ double2 jt_pqr(const PQR& k, double2 t, double2 n) const {
        return make_double2(fma(k.p, t.y, -fma(k.q, t.x, n.y)), fma(k.r, t.x, fma(k.q, t.y, n.x)));
    }
    // J t (isotropic: J t / c) from a = kv(...) of t and u0
    __device__ __forceinline__ double2 jt(double2 t, double2 a, double2 u0) const {
        const double pp = u0.x * u0.x, qq = u0.y * u0.y;
        const double al = fma(3.0, pp, qq), be = 2.0 * u0.x * u0.y, de = fma(3.0, qq, pp);
        const double nlx = fma(al, t.x, be * t.y);
        const double nly = fma(be, t.x, de * t.y);
        return make_double2(fma(-g(), nly, a.y), fma(g(), nlx, -a.x));
    }
};

template <int M, int NT, bool FIRST, bool ISO, bool GHOST, bool DEF = false>
struct March3 {
    using G = Geom3<M, NT>;
    // depth-1 later sweeps publish Phi itself (not T^-1 Phi) and correct by Phi + hA J Phi
    static constexpr bool DIRECT = M == 1 && !FIRST && MB4_LATER_DIRECT && MB4_LATER_PQR;
    // Phi accumulated in one chain per stage and component (MB4_PHI_FUSED)
    static constexpr bool FUSED = !FIRST && (MB4_PHI_FUSED == 2 || (MB4_PHI_FUSED == 1 && DIRECT));
    // element offset of local site (x, y) (both may lie in the halo)
    __device__ __forceinline__ static size_t at(const StepArgs& a, int x, int y) {
        if (GHOST) return static_cast<size_t>(y + a.ghost) * a.pitch + (x + a.ghost);
        return static_cast<size_t>(y) * a.nx + x;
    }
    double2* zu0;  // [S][ZWP] (shifted per segment by the alignment offset)
    double* zv;    // [S][ZW]
    double2* zU;   // [S][3][ZWP]
    double2* zu0_base;
    double2* zU_base;
    double2* pub;  // [M][2][3][ZW]

    double2 zw[3][4];  // own-column z rows; slot of z row k = k mod 3
    double vw[3];
    double2 pw[3][3];  // own-column Phi rows (MB4_PHI_REGS); slot of the row of iteration j = j mod 3
#if MB4_BULK
    unsigned long long* bars;  // one mbarrier per z ring slot (bulk row copies)
    __device__ static unsigned long long* ring_bars() {
        __shared__ unsigned long long b[G::S];
        return b;
    }
#endif

    __device__ March3(unsigned char* smem) {
#if MB4_BULK
        bars = ring_bars();
#endif
        zu0 = reinterpret_cast<double2*>(smem);
        zv = reinterpret_cast<double*>(smem + G::zu0_bytes);
        zU = reinterpret_cast<double2*>(smem + G::zu0_bytes + G::zv_bytes);
        zu0_base = zu0;
        zU_base = zU;
        pub = reinterpret_cast<double2*>(smem + G::zu0_bytes + G::zv_bytes + G::zU_bytes);
    }

    __device__ __forceinline__ double2* pub_row(int level, int parity, int k) {
        return pub + ((level * 2 + parity) * 3 + k) * G::ZW;
    }

    struct Seg {
        int X0, Y0, R, yz0, nzrows;
        int xlim;        // right edge (exclusive) of the output rectangle
        int smask;       // stages stored (bit q): 7, or 4 = U3 only (speculative final sweep)
        int gxa, gxb;    // global columns of smem column t + 1 and of halo column 0 / NT + 1 (t < 2)
        int gx0;         // global column of smem column 0 (wrapped; ghost-padded in GHOST mode)
        int next_row;    // global (periodic) row of the next z row to issue
        size_t next_off; // its element offset
    };

    // Issue z row k (rows are issued in order, so the row offset advances by one
    // pitch per call and wraps periodically without a division).
    __device__ __forceinline__ void issue_row(const StepArgs& a, const double2* const uin[3],
                                              Seg& s, int k, int slot) {
        if (k < s.nzrows) {
            const size_t rowoff = s.next_off;
            if (GHOST) {
                s.next_off += a.pitch;
            } else if (++s.next_row == a.ny) {
                s.next_row = 0;
                s.next_off = 0;
            } else {
                s.next_off += a.nx;
            }
            const int t = threadIdx.x;
#if MB4_BULK
            if (t == 0) {
                // the row segment's NT + 2 columns of u0 (and U1..U3) in one bulk copy each
                const int w = GHOST ? a.pitch : a.nx;
                const unsigned nb = bulk_row_bytes<!GHOST>(s.gx0, G::ZW, w);
                mbar_arrive_expect_tx(&bars[slot], nb * (FIRST ? 1 : 4));
                bulk_row<!GHOST>(&zu0[slot * G::ZWP], a.u0 + rowoff, s.gx0, G::ZW, w, &bars[slot]);
                if (!FIRST) {
#pragma unroll
                    for (int q = 0; q < 3; ++q)
                        bulk_row<!GHOST>(&zU[(slot * 3 + q) * G::ZWP], uin[q] + rowoff, s.gx0, G::ZW, w, &bars[slot]);
                }
            }
#endif
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                if (h == 1 && (G::SH || t >= 2)) break;
                // thread t fills its own column t + 1 (so it may read it before the row
                // barrier); threads 0 / 1 also fill the halo columns 0 / NT + 1
                const int col = h ? (t == 0 ? 0 : NT + 1) : t + 1;
                const size_t g = rowoff + (h ? s.gxb : s.gxa);
                cp_async8(&zv[slot * G::ZW + col], a.V + g);
#if !MB4_BULK
                cp_async16(&zu0[slot * G::ZWP + col], a.u0 + g);
                if (!FIRST) {
#pragma unroll
                    for (int q = 0; q < 3; ++q) cp_async16(&zU[(slot * 3 + q) * G::ZWP + col], uin[q] + g);
                }
#endif
            }
        }
        cp_async_commit();
    }

    // ||r||_inf on the high 32 bits of |r| (sign cleared): monotone, NaN/Inf above
    // every finite value.  The block result is widened to the largest double with
    // that high word, an upper bound within a factor 1 + 2^-20 of the true max, so
    // the convergence test can only be stricter than the reference's.
    __device__ __forceinline__ static void track(unsigned& rmax, double2 r) {
        const unsigned hx = static_cast<unsigned>(__double2hiint(r.x)) & 0x7FFFFFFFu;
        const unsigned hy = static_cast<unsigned>(__double2hiint(r.y)) & 0x7FFFFFFFu;
        rmax = max(rmax, max(hx, hy));
    }

    // cubic term of Phi at one site: sum_q WA[k][q] |U_q|^2 U_q over the 6 Gauss nodes,
    // U_q = sum_b L[q][b] z_b
    __device__ __forceinline__ static void cubic_site(const Coef<ISO, DEF>& cf, const double2 z[4], double2 cub[3]) {
#pragma unroll
        for (int k = 0; k < 3; ++k) cub[k] = make_double2(0.0, 0.0);
        if constexpr (DEF && MB4_SYM_PAIRS) {
            // default scheme: symmetric node pairs q, 5 - q (defscheme LS / LD):
            // U_q = E + O, U_{5-q} = E - O -- 12 instead of 24 node weights, 4 fewer FP64 ops
            const double2 s03 = make_double2(z[0].x + z[3].x, z[0].y + z[3].y);
            const double2 d03 = make_double2(z[0].x - z[3].x, z[0].y - z[3].y);
            const double2 s12 = make_double2(z[1].x + z[2].x, z[1].y + z[2].y);
            const double2 d12 = make_double2(z[1].x - z[2].x, z[1].y - z[2].y);
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                const double ex = fma(dsv::LS[q][1], s12.x, dsv::LS[q][0] * s03.x);
                const double ey = fma(dsv::LS[q][1], s12.y, dsv::LS[q][0] * s03.y);
                const double ox = fma(dsv::LD[q][1], d12.x, dsv::LD[q][0] * d03.x);
                const double oy = fma(dsv::LD[q][1], d12.y, dsv::LD[q][0] * d03.y);
#pragma unroll
                for (int side = 0; side < 2; ++side) {
                    const int qq = side ? 5 - q : q;
                    const double ur = side ? ex - ox : ex + ox, ui = side ? ey - oy : ey + oy;
                    const double n2 = fma(ur, ur, ui * ui);
                    const double gr = n2 * ur, gi = n2 * ui;
#pragma unroll
                    for (int k = 0; k < 3; ++k) {
                        cub[k].x = fma(cf.WAk(k, qq), gr, cub[k].x);
                        cub[k].y = fma(cf.WAk(k, qq), gi, cub[k].y);
                    }
                }
            }
            return;
        }
#pragma unroll
        for (int q = 0; q < 6; ++q) {
            double ur = cf.Lq(q, 0) * z[0].x, ui = cf.Lq(q, 0) * z[0].y;
#pragma unroll
            for (int b = 1; b < 4; ++b) {
                ur = fma(cf.Lq(q, b), z[b].x, ur);
                ui = fma(cf.Lq(q, b), z[b].y, ui);
            }
            const double n2 = fma(ur, ur, ui * ui);
            const double gr = n2 * ur, gi = n2 * ui;
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                cub[k].x = fma(cf.WAk(k, q), gr, cub[k].x);
                cub[k].y = fma(cf.WAk(k, q), gi, cub[k].y);
            }
        }
    }

    // Fused form: adds the cubic term of Phi_k to phi[k] (which holds z_k+1 - z_0):
    //   phi[k].x += sum_q (h gamma WA[k][q]) Im(|U_q|^2 U_q),  phi[k].y -= ... Re(...)
    __device__ __forceinline__ static void cubic_into(const Coef<ISO, DEF>& cf, const double2 z[4], double2 phi[3]) {
        if constexpr (DEF && MB4_SYM_PAIRS) {
            // default scheme (nodes 0, 1/3, 2/3, 1): with s = tau - 1/2 the even part of 2 U
            // is s12 + ce(s) (s03 - s12), ce = (36 s^2 - 1) / 8 = 2 LS[q][0]; the odd part
            // 2 (LD[q][0] d03 + LD[q][1] d12).  Node values at twice their scale: weights / 8.
            const double2 s03 = make_double2(z[0].x + z[3].x, z[0].y + z[3].y);
            const double2 d03 = make_double2(z[0].x - z[3].x, z[0].y - z[3].y);
            const double2 s12 = make_double2(z[1].x + z[2].x, z[1].y + z[2].y);
            const double2 d12 = make_double2(z[1].x - z[2].x, z[1].y - z[2].y);
            const double2 ds = make_double2(s03.x - s12.x, s03.y - s12.y);
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                const double ce = 2.0 * dsv::LS[q][0], o0 = 2.0 * dsv::LD[q][0], o1 = 2.0 * dsv::LD[q][1];
                const double ex = fma(ce, ds.x, s12.x), ey = fma(ce, ds.y, s12.y);
                const double ox = fma(o1, d12.x, o0 * d03.x), oy = fma(o1, d12.y, o0 * d03.y);
#pragma unroll
                for (int side = 0; side < 2; ++side) {
                    const int qq = side ? 5 - q : q;
                    const double ur = side ? ex - ox : ex + ox, ui = side ? ey - oy : ey + oy;
                    const double n2 = fma(ur, ur, ui * ui);
                    const double gr = n2 * ur, gi = n2 * ui;
#pragma unroll
                    for (int k = 0; k < 3; ++k) {
                        phi[k].x = fma(cf.hgW8(k, qq), gi, phi[k].x);
                        phi[k].y = fma(-cf.hgW8(k, qq), gr, phi[k].y);
                    }
                }
            }
        } else {
#pragma unroll
            for (int q = 0; q < 6; ++q) {
                double ur = cf.Lq(q, 0) * z[0].x, ui = cf.Lq(q, 0) * z[0].y;
#pragma unroll
                for (int b = 1; b < 4; ++b) {
                    ur = fma(cf.Lq(q, b), z[b].x, ur);
                    ui = fma(cf.Lq(q, b), z[b].y, ui);
                }
                const double n2 = fma(ur, ur, ui * ui);
                const double gr = n2 * ur, gi = n2 * ui;
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    phi[k].x = fma(cf.hgW(k, q), gi, phi[k].x);
                    phi[k].y = fma(-cf.hgW(k, q), gr, phi[k].y);
                }
            }
        }
    }

    // Iteration j (level-0 row i = j - 2).  PH = j mod 3 (static); h3 = 3 * ((j / 3) & 1).
    template <int PH>
    __device__ __forceinline__ void body(const StepArgs& a, const Coef<ISO, DEF>& cf,
                                         const double2* const uin[3], double2* const uout[3],
                                         Seg& s, int j, int h3, unsigned& rmax,
                                         double* acc) {
        constexpr int S_NEW = PH;            // z row j      (own column, newly loaded)
        constexpr int S_CEN = (PH + 2) % 3;  // z row j - 1  (level-0 centre row)
        constexpr int S_DN = (PH + 1) % 3;   // z row j - 2
        const SweepConsts& c = cf.c;
        const int t = threadIdx.x;
        const int cc = t + 1;
        const int i = j - 2;

        // ring slots: row j - k lives in slot (j - k) mod 6 = (h3 + PH - k) mod 6
        auto ring = [&](int k) {
            int x = h3 + PH - k + 6;
            x = x >= 6 ? x - 6 : x;
            return x >= 6 ? x - 6 : x;
        };
        const int slot_new = ring(0);
        const int slot_cen = ring(1);

        // ---- own column, before the row barrier --------------------------------
        // The new z row j (own column: this thread's own cp.async group) and, for later
        // sweeps, the cubic term of the centre row (own-column registers only) need no
        // other thread's data, so a warp that finished the previous row early does this
        // share (~40 % of the row's FP64 work) while slower warps of the CTA catch up.
        cp_async_wait<G::P - 1>();
#if MB4_BULK
        // this segment's z row j (use j / S of its slot); the unroll by 3 runs up to two
        // iterations past the last row, which read no new row
        if (j < s.nzrows) mbar_wait(&bars[slot_new], (j / G::S) & 1);
#endif
        zw[S_NEW][0] = zu0[slot_new * G::ZWP + cc];
        // (fused later sweeps keep the stencil diagonal d = dv(V) in the window, not V)
        vw[S_NEW] = FUSED ? cf.dv(zv[slot_new * G::ZW + cc]) : zv[slot_new * G::ZW + cc];
        if (!FIRST) {
#pragma unroll
            for (int q = 0; q < 3; ++q) zw[S_NEW][q + 1] = zU[(slot_new * 3 + q) * G::ZWP + cc];
        }
        double2 cub[3];  // cubic term at the 6 Gauss nodes of the collocation polynomial
        if (!FIRST && MB4_CUBIC_EARLY) cubic_site(cf, zw[S_CEN], cub);
        __syncthreads();
        issue_row(a, uin, s, j + G::P, ring(-G::P));

        const int yrel = i - 2 * M;  // output row offset from Y0
        const int xout = s.X0 - (M + G::SH) + t;
        const bool out_ok = yrel >= 0 && yrel < s.R && t >= M + G::SH && t < NT - (M + G::SH) && xout < s.xlim;
        const int par = j & 1, ppar = par ^ 1;

        // own-column level history, read before this iteration overwrites it
        double2 pb_m2[3];  // phibar row i-2 (M == 2)
        double2 b1_m3[3];  // b1 row i-3   (M == 2)
        if (M == 2) {
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                pb_m2[k] = pub_row(0, par, k)[cc];
                b1_m3[k] = pub_row(1, par, k)[cc];
            }
        }

        // ---- level 0 at row i ---------------------------------------------------
        const double v = vw[S_CEN];
        const double d0 = FUSED ? v : cf.dv(v);
        const double2 u0c = zw[S_CEN][0];
        double2 pb[3];
        {
            const double2 w0 = cf.kv(d0, u0c, zu0[slot_cen * G::ZWP + cc - 1], zu0[slot_cen * G::ZWP + cc + 1],
                                     zw[S_DN][0], zw[S_NEW][0]);
            if (FIRST) {
                // f(u0)/scale = -i(w0 - g |u0|^2 u0); phibar_k = fs_k * f
                const double n2 = fma(u0c.x, u0c.x, u0c.y * u0c.y);
                const double gx = fma(-cf.g() * n2, u0c.x, w0.x);
                const double gy = fma(-cf.g() * n2, u0c.y, w0.y);
                const double2 f = make_double2(gy, -gx);
                if (M == 0) {
                    if (out_ok) {
                        const size_t gi = at(a, xout, s.Y0 + yrel);
#pragma unroll
                        for (int q = 0; q < 3; ++q) {
                            const double2 r = make_double2(cf.fc(q) * f.x, cf.fc(q) * f.y);
                            uout[q][gi] = make_double2(u0c.x + r.x, u0c.y + r.y);
                            track(rmax, r);
                        }
                    }
                } else {
#pragma unroll
                    for (int k = 0; k < 3; ++k) pb[k] = make_double2(cf.fs(k) * f.x, cf.fs(k) * f.y);
                }
                // energy monitor of u0 on owned sites (lattice.cpp:106-137)
                if (i >= M && i < M + s.R && t >= M + G::SH && t < NT - (M + G::SH) && xout < s.xlim) {
                    const double vn = v * n2;
                    const double sc = ISO ? c.cx : 1.0;
                    monitor_add(acc, fma(sc, fma(u0c.x, w0.x, u0c.y * w0.y), -vn), sc * fma(u0c.x, w0.y, -u0c.y * w0.x), n2,
                                vn);
                }
            } else {
                double2 z[4], w[4];
                z[0] = u0c;
                w[0] = w0;
#pragma unroll
                for (int q = 1; q < 4; ++q) {
                    const double2* row = zU + (slot_cen * 3 + (q - 1)) * G::ZWP;
                    z[q] = zw[S_CEN][q];
                    w[q] = cf.kv(d0, z[q], row[cc - 1], row[cc + 1], zw[S_DN][q], zw[S_NEW][q]);
                }
                double2 phi[3];
                if constexpr (FUSED) {
#pragma unroll
                    for (int k = 0; k < 3; ++k) phi[k] = make_double2(z[k + 1].x - z[0].x, z[k + 1].y - z[0].y);
                    cubic_into(cf, z, phi);  // (own column only: may be scheduled before the neighbour loads)
#pragma unroll
                    for (int k = 0; k < 3; ++k) {
#pragma unroll
                        for (int b = 0; b < 4; ++b) {
                            phi[k].x = fma(-cf.hE(k, b), w[b].y, phi[k].x);
                            phi[k].y = fma(cf.hE(k, b), w[b].x, phi[k].y);
                        }
                    }
                } else {
                if (!MB4_CUBIC_EARLY) cubic_site(cf, z, cub);
#pragma unroll
                for (int k = 0; k < 3; ++k) {
                    double kr = cf.E0(k, 0) * w[0].x, ki = cf.E0(k, 0) * w[0].y;
#pragma unroll
                    for (int b = 1; b < 4; ++b) {
                        kr = fma(cf.E0(k, b), w[b].x, kr);
                        ki = fma(cf.E0(k, b), w[b].y, ki);
                    }
                    const double rr = fma(-cf.g0(), cub[k].y, ki);
                    const double ri = fma(cf.g0(), cub[k].x, -kr);
                    phi[k].x = fma(-cf.h0(), rr, z[k + 1].x - z[0].x);
                    phi[k].y = fma(-cf.h0(), ri, z[k + 1].y - z[0].y);
                }
                }
                if (M == 0) {
                    if (out_ok) {
                        const size_t gi = at(a, xout, s.Y0 + yrel);
#pragma unroll
                        for (int q = 0; q < 3; ++q) {
                            if ((s.smask >> q) & 1)
                                uout[q][gi] = make_double2(z[q + 1].x - phi[q].x, z[q + 1].y - phi[q].y);
                            track(rmax, phi[q]);
                        }
                    }
                } else if (DIRECT) {
#pragma unroll
                    for (int k = 0; k < 3; ++k) pb[k] = phi[k];
                } else {
                    cf.to_eigen(phi, pb);
                }
            }
        }
        if (M == 0) return;

        // ---- level 1 at row i - 1 ----------------------------------------------
        if constexpr (DIRECT) {
            // r = Phi + hA J Phi at row i - 1 (J of each stage's Phi through the site's
            // (P, Q, R); Phi of rows i - 2 / i - 1 own column and the neighbours from the
            // published rows)
            const auto K1 = cf.pqr(FUSED ? vw[S_DN] : cf.dv(vw[S_DN]), zw[S_DN][0]);
            double2 jk[3], tc[3];
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const double2* prow = pub_row(0, ppar, k);  // Phi row i - 1
                tc[k] = MB4_PHI_REGS ? pw[S_CEN][k] : prow[cc];
                const double2 td = MB4_PHI_REGS == 1 ? pw[S_DN][k] : pub_row(0, par, k)[cc];  // row i - 2
                jk[k] = cf.jt_pqr(K1, tc[k], cf.nsum(prow[cc - 1], prow[cc + 1], td, pb[k]));
                if (MB4_PHI_REGS) pw[S_NEW][k] = pb[k];
            }
#pragma unroll
            for (int k = 0; k < 3; ++k) pub_row(0, par, k)[cc] = pb[k];
            if (out_ok) {
                const size_t gi = at(a, xout, s.Y0 + yrel);
#pragma unroll
                for (int q = 0; q < 3; ++q) {
                    double rx = fma(cf.hA(q, 0), jk[0].x, tc[q].x), ry = fma(cf.hA(q, 0), jk[0].y, tc[q].y);
                    rx = fma(cf.hA(q, 1), jk[1].x, rx);
                    ry = fma(cf.hA(q, 1), jk[1].y, ry);
                    rx = fma(cf.hA(q, 2), jk[2].x, rx);
                    ry = fma(cf.hA(q, 2), jk[2].y, ry);
                    const double2 uo = zw[S_DN][q + 1];
                    if ((s.smask >> q) & 1) uout[q][gi] = make_double2(uo.x - rx, uo.y - ry);
                    track(rmax, make_double2(rx, ry));
                }
            }
            return;
        }
        double2 b1[3];
        {
            const double2 u0m = zw[S_DN][0];          // u0 of row i - 1 (z row j - 2)
            const double dm = FUSED ? vw[S_DN] : cf.dv(vw[S_DN]);
#if MB4_LATER_PQR
            const auto K1 = cf.pqr(dm, u0m);  // J at the site, formed once for the 3 stages
#endif
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const double2* prow = pub_row(0, ppar, k);  // phibar row i - 1
                const double2 tc = prow[cc];
                const double2 td = M == 2 ? pb_m2[k] : pub_row(0, par, k)[cc];  // row i - 2
#if MB4_LATER_PQR
                const double2 jk = cf.jt_pqr(K1, tc, cf.nsum(prow[cc - 1], prow[cc + 1], td, pb[k]));
                b1[k] = make_double2(fma(cf.hl(k), jk.x, tc.x), fma(cf.hl(k), jk.y, tc.y));
#else
                const double2 ak = cf.kv(dm, tc, prow[cc - 1], prow[cc + 1], td, pb[k]);
                b1[k] = cf.horner(k, tc, tc, ak, u0m);
#endif
            }
        }
        // publish phibar row i (after the own-column history reads above)
#pragma unroll
        for (int k = 0; k < 3; ++k) pub_row(0, par, k)[cc] = pb[k];

        if (M == 1) {
            if (out_ok) {
                // r = T rbar = -T b1
                double2 tb[3];
                cf.from_eigen(b1, tb);
                const size_t gi = at(a, xout, s.Y0 + yrel);
#pragma unroll
                for (int q = 0; q < 3; ++q) {
                    const double2 uo = FIRST ? zw[S_DN][0] : zw[S_DN][q + 1];
                    if ((s.smask >> q) & 1) uout[q][gi] = make_double2(uo.x - tb[q].x, uo.y - tb[q].y);
                    track(rmax, tb[q]);
                }
            }
            return;
        }

        // ---- level 2 at row i - 2 (final, M == 2) -------------------------------
        if (out_ok) {
            const int slot_m3 = ring(3);             // z row j - 3 == row i - 2
            const double2 u0m = zu0[slot_m3 * G::ZWP + cc];
            const double dm = cf.dv(zv[slot_m3 * G::ZW + cc]);
            double2 b2[3];
#if MB4_LATER_PQR
            const auto K2 = cf.pqr(dm, u0m);
#endif
#pragma unroll
            for (int k = 0; k < 3; ++k) {
                const double2* prow = pub_row(1, ppar, k);  // b1 row i - 2
                const double2 tc = prow[cc];
#if MB4_LATER_PQR
                const double2 jk = cf.jt_pqr(K2, tc, cf.nsum(prow[cc - 1], prow[cc + 1], b1_m3[k], b1[k]));
                b2[k] = make_double2(fma(cf.hl2(k), jk.x, pb_m2[k].x), fma(cf.hl2(k), jk.y, pb_m2[k].y));
#else
                const double2 ak = cf.kv(dm, tc, prow[cc - 1], prow[cc + 1], b1_m3[k], b1[k]);
                b2[k] = cf.template horner<2>(k, pb_m2[k], tc, ak, u0m);
#endif
            }
            double2 tb[3];
            cf.from_eigen(b2, tb);  // r = -T b2
            const size_t gi = at(a, xout, s.Y0 + yrel);
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                const double2 uo = FIRST ? u0m : zU[(slot_m3 * 3 + q) * G::ZWP + cc];
                if ((s.smask >> q) & 1) uout[q][gi] = make_double2(uo.x - tb[q].x, uo.y - tb[q].y);
                track(rmax, tb[q]);
            }
        }
#pragma unroll
        for (int k = 0; k < 3; ++k) pub_row(1, par, k)[cc] = b1[k];
    }

    __device__ void run(const StepArgs& a, const SweepConsts& c, const double2* const uin[3],
                        double2* const uout[3], int X0, int xlim, int Y0, int R, unsigned& rmax,
                        double* acc, int smask) {
        const Coef<ISO, DEF> cf{c};
        Seg s;
        s.smask = smask;
        s.X0 = X0;
        s.xlim = xlim;
        s.Y0 = Y0;
        s.R = R;
        s.yz0 = Y0 - M - 1;
        s.nzrows = R + 2 * M + 2;
        if (GHOST) {
            s.next_off = static_cast<size_t>(s.yz0 + a.ghost) * a.pitch;
        } else {
            s.next_row = wrap_index(s.yz0, a.ny);
            s.next_off = static_cast<size_t>(s.next_row) * a.nx;
        }
        const int xz0 = s.X0 - M - 1 - G::SH;  // global column of smem column 0
        const int t = static_cast<int>(threadIdx.x);
        const int xa = xz0 + t + 1, xb = t == 0 ? xz0 : xz0 + NT + 1;  // see issue_row
        if (GHOST) {
            // padded columns; columns past the right halo only feed masked outputs
            const int last = a.pitch - 1;
            const int ca = xa + a.ghost, cb = xb + a.ghost;
            s.gxa = ca < last ? ca : last;
            s.gxb = cb < last ? cb : last;
            s.gx0 = xz0 + a.ghost;
        } else {
            s.gxa = wrap_index(xa, a.nx);
            s.gxb = wrap_index(xb, a.nx);
            s.gx0 = wrap_index(xz0, a.nx);
        }
#if MB4_ALIGN_RING
        // column c of the ring rows at the alignment of global column gx0 + c (mod 128 B;
        // exact when the row pitch is a multiple of 8 sites, as for every BASELINE lattice)
        {
            const int su0 = static_cast<int>(smem_u32(zu0_base) >> 4), sU = static_cast<int>(smem_u32(zU_base) >> 4);
            zu0 = zu0_base + ((s.gx0 - su0) & 7);
            zU = zU_base + ((s.gx0 - sU) & 7);
        }
#endif
#if MB4_BULK
        // fresh ring barriers per segment (every row of the previous segment was consumed)
        if (t == 0) {
#pragma unroll
            for (int q = 0; q < G::S; ++q) mbar_init(&bars[q], 1);
            mbar_fence_init();
        }
        __syncthreads();
#endif
#pragma unroll
        for (int k = 0; k < G::P; ++k) issue_row(a, uin, s, k, k);
        const int jend = R + 2 * M + 2;
#if MB4_UNROLL3
        for (int j = 0; j < jend; j += 3) {
            const int h3 = ((j / 3) & 1) * 3;
            body<0>(a, cf, uin, uout, s, j, h3, rmax, acc);
            body<1>(a, cf, uin, uout, s, j + 1, h3, rmax, acc);
            body<2>(a, cf, uin, uout, s, j + 2, h3, rmax, acc);
            if (FIRST) monitor_flush(acc);  // (shallow first sweeps: every 3 rows)
        }
#else
        // one body per row; the register window rotates by explicit moves
        for (int j = 0; j < jend; ++j) {
            body<0>(a, cf, uin, uout, s, j, j % 6, rmax, acc);
            if (FIRST) monitor_flush(acc);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                zw[1][q] = zw[2][q];
                zw[2][q] = zw[0][q];
            }
            vw[1] = vw[2];
            vw[2] = vw[0];
        }
#endif
        cp_async_wait<0>();
        __syncthreads();
    }
};

// First sweep of a step at Neumann depth MF >= 1, specialised.  From U = (u0,u0,u0)
// every phibar_k = first_s[k] f(u0), so the MF-term recursion of all three stages
// reduces to ONE chain g_0 = f, g_n = J g_{n-1} (one complex per site and level
// instead of three) and U_i = u0 + sum_n fco[i][n] g_n.  The chain is cheap, so the
// first sweep runs deep (default MF = 6): on the nearly linear stage systems of the
// BASELINE configs it leaves only the nonlinear remainder for the later sweeps
// (cfg5: 4 -> 2 sweeps per step, profiles/).
//
// Same band march as March3: level n works on row i - n at iteration j (i = j - 2),
// one barrier per row.  Level n-1 publishes its row into a ring of own-column
// history (depth D_n) from which level n reads the centre row's left/right
// neighbours (previous iteration) and its own column two rows back; the output row
// i - MF reads the older chain values g_n(i - MF), n <= MF - 3, from the same rings.
template <int MF, int NT, bool ISO, bool GHOST>
struct MarchFirst {
    static_assert(MF >= 1 && MF <= kMaxNeumannFirst, "first-sweep depth");
    static constexpr int TX = NT - 2 * MF;  // output columns per band
    static constexpr int ZW = NT + 2;
    // z rows kept behind the newest: levels n >= 2 read u0 / V of row i - n from the ring
    static constexpr int BACK = MF >= 2 ? MF + 1 : 1;
    // rows in flight: light rows, prefetch deep to cover HBM latency (smem-bounded)
#ifndef MB4_FIRST_P
#define MB4_FIRST_P 8
#endif
    static constexpr int P = MF <= 2 ? 10 - (MF == 2 ? 2 : 0) : MB4_FIRST_P;
    static constexpr int S = P + 1 + BACK;
    // history depth of level n: the output reads g_n(i - MF), written MF - n iterations ago
    __host__ __device__ static constexpr int depth(int n) { return n >= MF - 2 ? 2 : MF - n + 1; }
    __host__ __device__ static constexpr int base(int n) { return n == 0 ? 0 : base(n - 1) + depth(n - 1); }
    static constexpr int HROWS = base(MF);
    static constexpr size_t zu0_bytes = sizeof(double2) * S * ZW;
    static constexpr size_t zv_bytes = ((sizeof(double) * S * ZW + 15) / 16) * 16;
    static constexpr size_t bytes = zu0_bytes + zv_bytes + sizeof(double2) * HROWS * ZW;

    double2* zu0;
    double* zv;
    double2* hist;  // [HROWS][ZW]
    double2 zw[3];
    double vw[3];
    // own-column g_n of the last two iterations, slot = iteration parity (static
    // after the unroll by 2): the centre and down values of level n + 1 come from
    // registers, only the left/right neighbours from shared memory
    double2 gp[MF][2];
    // ring positions of iteration j, advanced incrementally (no integer division):
    // zs = j mod S, hs[n] = j mod depth(n) for the deep-history levels n <= MF - 3
    int zs;
    int hs[MF > 3 ? MF - 2 : 1];
    __device__ __forceinline__ int zslot(int back) const {  // z ring slot of z row j - back
        const int x = zs - back;
        return x < 0 ? x + S : x;
    }

    __device__ MarchFirst(unsigned char* smem) {
        zu0 = reinterpret_cast<double2*>(smem);
        zv = reinterpret_cast<double*>(smem + zu0_bytes);
        hist = reinterpret_cast<double2*>(smem + zu0_bytes + zv_bytes);
    }
    // own-column g_N(i - MF) for N <= MF - 3, written at iteration j - MF + N
    template <int N>
    __device__ __forceinline__ void gather(double2* gout) {
        if constexpr (N + 3 <= MF) {
            // slot (j - (MF - N)) mod D = (j + 1) mod D, as D = MF - N + 1
            constexpr int D = depth(N);
            const int sl = hs[N] + 1 == D ? 0 : hs[N] + 1;
            gout[N] = hist[(base(N) + sl) * ZW + threadIdx.x + 1];
            gather<N + 1>(gout);
        }
    }
    __device__ __forceinline__ static size_t at(const StepArgs& a, int x, int y) {
        if (GHOST) return static_cast<size_t>(y + a.ghost) * a.pitch + (x + a.ghost);
        return static_cast<size_t>(y) * a.nx + x;
    }

    struct Seg {
        int X0, Y0, R, nzrows, gxa, gxb, next_row;
        int xlim;  // right edge (exclusive) of the output rectangle
        size_t next_off;
    };

    __device__ __forceinline__ void issue_row(const StepArgs& a, Seg& s, int k, int slot) {
        if (k < s.nzrows) {
            const size_t rowoff = s.next_off;
            if (GHOST) {
                s.next_off += a.pitch;
            } else if (++s.next_row == a.ny) {
                s.next_row = 0;
                s.next_off = 0;
            } else {
                s.next_off += a.nx;
            }
            const int t = threadIdx.x;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                if (h == 1 && t >= 2) break;
                const int col = t + h * NT;
                const size_t g = rowoff + (h ? s.gxb : s.gxa);
                cp_async16(&zu0[slot * ZW + col], a.u0 + g);
                cp_async8(&zv[slot * ZW + col], a.V + g);
            }
        }
        cp_async_commit();
    }

    struct Chain {
        double2 up;   // g_{n-1}(i - n + 1), computed this iteration
        double2 low;  // g_{MF-2}(i - MF)
        double2 mid;  // g_{MF-1}(i - MF)
        double2 u0o;  // u0(i - MF), loaded by level MF (the output row)
    };

    // level N (compile-time recursion: every ring offset and slot depth is static)
    template <int N, int PAR>
    __device__ __forceinline__ void levels(const Coef<ISO>& cf, int j, Chain& ch) {
        if constexpr (N <= MF) {
            constexpr int D = depth(N - 1);
            const int cc = threadIdx.x + 1;
            int s_own = PAR, s_prev = PAR ^ 1;  // depth 2: slot = iteration parity
            if constexpr (D != 2) {
                s_own = hs[N - 1];
                s_prev = s_own == 0 ? D - 1 : s_own - 1;
            }
            const double2* crow = hist + (base(N - 1) + s_prev) * ZW;  // iteration j - 1
            double2* own = hist + (base(N - 1) + s_own) * ZW;          // iteration j
            const double2 gc = gp[N - 1][PAR ^ 1];                       // iteration j - 1
            const double2 gd = gp[N - 1][PAR];                           // iteration j - 2
            const int zrow = zslot(N + 1);                               // z row of i - N
            const double2 u0n = N == 1 ? zw[2] : zu0[zrow * ZW + cc];
            const double vn = N == 1 ? vw[2] : zv[zrow * ZW + cc];
            const double2 an = cf.kv(cf.dv(vn), gc, crow[cc - 1], crow[cc + 1], gd, ch.up);
            const double2 gn = cf.jt(gc, an, u0n);
            own[cc] = ch.up;  // publish g_{N-1}(i - N + 1) for the neighbours / the output
            gp[N - 1][PAR] = ch.up;
            if (N == MF - 1) ch.low = gd;
            if (N == MF) {
                ch.mid = gc;
                ch.u0o = u0n;
            }
            ch.up = gn;
            levels<N + 1, PAR>(cf, j, ch);
        }
    }

    // j >= 0; iterations before a level's first valid row compute on stale rows and
    // are masked (out_ok / the monitor window), as in March3.
    template <int PAR>  // = j & 1
    __device__ __forceinline__ void body(const StepArgs& a, const Coef<ISO>& cf, double2* const uout[3],
                                         Seg& s, int j, unsigned& rmax, double* acc) {
        const SweepConsts& c = cf.c;
        const int t = threadIdx.x, cc = t + 1, i = j - 2;
        const int slot_new = zs, slot_cen = zslot(1);
        cp_async_wait<P - 1>();
        __syncthreads();
        issue_row(a, s, j + P, zs + P >= S ? zs + P - S : zs + P);

        const int yrel = i - 2 * MF;
        const int xout = s.X0 - MF + t;
        const bool out_ok = yrel >= 0 && yrel < s.R && t >= MF && t < NT - MF && xout < s.xlim;

        zw[0] = zu0[slot_new * ZW + cc];  // window: [0] new (z row j), [1] centre, [2] down
        vw[0] = zv[slot_new * ZW + cc];

        // ---- level 0 at row i: f(u0) and the energy monitor --------------------
        const double v = vw[1];
        const double2 u0c = zw[1];
        const double2 w0 = cf.kv(cf.dv(v), u0c, zu0[slot_cen * ZW + cc - 1], zu0[slot_cen * ZW + cc + 1],
                                 zw[2], zw[0]);
        const double n2 = fma(u0c.x, u0c.x, u0c.y * u0c.y);
        const double gx = fma(-cf.g() * n2, u0c.x, w0.x);
        const double gy = fma(-cf.g() * n2, u0c.y, w0.y);
        const double2 f = make_double2(gy, -gx);
        if (i >= MF && i < MF + s.R && t >= MF && t < NT - MF && xout < s.xlim) {
            const double vn = v * n2;
            const double sc = ISO ? c.cx : 1.0;
            monitor_add(acc, fma(sc, fma(u0c.x, w0.x, u0c.y * w0.y), -vn), sc * fma(u0c.x, w0.y, -u0c.y * w0.x), n2,
                        vn);
        }

        // ---- levels 1..MF: g_n at row i - n from g_{n-1} rows i-n-1, i-n, i-n+1 ----
        Chain ch{f, f, f, f};
        levels<1, PAR>(cf, j, ch);
        const double2 up = ch.up;
        const double2 g_low = ch.low, g_mid = ch.mid;

        if (out_ok) {
            // g_n(i - MF): n <= MF - 3 from the history rings, MF - 2 / MF - 1 / MF in registers
            double2 gout[MF + 1];
            gather<0>(gout);
            if (MF >= 2) gout[MF - 2] = g_low;
            gout[MF - 1] = g_mid;
            gout[MF] = up;
            const double2 u0o = ch.u0o;
            const size_t gi = at(a, xout, s.Y0 + yrel);
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                double rx = c.fco[q][MF] * gout[MF].x, ry = c.fco[q][MF] * gout[MF].y;
#pragma unroll
                for (int n = MF - 1; n >= 0; --n) {
                    rx = fma(c.fco[q][n], gout[n].x, rx);
                    ry = fma(c.fco[q][n], gout[n].y, ry);
                }
                uout[q][gi] = make_double2(u0o.x + rx, u0o.y + ry);
                March3<MF, NT, true, ISO, GHOST>::track(rmax, make_double2(rx, ry));
            }
        }
        // rotate the window: down <- centre <- new; advance the ring positions
        zw[2] = zw[1];
        zw[1] = zw[0];
        vw[2] = vw[1];
        vw[1] = vw[0];
        zs = zs + 1 == S ? 0 : zs + 1;
#pragma unroll
        for (int n = 0; n + 3 <= MF; ++n) hs[n] = hs[n] + 1 == depth(n) ? 0 : hs[n] + 1;
    }

    __device__ void run(const StepArgs& a, const SweepConsts& c, double2* const uout[3], int X0, int xlim,
                        int Y0, int R, unsigned& rmax, double* acc) {
        const Coef<ISO> cf{c};
        Seg s;
        s.X0 = X0;
        s.xlim = xlim;
        s.Y0 = Y0;
        s.R = R;
        s.nzrows = R + 2 * MF + 2;
        const int yz0 = Y0 - MF - 1, xz0 = s.X0 - MF - 1;
        if (GHOST) {
            s.next_off = static_cast<size_t>(yz0 + a.ghost) * a.pitch;
            const int last = a.pitch - 1;
            const int ca = xz0 + static_cast<int>(threadIdx.x) + a.ghost, cb = ca + NT;
            s.gxa = ca < last ? ca : last;
            s.gxb = cb < last ? cb : last;
        } else {
            s.next_row = wrap_index(yz0, a.ny);
            s.next_off = static_cast<size_t>(s.next_row) * a.nx;
            s.gxa = wrap_index(xz0 + static_cast<int>(threadIdx.x), a.nx);
            s.gxb = wrap_index(xz0 + static_cast<int>(threadIdx.x) + NT, a.nx);
        }
#pragma unroll
        for (int k = 0; k < P; ++k) issue_row(a, s, k, k);
        zs = 0;
#pragma unroll
        for (int n = 0; n + 3 <= MF; ++n) hs[n] = 0;
        const int jend = R + 2 * MF + 2;
        int j = 0;
        for (; j + 1 < jend; j += 2) {
            body<0>(a, cf, uout, s, j, rmax, acc);
            body<1>(a, cf, uout, s, j + 1, rmax, acc);
            if ((j & (kMonitorRows - 1)) == kMonitorRows - 2) monitor_flush(acc);  // every kMonitorRows rows
        }
        if (j < jend) body<0>(a, cf, uout, s, j, rmax, acc);
        cp_async_wait<0>();
        __syncthreads();
    }
};

// First sweep, v2: the MarchFirst algorithm (same per-site arithmetic, bit for bit)
// with its shared-memory rings laid out for cheap addressing.  v1 spends ~40 % of its
// instructions on ring-slot and row arithmetic (profiles/): here every ring row is
// NT double2 = 2 KiB (no halo columns: a band is 2 (MF + 1) columns wider than its
// output instead of 2 MF + 2 -- lanes 0 and NT-1 read a neighbour's stale column,
// which only reaches lanes the output masks), every ring depth is a power of two,
// and one slot offset per ring depth and iteration serves all levels through
// immediate offsets.  Depth of the history of g_n: 2 for the levels the output reads
// from registers, else the next power of two >= MF - n + 1 (the output reads g_n
// written MF - n iterations earlier).
template <int MF, int NT, bool ISO, bool GHOST>
struct MarchFirst2 {
    static_assert(MF >= 3 && MF <= 7, "first-sweep v2 depth");
    static constexpr int TX = NT - 2 * (MF + 1);  // output columns per band
    static constexpr int RB = NT * 16;            // bytes of a double2 ring row
    static_assert((RB & (RB - 1)) == 0, "power-of-two ring rows");
    static constexpr int SZ = 16;                 // z ring rows
    static constexpr int BACK = MF + 1;           // level MF reads z row j - (MF + 1)
    static constexpr int P = SZ - 1 - BACK;       // rows in flight
    static constexpr int PAD = 16;                // lanes 0 / NT-1 read 16 B beyond a row
    static constexpr int ZU = PAD;                // u0 ring: SZ rows of RB bytes
    static constexpr int ZV = ZU + SZ * RB;       // V ring: SZ rows of RB / 2 bytes
    static constexpr int H0 = ZV + SZ * RB / 2;   // g_n history rings
    __host__ __device__ static constexpr int pow2ceil(int x) { return x <= 1 ? 1 : 2 * pow2ceil((x + 1) / 2); }
    __host__ __device__ static constexpr int depth(int n) { return n >= MF - 2 ? 2 : pow2ceil(MF - n + 1); }
    __host__ __device__ static constexpr int hrow(int n) { return n == 0 ? 0 : hrow(n - 1) + depth(n - 1); }
    // + 128: the per-segment alignment shift of every ring (MB4_ALIGN_RING)
    static constexpr size_t bytes = static_cast<size_t>(H0) + static_cast<size_t>(hrow(MF)) * RB + PAD + 128;

    unsigned char* sm;   // dynamic shared memory, shifted per segment (MB4_ALIGN_RING)
    unsigned char* sm0;  // its unshifted base
    // own-column u0 / V of z rows j, j-1, ..., j-MF-1: level N reads row j-N-1, which
    // level N-1 read one iteration earlier, so the rows move down a register pipeline
    // (one shift per iteration) instead of being re-read from the ring per level
    // (30 shared-memory wavefronts per warp-row at MF = 6; the sweep is L1-bound)
#if MB4_FIRST_PQR
    // own-column u0 of z rows j, j-1, j-2 (level 0's stencil) and V of rows j, j-1;
    // the J coefficients (P, Q, R) of z rows j-2 .. j-MF-1 move down a register
    // pipeline (level N reads row j-N-1's, formed by level 0 N iterations earlier)
    static constexpr int NZW = 3;
    double2 zw[NZW];
    double vw[NZW];
    typename Coef<ISO>::PQR kw[MF + 2];  // kw[k]: z row j - k, k >= 2
#else
    static constexpr int NZW = MB4_FIRST_REGZ ? MF + 2 : 3;
    double2 zw[NZW];
    double vw[NZW];
#endif
    // own-column g_n of the last iterations: slot = iteration mod gring(n) (2 = parity)
    static constexpr bool U6pre = MB4_FIRST_UNROLL6 && MB4_FIRST_PQR && MF == 6;
    __host__ __device__ static constexpr int gring(int n) {
        return U6pre && MB4_FIRST_GREG >= 1 && n == MF - 3 ? 3
               : U6pre && ((MB4_FIRST_GREG >= 2 && n == MF - 4) || (MB4_FIRST_GREG >= 3 && n == MF - 5)) ? 6
                                                                                                         : 2;
    }
    double2 gp[MF][U6pre ? 6 : 2];
    // MB4_FIRST_UNROLL6: physical slots of the logical pipeline entries at iteration j, ROT = j mod 6
    static constexpr bool U6 = MB4_FIRST_UNROLL6 && MB4_FIRST_PQR && MF == 6;
    __host__ __device__ static constexpr int kix(int k, int rot) { return U6 ? (k - 2 + 12 - rot) % 6 + 2 : k; }
    __host__ __device__ static constexpr int zix(int k, int rot) { return U6 ? (k + 6 - rot) % 3 : k; }

#if MB4_BULK
    unsigned long long* bars;  // one mbarrier per z ring slot (bulk u0 row copies)
    __device__ static unsigned long long* ring_bars() {
        __shared__ unsigned long long b[SZ];
        return b;
    }
    __device__ MarchFirst2(unsigned char* smem) : sm(smem), sm0(smem), bars(ring_bars()) {}
#else
    __device__ MarchFirst2(unsigned char* smem) : sm(smem), sm0(smem) {}
#endif

    __device__ __forceinline__ static size_t at(const StepArgs& a, int x, int y) {
        if (GHOST) return static_cast<size_t>(y + a.ghost) * a.pitch + (x + a.ghost);
        return static_cast<size_t>(y) * a.nx + x;
    }
    template <class T>
    __device__ __forceinline__ static T& ref(unsigned char* p) { return *reinterpret_cast<T*>(p); }

    struct Seg {
        int X0, Y0, R, nzrows, gx, next_row;
        int xlim;
        int gx0;  // global column of lane 0 (wrapped; ghost-padded in GHOST mode)
        size_t next_off;
    };

    __device__ __forceinline__ void issue_row(const StepArgs& a, Seg& s, int k) {
        if (k < s.nzrows) {
            const size_t rowoff = s.next_off;
            if (GHOST) {
                s.next_off += a.pitch;
            } else if (++s.next_row == a.ny) {
                s.next_row = 0;
                s.next_off = 0;
            } else {
                s.next_off += a.nx;
            }
            const int slot = k & (SZ - 1);
            const size_t g = rowoff + s.gx;
#if MB4_BULK
            if (threadIdx.x == 0) {
                const int w = GHOST ? a.pitch : a.nx;
                mbar_arrive_expect_tx(&bars[slot], bulk_row_bytes<!GHOST>(s.gx0, NT, w));
                bulk_row<!GHOST>(reinterpret_cast<double2*>(sm + ZU + slot * RB), a.u0 + rowoff, s.gx0, NT, w,
                                 &bars[slot]);
            }
#else
            cp_async16(sm + ZU + slot * RB + threadIdx.x * 16, a.u0 + g);
#endif
            cp_async8(sm + ZV + slot * (RB / 2) + threadIdx.x * 8, a.V + g);
        }
        cp_async_commit();
    }

    struct Chain {
        double2 up, low, mid, u0o;
        double2 old3, old4, old5;  // g_{MF-3}, g_{MF-4}, g_{MF-5} of the output row (MB4_FIRST_GREG)
        double2 nl, nr;            // left / right neighbours of the level to come (MB4_FIRST_PREFETCH)
        double2 nl2, nr2;          // ... and of the one after it (MB4_FIRST_PREFETCH == 2)
    };
    // shared-memory row of g_n written in the previous iteration (this thread's column)
    template <int n, int PAR>
    __device__ __forceinline__ static unsigned char* prev_row(unsigned char* smt, int p8, int p4) {
        constexpr int D = depth(n);
        constexpr int HB = H0 + hrow(n) * RB;
        return smt + HB + (D == 2 ? (PAR ^ 1) * RB : (D == 8 ? p8 : p4));
    }

    // level N: g_N at row i - N from g_{N-1} rows i-N-1 (register), i-N (ring, previous
    // iteration), i-N+1 (this iteration, ch.up)
    template <int N, int ROT>
    __device__ __forceinline__ void levels(const Coef<ISO>& cf, unsigned char* smt, unsigned char* smv,
                                           int jrb, int o8, int p8, int o4, int p4, Chain& ch) {
        if constexpr (N <= MF) {
            constexpr int PAR = ROT & 1;
            constexpr int n = N - 1;
            constexpr int D = depth(n);
            constexpr int HB = H0 + hrow(n) * RB;
            const int so = D == 2 ? PAR * RB : (D == 8 ? o8 : o4);
            const int sp = D == 2 ? (PAR ^ 1) * RB : (D == 8 ? p8 : p4);
            unsigned char* crow = smt + HB + sp;  // g_n, iteration j - 1
            unsigned char* own = smt + HB + so;   // g_n, iteration j
            constexpr int RS = gring(n);
            constexpr int S_NOW = ROT % RS, S_M1 = (ROT + RS - 1) % RS, S_M2 = (ROT + RS - 2) % RS;
            const double2 gc = gp[n][S_M1];
            const double2 gd = gp[n][S_M2];
            // the output row's g_n: written MF - n iterations ago
            if constexpr (RS == 3) ch.old3 = gp[n][S_NOW];
            if constexpr (RS == 6 && n == MF - 4) ch.old4 = gp[n][(ROT + 6 - (MF - n)) % 6];
            if constexpr (RS == 6 && n == MF - 5) ch.old5 = gp[n][(ROT + 6 - (MF - n)) % 6];
#if MB4_FIRST_PQR
            double2 nl, nr;
            if constexpr (MB4_FIRST_PREFETCH) {
                nl = ch.nl;
                nr = ch.nr;
                constexpr int AHEAD = MB4_FIRST_PREFETCH;  // levels ahead
                if constexpr (AHEAD == 2) {
                    ch.nl = ch.nl2;
                    ch.nr = ch.nr2;
                }
                if constexpr (N + AHEAD <= MF) {
                    // g_{N + AHEAD - 1} of the previous iteration
                    unsigned char* nrow = prev_row<N + AHEAD - 1, PAR>(smt, p8, p4);
                    (AHEAD == 2 ? ch.nl2 : ch.nl) = ref<double2>(nrow - 16);
                    (AHEAD == 2 ? ch.nr2 : ch.nr) = ref<double2>(nrow + 16);
                }
            } else {
                nl = ref<double2>(crow - 16);
                nr = ref<double2>(crow + 16);
            }
            const double2 gn = cf.jt_pqr(kw[kix(N + 1, ROT)], gc, cf.nsum(nl, nr, gd, ch.up));
#else
            double2 u0n;
            double vn;
            if (N == 1 || MB4_FIRST_REGZ) {
                u0n = zw[N + 1];
                vn = vw[N + 1];
            } else {
                const int zo = (jrb - (N + 1) * RB) & (SZ * RB - 1);  // z row j - N - 1
                u0n = ref<double2>(smt + ZU + zo);
                vn = ref<double>(smv + ZV + (zo >> 1));
            }
            const double2 an = cf.kv(cf.dv(vn), gc, ref<double2>(crow - 16), ref<double2>(crow + 16), gd, ch.up);
            const double2 gn = cf.jt(gc, an, u0n);
            if (N == MF) ch.u0o = u0n;
#endif
            ref<double2>(own) = ch.up;
            gp[n][S_NOW] = ch.up;
            if (N == MF - 1) ch.low = gd;
            if (N == MF) ch.mid = gc;
            ch.up = gn;
            levels<N + 1, ROT>(cf, smt, smv, jrb, o8, p8, o4, p4, ch);
        }
    }

    // own-column g_n(i - MF), n <= MF - 3, written at iteration j - (MF - n)
    template <int N>
    __device__ __forceinline__ void gather(unsigned char* smt, int jrb, double2* gout) {
        if constexpr (N + 3 <= MF) {
            if constexpr (gring(N) == 2) {
                constexpr int D = depth(N);
                const int so = (jrb - (MF - N) * RB) & (D * RB - 1);
                gout[N] = ref<double2>(smt + H0 + hrow(N) * RB + so);
            }
            gather<N + 1>(smt, jrb, gout);
        }
    }

    template <int ROT>  // = j mod 6 (MB4_FIRST_UNROLL6) or j & 1
    __device__ __forceinline__ void body(const StepArgs& a, const Coef<ISO>& cf, double2* const uout[3], Seg& s,
                                         int j, unsigned& rmax, double* acc) {
        constexpr int Z0 = zix(0, ROT), Z1 = zix(1, ROT), Z2 = zix(2, ROT);
        const SweepConsts& c = cf.c;
        const int t = threadIdx.x, i = j - 2;
        unsigned char* smt = sm + t * 16;
        unsigned char* smv = sm + t * 8;
        cp_async_wait<P - 1>();
#if MB4_BULK
        mbar_wait(&bars[j & (SZ - 1)], (j / SZ) & 1);
#endif
        __syncthreads();
        issue_row(a, s, j + P);

        const int jrb = j * RB;
        const int zn = jrb & (SZ * RB - 1);         // z row j
        const int zc = (jrb - RB) & (SZ * RB - 1);  // z row j - 1
        const int o8 = jrb & (8 * RB - 1), p8 = (jrb - RB) & (8 * RB - 1);
        const int o4 = jrb & (4 * RB - 1), p4 = (jrb - RB) & (4 * RB - 1);

        const int yrel = i - 2 * MF;
        const int xout = s.X0 - MF - 1 + t;
        const bool lane_ok = t >= MF + 1 && t < NT - MF - 1 && xout < s.xlim;
        const bool out_ok = lane_ok && yrel >= 0 && yrel < s.R;

        zw[Z0] = ref<double2>(smt + ZU + zn);
        vw[Z0] = ref<double>(smv + ZV + (zn >> 1));
        // level 1's neighbours (g_0 of the previous iteration), loaded before level 0's arithmetic
        double2 pre_l, pre_r;
        if constexpr (MB4_FIRST_PREFETCH && MB4_FIRST_PQR) {
            unsigned char* nrow = prev_row<0, (ROT & 1)>(smt, p8, p4);
            pre_l = ref<double2>(nrow - 16);
            pre_r = ref<double2>(nrow + 16);
        }

        // ---- level 0 at row i: f(u0) and the energy monitor --------------------
        const double v = vw[Z1];
        const double2 u0c = zw[Z1];
        const double d0 = cf.dv(v);
        const double2 w0 = cf.kv(d0, u0c, ref<double2>(smt + ZU + zc - 16), ref<double2>(smt + ZU + zc + 16),
                                 zw[Z2], zw[Z0]);
        const double n2 = fma(u0c.x, u0c.x, u0c.y * u0c.y);
        const double gx = fma(-cf.g() * n2, u0c.x, w0.x);
        const double gy = fma(-cf.g() * n2, u0c.y, w0.y);
        const double2 f = make_double2(gy, -gx);
        if (lane_ok && i >= MF && i < MF + s.R) {
            const double vn = v * n2;
            const double sc = ISO ? c.cx : 1.0;
            monitor_add(acc, fma(sc, fma(u0c.x, w0.x, u0c.y * w0.y), -vn), sc * fma(u0c.x, w0.y, -u0c.y * w0.x), n2,
                        vn);
        }

        // ---- levels 1..MF --------------------------------------------------------
        Chain ch{f, f, f, f};
        if constexpr (MB4_FIRST_PREFETCH && MB4_FIRST_PQR) {
            ch.nl = pre_l;
            ch.nr = pre_r;
            if constexpr (MB4_FIRST_PREFETCH == 2 && MF >= 2) {
                unsigned char* nrow = prev_row<1, (ROT & 1)>(smt, p8, p4);
                ch.nl2 = ref<double2>(nrow - 16);
                ch.nr2 = ref<double2>(nrow + 16);
            }
        }
        levels<1, ROT>(cf, smt, smv, jrb, o8, p8, o4, p4, ch);

        if (out_ok) {
            double2 gout[MF + 1];
            gather<0>(smt, jrb, gout);
            if constexpr (gring(MF - 3) == 3) gout[MF - 3] = ch.old3;
            if constexpr (MF >= 4 && gring(MF >= 4 ? MF - 4 : 0) == 6) gout[MF - 4] = ch.old4;
            if constexpr (MF >= 5 && gring(MF >= 5 ? MF - 5 : 0) == 6) gout[MF - 5] = ch.old5;
            gout[MF - 2] = ch.low;
            gout[MF - 1] = ch.mid;
            gout[MF] = ch.up;
#if MB4_FIRST_PQR
            // u0 of the output row (z row j - MF - 1) from the ring (BACK = MF + 1 rows kept)
            const double2 u0o = ref<double2>(smt + ZU + ((jrb - (MF + 1) * RB) & (SZ * RB - 1)));
#else
            const double2 u0o = ch.u0o;
#endif
            const size_t gi = at(a, xout, s.Y0 + yrel);
#pragma unroll
            for (int q = 0; q < 3; ++q) {
                double rx = c.fco[q][MF] * gout[MF].x, ry = c.fco[q][MF] * gout[MF].y;
#pragma unroll
                for (int n = MF - 1; n >= 0; --n) {
                    rx = fma(c.fco[q][n], gout[n].x, rx);
                    ry = fma(c.fco[q][n], gout[n].y, ry);
                }
                uout[q][gi] = make_double2(u0o.x + rx, u0o.y + ry);
                March3<MF, NT, true, ISO, GHOST>::track(rmax, make_double2(rx, ry));
            }
        }
#if MB4_FIRST_PQR
        if constexpr (U6) {
            // the next iteration's entry 2 takes the slot of this iteration's oldest entry
            kw[kix(2, (ROT + 1) % 6)] = cf.pqr(d0, u0c);
        } else {
#pragma unroll
            for (int k = MF + 1; k > 2; --k) kw[k] = kw[k - 1];
            kw[2] = cf.pqr(d0, u0c);  // z row j - 1 becomes row j - 2 for level 1
        }
#endif
        if constexpr (!U6) {
#pragma unroll
            for (int k = NZW - 1; k > 0; --k) {
                zw[k] = zw[k - 1];
                vw[k] = vw[k - 1];
            }
        }
    }

    __device__ void run(const StepArgs& a, const SweepConsts& c, double2* const uout[3], int X0, int xlim,
                        int Y0, int R, unsigned& rmax, double* acc) {
        const Coef<ISO> cf{c};
        Seg s;
        s.X0 = X0;
        s.xlim = xlim;
        s.Y0 = Y0;
        s.R = R;
        s.nzrows = R + 2 * MF + 2;
        const int yz0 = Y0 - MF - 1, xz = X0 - MF - 1 + static_cast<int>(threadIdx.x);
        if (GHOST) {
            s.next_off = static_cast<size_t>(yz0 + a.ghost) * a.pitch;
            const int last = a.pitch - 1, ca = xz + a.ghost;
            s.gx = ca < last ? ca : last;
            s.gx0 = X0 - MF - 1 + a.ghost;
        } else {
            s.next_row = wrap_index(yz0, a.ny);
            s.next_off = static_cast<size_t>(s.next_row) * a.nx;
            s.gx = wrap_index(xz, a.nx);
            s.gx0 = wrap_index(X0 - MF - 1, a.nx);
        }
#if MB4_ALIGN_RING
        // lane t's u0 ring entry at the alignment of its global source modulo 128 B
        sm = sm0 + 16 * ((s.gx0 - static_cast<int>((smem_u32(sm0) + ZU) >> 4)) & 7);
#endif
#if MB4_BULK
        if (threadIdx.x == 0) {
#pragma unroll
            for (int q = 0; q < SZ; ++q) mbar_init(&bars[q], 1);
            mbar_fence_init();
        }
        __syncthreads();
#endif
#pragma unroll
        for (int k = 0; k < P; ++k) issue_row(a, s, k);
        const int jend = R + 2 * MF + 2;
        int j = 0;
        if constexpr (U6) {
            // (up to five iterations past the last row: they read the rings and store nothing)
            for (; j < jend; j += 6) {
                body<0>(a, cf, uout, s, j, rmax, acc);
                body<1>(a, cf, uout, s, j + 1, rmax, acc);
                body<2>(a, cf, uout, s, j + 2, rmax, acc);
                body<3>(a, cf, uout, s, j + 3, rmax, acc);
                body<4>(a, cf, uout, s, j + 4, rmax, acc);
                body<5>(a, cf, uout, s, j + 5, rmax, acc);
                if ((j / 6) & 1) monitor_flush(acc);  // every 12 rows
            }
        } else {
            for (; j + 1 < jend; j += 2) {
                body<0>(a, cf, uout, s, j, rmax, acc);
                body<1>(a, cf, uout, s, j + 1, rmax, acc);
                if ((j & (kMonitorRows - 1)) == kMonitorRows - 2) monitor_flush(acc);  // every kMonitorRows rows
            }
            if (j < jend) body<0>(a, cf, uout, s, j, rmax, acc);
        }
        cp_async_wait<0>();
        __syncthreads();
    }
};

// Split the band-rows of this launch's output rectangles evenly over the grid and
// march each segment (a run of rows of one band of one rectangle).
// Band-rows of this launch's output rectangles (the whole domain if it has none) in one flat
// order: rectangle by rectangle, band by band, row by row.
template <int TX>
struct BandRows {
    const StepArgs& a;
    int nr;
    __device__ explicit BandRows(const StepArgs& args) : a(args), nr(args.nrect > 0 ? args.nrect : 1) {}
    __device__ __forceinline__ int rect(int r, int k) const {
        if (a.nrect > 0) return a.rect[r][k];
        return k == 2 ? a.nx : (k == 3 ? a.ny : 0);
    }
    __device__ __forceinline__ long long total() const {
        long long t = 0;
        for (int r = 0; r < nr; ++r) t += static_cast<long long>((rect(r, 2) + TX - 1) / TX) * rect(r, 3);
        return t;
    }
    // march the band-rows [p0, p1): one segment per run of rows of one band
    template <class Run>
    __device__ __forceinline__ void march(long long p0, long long p1, const Run& run) const {
        for (long long pos = p0; pos < p1;) {
            long long base = 0;
            int r = 0;
            for (; r + 1 < nr; ++r) {
                const long long cnt = static_cast<long long>((rect(r, 2) + TX - 1) / TX) * rect(r, 3);
                if (pos < base + cnt) break;
                base += cnt;
            }
            const int h = rect(r, 3);
            const long long local = pos - base;
            const int band = static_cast<int>(local / h);
            const int row = static_cast<int>(local - static_cast<long long>(band) * h);
            const long long band_end = base + static_cast<long long>(band + 1) * h;
            const long long seg_end = band_end < p1 ? band_end : p1;
            run(rect(r, 0) + band * TX, rect(r, 0) + rect(r, 2), rect(r, 1) + row, static_cast<int>(seg_end - pos));
            pos = seg_end;
        }
    }
};

template <int TX, class Run>
__device__ __forceinline__ void for_segments(const StepArgs& a, const Run& run) {
    const BandRows<TX> rows(a);
    const long long total = rows.total();
    const long long G = gridDim.x;
    rows.march(total * blockIdx.x / G, total * (blockIdx.x + 1) / G, run);
}

// Chunk c of the guided split of `total` band-rows over a grid of G CTAs -> [p0, p1); false
// past the last chunk.  Round c / G has chunks of (total / G) >> (round + 1) rows, at least smin.
__host__ __device__ inline bool dyn_chunk(long long c, long long total, long long G, long long smin, long long& p0,
                                          long long& p1) {
    long long start = 0, sz = (total / G) * MB4_DYN_NUM / 8;
    for (;;) {
        if (sz <= smin) {
            sz = smin;
            break;
        }
        if (c < G) break;
        start += G * sz;
        c -= G;
        sz >>= 1;
    }
    p0 = start + c * sz;
    if (p0 >= total) return false;
    p1 = p0 + sz < total ? p0 + sz : total;
    return true;
}
inline long long dyn_chunk_count(long long total, long long G, long long smin) {
    long long n = 0, start = 0, sz = (total / G) * MB4_DYN_NUM / 8;
    while (sz > smin && start + G * sz <= total) {  // full rounds
        start += G * sz;
        n += G;
        sz >>= 1;
    }
    if (sz < smin) sz = smin;
    return n + (total - start + sz - 1) / sz;
}

// The same march over chunks of band-rows taken from the counter *ctr.
// Chunk c of round c / G (G = gridDim.x) has q >> (round + 1) rows, q = total / G, at least
// MB4_DYN_SMIN: a fixed map chunk -> rows, so only the CTA that computes a row varies.
template <int TX, class Run, class Done>
__device__ __forceinline__ void for_segments_dyn(const StepArgs& a, unsigned* ctr, const Run& run, const Done& done) {
    __shared__ unsigned s_chunk[2];
    const BandRows<TX> rows(a);
    const long long total = rows.total();
    int flip = 0;
    for (;;) {
        if (threadIdx.x == 0) s_chunk[flip] = atomicAdd(ctr, 1u);
        __syncthreads();
        const long long c = s_chunk[flip];
        flip ^= 1;
        long long p0, p1;
        if (!dyn_chunk(c, total, gridDim.x, MB4_DYN_SMIN, p0, p1)) break;
        rows.march(p0, p1, run);
        done(c);
    }
}

template <int M, int NT, bool FIRST, bool ISO, bool GHOST, bool DEF>
__device__ void sweep_all3(const StepArgs& a, const SweepConsts& c, unsigned char* smem,
                           const double2* const uin[3], double2* const uout[3],
                           unsigned& rmax, double* acc, int smask = 7, unsigned* work = nullptr) {
    if constexpr (FIRST && M >= 3 && M <= 7 && MB4_FIRST_V2) {
        using MFirst = MarchFirst2<M, NT, ISO, GHOST>;
        MFirst mf(smem);
        auto seg = [&](int X0, int xlim, int Y0, int R) { mf.run(a, c, uout, X0, xlim, Y0, R, rmax, acc); };
        if (MB4_DYN_SPLIT && MB4_DYN_FIRST && !GHOST && work) {
            for_segments_dyn<MFirst::TX>(a, work, seg, [&](long long chunk) {
                if (!a.want_obs) return;
                // this chunk's energy sums (compensated warp and block trees)
                monitor_flush(acc);
                block_csum_store<NT, kObsFields>(acc + kAccTot, acc + kAccCarry, a.obs_partial + chunk * kObsFields);
#pragma unroll
                for (int f = 0; f < kObsFields; ++f) acc[kAccTot + f] = acc[kAccCarry + f] = 0.0;
            });
        } else {
            for_segments<MFirst::TX>(a, seg);
        }
    } else if constexpr (FIRST && M >= 1) {
        using MFirst = MarchFirst<M, NT, ISO, GHOST>;
        MFirst mf(smem);
        for_segments<MFirst::TX>(a, [&](int X0, int xlim, int Y0, int R) {
            mf.run(a, c, uout, X0, xlim, Y0, R, rmax, acc);
        });
    } else {
        March3<M, NT, FIRST, ISO, GHOST, DEF> m(smem);
        // band-rows of this sweep's band width (TX depends on M)
        auto seg = [&](int X0, int xlim, int Y0, int R) { m.run(a, c, uin, uout, X0, xlim, Y0, R, rmax, acc, smask); };
        // (depth-2 sweeps run 2 CTAs per SM, which finish together: measured 2.5 % slower
        // with chunks at cfg4, so they keep the fixed shares)
        // (small lattices keep the fixed shares too: below ~4 minimum chunks per CTA the chunk
        // restarts and the idle CTAs cost more than the uneven finish -- cfg1's depth-1 sweeps
        // ran 0.023 instead of 0.0075 ms in chunks)
        if (MB4_DYN_SPLIT && !FIRST && M == 1 && work &&
            BandRows<Geom3<M, NT>::TX>(a).total() >= 4ll * MB4_DYN_SMIN * gridDim.x) {
            for_segments_dyn<Geom3<M, NT>::TX>(a, work, seg, [](long long) {});
        } else {
            for_segments<Geom3<M, NT>::TX>(a, seg);
        }
    }
}

// MF: Neumann depth of the first sweep of a step (whose level 0 is the cheap closed
// form, so a deeper first sweep costs little and saves one later sweep: measured
// 5 -> 4 sweeps/step at cfg5 for (MF, M) = (2, 1)); M: depth of the other sweeps.
// PH: 0 = all sweeps of the (sub)step in one launch; 1 = the first sweep only;
// 2 = the later sweeps, continuing from a PH = 1 launch (its residual in rmax[0]);
// 3 = the first sweep as a one-sweep launch with its status (sub-domain sweeps).
// (PH 1 is kept free of the status path: a runtime switch costs it registers.)
// the first sweep's kernel geometry (instantiated only where a first sweep runs)
template <int MF, int NT>
constexpr size_t first_sweep_bytes() {
    if constexpr (MF >= 3 && MF <= 7 && MB4_FIRST_V2) return MarchFirst2<MF, NT, true, false>::bytes;
    else if constexpr (MF >= 1) return MarchFirst<MF, NT, true, false>::bytes;
    else return Geom3<0, NT>::bytes;
}
template <int MF, int NT>
constexpr int first_sweep_tx() {
    if constexpr (MF >= 3 && MF <= 7 && MB4_FIRST_V2) return MarchFirst2<MF, NT, true, false>::TX;
    else if constexpr (MF >= 1) return MarchFirst<MF, NT, true, false>::TX;
    else return Geom3<0, NT>::TX;
}

template <int MF, int M, int NT, int PH = 0>
struct KGeom {
    // the first sweep runs MarchFirst (MF >= 1) or March3<0>; later sweeps March3<M>
    static constexpr size_t first_bytes = PH == 2 ? 0 : first_sweep_bytes<MF, (PH == 2 ? 128 : NT)>();
    static constexpr size_t later_bytes = Geom3<M, NT>::bytes;
    static constexpr size_t bytes = PH == 1 || PH == 3 ? first_bytes
                                    : PH == 2 ? later_bytes
                                              : (first_bytes > later_bytes ? first_bytes : later_bytes);
    static constexpr int MINB = NT >= 256 ? 1
                                : PH == 1 || PH == 3 ? 2
                                : PH == 2 ? (NT > 128 ? (M <= 1 ? 2 : 1) : (M <= 1 ? MB4_MINB_LATER : 2) * (128 / NT))
                                          : (M == 2 ? 2 : MB4_MINB_M1);
};

// The energy record of the step's entry state: the first sweep's partial sums (one per CTA,
// or per chunk of a chunked first sweep), each thread of block 0 a fixed strided subset, then
// the compensated warp and block trees -- a fixed order.
template <int NT>
__device__ __forceinline__ void reduce_obs(const StepArgs& a) {
    if (!a.want_obs || blockIdx.x != 0) return;
    double v[kObsFields] = {}, cv[kObsFields] = {};
    const int nb = a.obs_blocks > 0 ? a.obs_blocks : static_cast<int>(gridDim.x);
    for (int b = threadIdx.x; b < nb; b += NT) {
#pragma unroll
        for (int f = 0; f < kObsFields; ++f) two_sum_add(v[f], cv[f], a.obs_partial[b * kObsFields + f]);
    }
    if (a.obs_accumulate && threadIdx.x == 0) {
#pragma unroll
        for (int f = 0; f < kObsFields; ++f) two_sum_add(v[f], cv[f], a.status->obs[f]);
    }
    block_csum_store<NT, kObsFields>(v, cv, a.status->obs);
}

template <int MF, int M, int NT, bool ISO, bool GHOST, bool DEF, int PH>
__global__ void __launch_bounds__(NT, (KGeom<MF, M, NT, PH>::MINB))
mb4_step3_kernel(const StepArgs a, const __grid_constant__ SweepConsts c) {
    extern __shared__ __align__(16) unsigned char smem[];
    // a batched step after one that ended the batch: nothing to do (the flag was set by
    // an earlier launch on this stream, so every CTA of this grid reads the same value)
    // (one-sweep launches rotate through the chunk counters: this one resets the counter of the
    // launch kWorkCounters / 2 launches ahead -- also when it is skipped below)
    if (PH == 2 && a.work && a.work_idx >= 0 && blockIdx.x == 0 && threadIdx.x == 0)
        a.work[(a.work_idx + kWorkCounters / 2) % kWorkCounters] = 0u;
    if (a.batch_abort && *reinterpret_cast<volatile const int*>(a.batch_abort)) return;
    if (a.skip && *reinterpret_cast<volatile const int*>(a.skip)) return;
    cg::grid_group grid = cg::this_grid();
#ifdef MB4_CTA_TIMES
    const unsigned long long cta_t0 = global_timer_ns();
    if (PH == 1 && blockIdx.x == 0 && threadIdx.x == 0) {
        const unsigned long long n = g_cta_times[0][2][0]++;
        g_cta_times[0][1][n & 1] = cta_t0;
    }
#endif
    double acc[kAccSize] = {};  // energy sums, max |u0|^2, carries (monitor_add)
#if MB4_CONSTS_IN_SMEM
    // M = 2: scheme / step constants as a shared-memory broadcast table (LDS)
    // instead of the constant bank (LDCU + uniform-register shuffling), which
    // relieves the register pressure of the two-level kernel (measured: +2 %);
    // for M <= 1 the constant bank is faster (measured: +18 %).
    // (not in first-sweep launches: their shared-memory rings need every byte)
    const SweepConsts* cptr = &c;
    if constexpr (M == 2 && PH != 1 && PH != 3) {
        __shared__ __align__(16) SweepConsts csm;
        const double* src = reinterpret_cast<const double*>(&c);
        double* dst = reinterpret_cast<double*>(&csm);
        for (int q = threadIdx.x; q < static_cast<int>(sizeof(SweepConsts) / sizeof(double)); q += NT) dst[q] = src[q];
        __syncthreads();
        cptr = &csm;
    }
    const SweepConsts& cc = *cptr;
#else
    const SweepConsts& cc = c;
#endif
#ifdef MB4_POISON_SMEM
    // debug builds: stale shared memory must never reach an output
    for (size_t q = threadIdx.x; q < KGeom<MF, M, NT, PH>::bytes / 8; q += NT)
        reinterpret_cast<unsigned long long*>(smem)[q] = MB4_POISON_SMEM;
    __syncthreads();
#endif
    // the later-sweep launch of this step takes its chunks from these counters
    // (counter 0 is the first sweep's own: the later-sweep launch of the previous step reset it)
    if (PH == 1 && a.work && a.work_idx < 0 && blockIdx.x == 0)
        for (int q = 1 + threadIdx.x; q < kWorkCounters; q += NT) a.work[q] = 0u;
    if (PH == 2 && a.work && a.work_idx < 0 && blockIdx.x == 0 && threadIdx.x == 0) a.work[0] = 0u;
    // The later-sweep launch of a split step sums the first-sweep launch's energy partials
    // before its sweeps, not after them (a serial pass of ~17 us at cfg5 by one warp of
    // block 0: the chunked sweeps give its rows to the other CTAs meanwhile).
    const bool obs_early = PH == 2 && a.sweep0 == 0;
    if (obs_early) reduce_obs<NT>(a);
    int pass = 0;  // sweep passes of this launch (one chunk counter each)
    int sweeps = 0, set = 0, converged = 0, redone = 0;
    bool redo = false;  // this pass repeats the missed speculative sweep with all stages
    double rlast = 0.0;
    int s_begin = 0;
    if (PH != 2) {
        if (blockIdx.x == 0 && threadIdx.x == 0) a.status->t[0] = global_timer_ns();
    } else if (a.sweep0 == 0) {
        // continue the first-sweep launch of this (sub)step: sweep 0 left its residual
        // in rmax[0]; the same tests as after sweep 0 of the single launch.  (Sub-domain
        // sweeps launch one sweep at a time: sweep0 > 0, nothing to continue.)
        if (blockIdx.x == 0 && threadIdx.x == 0) a.status->t[1] = global_timer_ns();
        rlast = __longlong_as_double(static_cast<long long>(__ldcg(&a.rmax[0])));
        sweeps = 1;
        s_begin = 1;
        if (!isfinite(rlast)) {
            s_begin = a.max_iters;
        } else if (stage_converged(rlast, 0.0, 0, a.eps)) {
            converged = 1;
            s_begin = a.max_iters;
        }
    }
    for (int s = s_begin; s < a.max_iters; ++s) {
        const int sg = s + a.sweep0;  // global sweep index within the (sub)step
        const int out = sg & 1;
        double2* const uout[3] = {a.U[out][0], a.U[out][1], a.U[out][2]};
        unsigned rmax = 0u;
        if (PH == 1 || PH == 3 || (PH == 0 && sg == 0)) {
            const double2* const uin[3] = {a.u0, a.u0, a.u0};
            // (chunked first sweep of a split step: counter 0, one set of partials per chunk)
            unsigned* const fwork = PH == 1 && a.work && a.dyn_first ? a.work : nullptr;
            if constexpr (PH != 2)  // (not instantiated for the later-sweep kernel)
                sweep_all3<MF, NT, true, ISO, GHOST, DEF>(a, cc, smem, uin, uout, rmax, acc, 7, fwork);
            if (a.want_obs) {
                // compensated warp and block trees; one rounding per block partial
                if (!(MB4_DYN_SPLIT && MB4_DYN_FIRST && MF >= 3 && MF <= 7 && MB4_FIRST_V2 && fwork)) {
                    monitor_flush(acc);
                    block_csum_store<NT, kObsFields>(acc + kAccTot, acc + kAccCarry,
                                                     a.obs_partial + blockIdx.x * kObsFields);
                }
                // max |u0|^2 of the entry state (non-negative: its bits order as integers)
                double mx = acc[kAccMax];
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
                if ((threadIdx.x & 31) == 0 && mx > 0.0)
                    atomicMax(&a.rmax[a.max_iters], static_cast<unsigned long long>(__double_as_longlong(mx)));
            }
        } else if constexpr (PH != 1 && PH != 3) {
            // Speculative final sweep (sg == spec_sweep, predicted by the host from the
            // previous step): only U3 -- the step result -- is stored, saving 32 of the
            // 120 B/site.  If it does not converge, it is redone below with all stages
            // (same inputs, same arithmetic, so the result is independent of the guess).
            const int in = 1 - out;
            const double2* const uin[3] = {a.U[in][0], a.U[in][1], a.U[in][2]};
            unsigned* const work = PH != 2 || !a.work ? nullptr
                                   : a.work_idx >= 0           ? a.work + a.work_idx  // (one-sweep launches)
                                   : pass + 1 < kWorkCounters  ? a.work + 1 + pass
                                                               : nullptr;
            ++pass;
            sweep_all3<M, NT, false, ISO, GHOST, DEF>(a, cc, smem, uin, uout, rmax, acc,
                                                       sg == a.spec_sweep && !redo ? 4 : 7, work);
        }
#ifdef MB4_CTA_TIMES
        __syncthreads();
        if (threadIdx.x == 0 && blockIdx.x < 2048) {
            unsigned smid;
            asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
            g_cta_times[PH][blockIdx.x][0] = cta_t0;
            g_cta_times[PH][blockIdx.x][1] = global_timer_ns();
            g_cta_times[PH][blockIdx.x][2] = smid;
        }
#endif
        if constexpr (PH == 1) {  // the later-sweep launch takes it from here
            block_max_to(rmax ? ((static_cast<unsigned long long>(rmax) << 32) | 0xFFFFFFFFull) : 0ull, &a.rmax[0]);
#ifdef MB4_CTA_TIMES
            if (threadIdx.x == 0 && blockIdx.x < 2048) g_cta_times[PH][blockIdx.x][3] = global_timer_ns();
#endif
            return;
        }
        if (redo) {  // same residual as the speculative pass: no new test
            redo = false;
            ++redone;
            grid.sync();
            continue;
        }
        block_max_to(rmax ? ((static_cast<unsigned long long>(rmax) << 32) | 0xFFFFFFFFull) : 0ull, &a.rmax[s]);
        grid.sync();
        if (blockIdx.x == 0 && threadIdx.x == 0 && s < StepStatus::kMaxTimed)
            a.status->t[s + 1] = global_timer_ns();
        const unsigned long long bits = __ldcg(&a.rmax[s]);
        const double rprev = rlast;
        rlast = __longlong_as_double(static_cast<long long>(bits));
        sweeps = sg + 1;
        set = out;
        if (!isfinite(rlast)) break;
        if (stage_converged(rlast, rprev, sg, a.eps)) {
            converged = 1;
            break;
        }
        if (sg > 0 && sg == a.spec_sweep && s + 1 < a.max_iters) {
            redo = true;
            --s;  // repeat sweep sg with all stages stored
        }
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        a.status->sweeps = sweeps;
        a.status->set = set;
        a.status->converged = converged;
        a.status->redone = redone;
        // a non-finite residual (NaN update somewhere) is reported as +inf: the MAX
        // all-reduce of a decomposed lattice (fmax) would drop a NaN, never an inf
        a.status->rlast = isfinite(rlast) ? rlast : __longlong_as_double(0x7FF0000000000000ll);
        const double amax2 = a.want_obs ? __longlong_as_double(static_cast<long long>(__ldcg(&a.rmax[a.max_iters]))) : 0.0;
        a.status->amax2 = amax2;
        if (a.batch_abort &&
            (!converged || sweeps != a.expect_sweeps || (a.switch_sweeps > 0 && sweeps >= a.switch_sweeps) ||
             !(amax2 >= a.amax2_lo && amax2 <= a.amax2_hi)))
            *a.batch_abort = 1;
    }
    if (!obs_early) reduce_obs<NT>(a);
#ifdef MB4_CTA_TIMES
    if (threadIdx.x == 0 && blockIdx.x < 2048) g_cta_times[PH][blockIdx.x][3] = global_timer_ns();
#endif
}

template <int MF, int M, int NT, bool ISO, bool GHOST, bool DEF, int PH = 0>
struct Launcher3 {
    static int grid_size(int device) {
        static std::atomic<int> cached[64];  // per device (0 = not yet computed)
        if (device >= 0 && device < 64 && cached[device].load(std::memory_order_acquire))
            return cached[device].load(std::memory_order_acquire);
        const size_t smem = KGeom<MF, M, NT, PH>::bytes;
        cudaFuncSetAttribute(mb4_step3_kernel<MF, M, NT, ISO, GHOST, DEF, PH>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
        int per_sm = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, mb4_step3_kernel<MF, M, NT, ISO, GHOST, DEF, PH>, NT,
                                                      smem);
        int sms = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
        const int g = per_sm * sms;
        if (device >= 0 && device < 64) cached[device].store(g, std::memory_order_release);
        return g;
    }

    // output columns per band of this launch's sweeps (the smaller one if it runs both kinds)
    static constexpr int TX_FIRST = first_sweep_tx<MF, (PH == 2 ? 128 : NT)>();
    static constexpr int TX_LATER = Geom3<M, NT>::TX;
    static constexpr int TXK = PH == 2 ? TX_LATER : PH == 0 && TX_LATER < TX_FIRST ? TX_LATER : TX_FIRST;
    static constexpr long long kMinRowsPerCta = MB4_MIN_ROWS_PER_CTA;

    // CTAs of a launch: the co-resident grid, capped by grid_cap and, for small lattices, by
    // the band-rows to march (no CTAs that only take part in the grid barriers)
    static int launch_grid(const StepArgs& a, int device) {
        int grid = grid_size(device);
#ifdef MB4_CTA_TIMES
        // profiling builds: MB4_DEBUG_GRID_CAP=<CTAs> (e.g. one CTA per SM: a warp's own stalls)
        if (const char* e = std::getenv("MB4_DEBUG_GRID_CAP")) {
            const int cap = std::atoi(e);
            if (PH == 2 && cap > 0 && cap < grid) grid = cap;
        }
#endif
        if (a.grid_cap > 0 && a.grid_cap < grid) {
            grid = a.grid_cap;
        } else if (a.grid_cap < 0) {  // leave -grid_cap SMs to concurrent kernels (NCCL)
            int sms = 0;
            cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
            const int keep = sms + a.grid_cap > 0 ? sms + a.grid_cap : 1;
            grid = sms > 0 ? grid / sms * keep : grid;
        }
        long long total = 0;  // band-rows, as for_segments counts them
        const int nr = a.nrect > 0 ? a.nrect : 1;
        for (int r = 0; r < nr; ++r) {
            const long long w = a.nrect > 0 ? a.rect[r][2] : a.nx, h = a.nrect > 0 ? a.rect[r][3] : a.ny;
            total += (w + TXK - 1) / TXK * h;
        }
        const long long want = (total + kMinRowsPerCta - 1) / kMinRowsPerCta;
        if (want < grid) grid = want > 0 ? static_cast<int>(want) : 1;
        return grid;
    }

    static cudaError_t launch(StepArgs a, const SweepConsts& c, int device, cudaStream_t s) {
        const int grid = launch_grid(a, device);
        if (grid <= 0) return cudaErrorLaunchOutOfResources;
        void* params[] = {&a, const_cast<SweepConsts*>(&c)};
        return cudaLaunchCooperativeKernel(reinterpret_cast<void*>(mb4_step3_kernel<MF, M, NT, ISO, GHOST, DEF, PH>),
                                           dim3(grid), dim3(NT), params, KGeom<MF, M, NT, PH>::bytes, s);
    }
};

// the split pair: first sweep (PH 1), then the later sweeps (PH 2) on the same stream
template <int MF, int M, int NT, bool ISO, bool DEF>
cudaError_t launch_split(StepArgs a, const SweepConsts& c, int device, cudaStream_t s) {
    a.obs_blocks = Launcher3<MF, M, MB4_NT_FIRST, ISO, false, DEF, 1>::launch_grid(a, device);
    a.dyn_first = 0;
    if constexpr (MB4_DYN_SPLIT && MB4_DYN_FIRST && MF >= 3 && MF <= 7 && MB4_FIRST_V2) {
        if (a.work) {
            // one set of energy partials per chunk of the first sweep, if the buffer holds them
            constexpr int TXF = first_sweep_tx<MF, MB4_NT_FIRST>();
            const long long total = static_cast<long long>((a.nx + TXF - 1) / TXF) * a.ny;
            const long long chunks = dyn_chunk_count(total, a.obs_blocks, MB4_DYN_SMIN);
            if (chunks <= a.obs_cap) {
                a.dyn_first = 1;
                a.obs_blocks = static_cast<int>(chunks);
            }
        }
    }
    const cudaError_t e = Launcher3<MF, M, MB4_NT_FIRST, ISO, false, DEF, 1>::launch(a, c, device, s);
    if (e != cudaSuccess) return e;
    return Launcher3<MF, M, MB4_NT_LATER, ISO, false, DEF, 2>::launch(a, c, device, s);
}

template <int MF, int M>
cudaError_t dispatch3(const StepArgs& a0, const SweepConsts& c, int device, cudaStream_t s) {
    StepArgs a = a0;
    // chunk counters: only the split pair of a whole domain (its first-sweep launch zeroes them)
    const bool split = MB4_SPLIT && MF >= 4 && a.ghost == 0 && a.sweep0 == 0 && a.max_iters > 1;
    // ... and the one-sweep later-sweep launches of a sub-domain (a rotating counter, work_idx)
    const bool region = MB4_SPLIT && MF >= 4 && a.ghost > 0 && a.max_iters == 1 && a.sweep0 > 0 && a.work_idx >= 0;
    if (!(split && a.nrect == 0 && a.work_idx < 0) && !region) a.work = nullptr;
    if constexpr (MB4_SPLIT && MF >= 4) {
        if (a.ghost == 0 && a.sweep0 == 0 && a.max_iters > 1) {
            if (c.iso && c.def) return launch_split<MF, M, MB4_NT, true, true>(a, c, device, s);
            return c.iso ? launch_split<MF, M, MB4_NT, true, false>(a, c, device, s)
                         : launch_split<MF, M, MB4_NT, false, false>(a, c, device, s);
        }
    }
    if constexpr (MB4_SPLIT && MF >= 4) {
        // sub-domain sweeps (one sweep per launch): the first / later sweep kernels with
        // their own register and shared-memory footprints
        if (a.ghost > 0 && a.max_iters == 1) {
            if (a.sweep0 == 0) {
                if (c.iso && c.def) return Launcher3<MF, M, MB4_NT_FIRST, true, true, true, 3>::launch(a, c, device, s);
                return c.iso ? Launcher3<MF, M, MB4_NT_FIRST, true, true, false, 3>::launch(a, c, device, s)
                             : Launcher3<MF, M, MB4_NT_FIRST, false, true, false, 3>::launch(a, c, device, s);
            }
            if (c.iso && c.def) return Launcher3<MF, M, MB4_NT_LATER, true, true, true, 2>::launch(a, c, device, s);
            return c.iso ? Launcher3<MF, M, MB4_NT_LATER, true, true, false, 2>::launch(a, c, device, s)
                         : Launcher3<MF, M, MB4_NT_LATER, false, true, false, 2>::launch(a, c, device, s);
        }
    }
    // compile-time scheme tables for the (common) isotropic default-scheme case
    if (a.ghost > 0) {
        if (c.iso && c.def) return Launcher3<MF, M, MB4_NT, true, true, true>::launch(a, c, device, s);
        return c.iso ? Launcher3<MF, M, MB4_NT, true, true, false>::launch(a, c, device, s)
                     : Launcher3<MF, M, MB4_NT, false, true, false>::launch(a, c, device, s);
    }
    if (c.iso && c.def) return Launcher3<MF, M, MB4_NT, true, false, true>::launch(a, c, device, s);
    return c.iso ? Launcher3<MF, M, MB4_NT, true, false, false>::launch(a, c, device, s)
                 : Launcher3<MF, M, MB4_NT, false, false, false>::launch(a, c, device, s);
}

template <int MF, int M>
int grid3(int device) {
    int g = 0;
    const int v[6] = {Launcher3<MF, M, MB4_NT, true, false, false>::grid_size(device),
                      Launcher3<MF, M, MB4_NT, false, false, false>::grid_size(device),
                      Launcher3<MF, M, MB4_NT, true, true, false>::grid_size(device),
                      Launcher3<MF, M, MB4_NT, false, true, false>::grid_size(device),
                      Launcher3<MF, M, MB4_NT, true, false, true>::grid_size(device),
                      Launcher3<MF, M, MB4_NT, true, true, true>::grid_size(device)};
    for (int x : v) g = x > g ? x : g;
    if constexpr (MB4_SPLIT && MF >= 4) {
        const int w[6] = {Launcher3<MF, M, MB4_NT_FIRST, true, false, false, 1>::grid_size(device),
                          Launcher3<MF, M, MB4_NT_FIRST, false, false, false, 1>::grid_size(device),
                          Launcher3<MF, M, MB4_NT_FIRST, true, false, true, 1>::grid_size(device),
                          Launcher3<MF, M, MB4_NT_LATER, true, false, false, 2>::grid_size(device),
                          Launcher3<MF, M, MB4_NT_LATER, false, false, false, 2>::grid_size(device),
                          Launcher3<MF, M, MB4_NT_LATER, true, false, true, 2>::grid_size(device)};
        for (int x : w) g = x > g ? x : g;
        const int wg[6] = {Launcher3<MF, M, MB4_NT_FIRST, true, true, false, 3>::grid_size(device),
                           Launcher3<MF, M, MB4_NT_FIRST, false, true, false, 3>::grid_size(device),
                           Launcher3<MF, M, MB4_NT_FIRST, true, true, true, 3>::grid_size(device),
                           Launcher3<MF, M, MB4_NT_LATER, true, true, false, 2>::grid_size(device),
                           Launcher3<MF, M, MB4_NT_LATER, false, true, false, 2>::grid_size(device),
                           Launcher3<MF, M, MB4_NT_LATER, true, true, true, 2>::grid_size(device)};
        for (int x : wg) g = x > g ? x : g;
    }
    return g;
}

}  // namespace

// (first-sweep depth, later-sweep depth) pairs with a compiled kernel
#ifdef MB4_QUICK_PAIRS  // register / SASS checks of the production pair only (not a usable library)
#define MB4_MARCH2_PAIRS(X) X(6, 1) X(6, 2)
#else
#define MB4_MARCH2_PAIRS(X) X(0, 0) X(1, 1) X(2, 2) X(2, 0) X(2, 1) X(3, 1) X(4, 1) X(5, 1) X(6, 1) X(4, 2) X(5, 2) X(6, 2) X(6, 0)
#endif

// The chunk map of the chunked later sweeps, for the host-side tests (every band-row belongs
// to exactly one chunk): chunk c of `total` band-rows over a grid of G CTAs.
bool march2_chunk_range(long long c, long long total, long long G, long long* p0, long long* p1) {
    return dyn_chunk(c, total, G, MB4_DYN_SMIN, *p0, *p1);
}
long long march2_chunk_count(long long total, long long G) { return dyn_chunk_count(total, G, MB4_DYN_SMIN); }

int march2_launches(int mf, int ghost, int sweep0, int max_iters) {
    return MB4_SPLIT && mf >= 4 && ghost == 0 && sweep0 == 0 && max_iters > 1 ? 2 : 1;
}

bool march2_supported(int mf, int m) {
#define MB4_PAIR_EQ(F, N) if (mf == F && m == N) return true;
    MB4_MARCH2_PAIRS(MB4_PAIR_EQ)
#undef MB4_PAIR_EQ
    return false;
}

cudaError_t launch_step_march2(int mf, int m, int nx, int ny, const double2* u0, const double* V,
                               double2* const U[2][3], unsigned long long* rmax,
                               double* obs_partial, void* status, int max_iters, double eps,
                               int want_obs, const SweepConsts& c, int device, cudaStream_t s,
                               int ghost, int sweep0, int spec_sweep, int nrect, const int (*rects)[4],
                               int obs_accumulate, int grid_cap, const BatchCtl* batch, int pitch, unsigned* work,
                               int obs_cap, int work_idx) {
    StepArgs a{};
    a.work = work;
    a.work_idx = work && work_idx >= 0 ? work_idx % kWorkCounters : -1;
    a.obs_cap = obs_cap;
    if (batch) {
        a.batch_abort = batch->abort;
        a.expect_sweeps = batch->expect_sweeps;
        a.switch_sweeps = batch->switch_sweeps;
        a.amax2_lo = batch->amax2_lo;
        a.amax2_hi = batch->amax2_hi;
        a.skip = batch->skip;
    }
    a.nrect = nrect;
    for (int r = 0; r < nrect && r < 4; ++r)
        for (int k = 0; k < 4; ++k) a.rect[r][k] = rects[r][k];
    a.obs_accumulate = obs_accumulate;
    a.grid_cap = grid_cap;
    a.nx = nx;
    a.ny = ny;
    a.u0 = u0;
    a.V = V;
    for (int b = 0; b < 2; ++b)
        for (int q = 0; q < 3; ++q) a.U[b][q] = U[b][q];
    a.rmax = rmax;
    a.obs_partial = obs_partial;
    a.status = static_cast<StepStatus*>(status);
    a.max_iters = max_iters;
    a.eps = eps;
    a.want_obs = want_obs;
    a.ghost = ghost;
    a.pitch = pitch > 0 ? pitch : nx + 2 * ghost;  // (sub-domain contexts pad it to 8 sites)
    a.sweep0 = sweep0;
    a.spec_sweep = spec_sweep;
#ifdef MB4_DEBUG_FIRST_ONLY
    a.max_iters = 1;  // profiling builds: the first sweep alone
#endif
#define MB4_PAIR_LAUNCH(F, N) if (mf == F && m == N) return dispatch3<F, N>(a, c, device, s);
    MB4_MARCH2_PAIRS(MB4_PAIR_LAUNCH)
#undef MB4_PAIR_LAUNCH
    return cudaErrorInvalidValue;
}

int march2_band_width(int mf, int m, bool first) {
    // output columns per band of the sub-domain sweep kernels (MB4_NT_FIRST / MB4_NT_LATER wide)
    if (!first) {
        if (m == 1) return Geom3<1, MB4_NT_LATER>::TX;
        return m == 2 ? Geom3<2, MB4_NT_LATER>::TX : Geom3<0, MB4_NT_LATER>::TX;
    }
    switch (mf) {
        case 6: return first_sweep_tx<6, MB4_NT_FIRST>();
        case 5: return first_sweep_tx<5, MB4_NT_FIRST>();
        case 4: return first_sweep_tx<4, MB4_NT_FIRST>();
        default: return 0;
    }
}

int march2_grid_size(int mf, int m, int device) {
#define MB4_PAIR_GRID(F, N) if (mf == F && m == N) return grid3<F, N>(device);
    MB4_MARCH2_PAIRS(MB4_PAIR_GRID)
#undef MB4_PAIR_GRID
    return 0;
}

}  // namespace mb4cu
