// sm_100a kernels of the B200 H^2-MMP.
//
// FP64 has no tcgen05 kind on sm_100a: the tensor path for
// double is mma.sync m8n8k4 f64 -> DMMA.8x8x4, measured at 37.1 TFLOP/s on the
// pool's B200 (profiles/FP64_PEAKS.json).  Every product of the pipeline goes
// through ONE segmented batched small-GEMM kernel (seg_gemm): for each output
// block t it accumulates sum_e op(L_e) * op(R_e) over a CSR segment of entries
// (one CTA per output tile, fixed entry order -> deterministic, no atomics),
// which covers the per-block products, the Gram sums and the triple sums of
// the reference's four product cases.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace h2b {

enum OpCode : int { OP_N = 0, OP_T = 1, OP_H = 2, OP_C = 3 };  // none, transpose, adjoint, conjugate

struct SegGroup {
  const double* L;
  long long Ls, Loff;  // element stride between matrices, element offset (view)
  int Lld, opL;
  const double* R;
  long long Rs, Roff;
  int Rld, opR;
  int K;               // inner dimension (padded)
  const int* ptr;      // CSR over outputs, or nullptr: exactly one entry per output
  const int* li;       // entry (or per-output, if ptr==nullptr) left index; nullptr = output index
  const int* ri;
  // chunked operand storage (the merged 2x2 blocks of the largest configurations): matrix l
  // lives at Lch[l >> Lsh] + Ls * (l & (2^Lsh - 1)) instead of L + Ls * l (nullptr: contiguous)
  const double* const* Lch;
  const double* const* Rch;
  int Lsh, Rsh;
};

constexpr int kMaxGroups = 4;

struct SegParams {
  double* out;
  long long Os, Ooff;
  int Old;
  const int* omap;     // storage index of output t (nullptr = t)
  int M, N;            // output dims (padded)
  int n_out;
  int accumulate;      // out (+)= sum (bit 0); bit 1: prefetch the output tile to L2 first
  int sym;             // Hermitian output (Gram): only tiles m0 >= n0 are computed, mirrored
  int ngroups;
  // optional quadrant scatter (children targets written straight into their
  // parents' merged 2x2 blocks): output t -> block oquad[t] >> 2, quadrant
  // q = oquad[t] & 3 at row offset (q >> 1) * qm and column offset (q & 1) * qn
  const int* oquad;
  int qm, qn;
  // chunked output storage (see SegGroup::Lch): output block b at och[b >> osh] + Os * (b & mask)
  double* const* och;
  int osh;
  SegGroup g[kMaxGroups];
};

// address of output t's block (W = scalars per element)
__device__ __forceinline__ double* seg_out_ptr(const SegParams& p, int t, int W) {
  long long blk, extra = 0;
  if (p.oquad) {
    const int v = p.oquad[t];
    const int q = v & 3;
    blk = v >> 2;
    extra = (q >> 1) * p.qm + (long long)((q & 1) * p.qn) * p.Old;
  } else {
    blk = p.omap ? p.omap[t] : t;
  }
  if (p.och)
    return p.och[blk >> p.osh] + (p.Os * (blk & ((1LL << p.osh) - 1)) + p.Ooff + extra) * W;
  return p.out + (p.Os * blk + p.Ooff + extra) * W;
}

// ---------------------------------------------------------------------------
// scalar helpers (complex values are interleaved re, im)
template <bool CPLX>
struct Sc;
template <>
struct Sc<false> {
  static constexpr int W = 1;
};
template <>
struct Sc<true> {
  static constexpr int W = 2;
};

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// ---------------------------------------------------------------------------
// seg_gemm pipeline configuration: STAGES-deep cp.async pipeline of raw (untransformed) tiles.
// Each operand chunk is copied in its native layout ([k][m] for op N/C of a
// column-major L, [m][k] for op T/H; mirrored for R), 16 B per cp.async with
// zero fill past the padded bounds; the fragment loads pick the addressing of
// the layout (both conflict-free with a +4 double pad).  No register staging:
// fewer registers, more CTAs per SM, and STAGES-1 chunks in flight hide the
// L2/HBM latency of the next entry's operands.
template <int TM, int TN, bool CPLX, int KC_ = 16, int ST_ = 3, int WM_ = 2, int WN_ = 2>
struct Seg2Cfg {
  static constexpr int WM = WM_, WN = WN_, NT = 32 * WM_ * WN_;
  static constexpr int W = CPLX ? 2 : 1;
  static constexpr int KC = CPLX ? KC_ / 2 : KC_;
  static constexpr int STAGES = ST_;
  static constexpr int LKM = KC * (TM + 4), LMK = TM * (KC + 4);
  static constexpr int RKN = KC * (TN + 4), RNK = TN * (KC + 4);
  static constexpr int LSZ = (LKM > LMK ? LKM : LMK) * W;
  static constexpr int RSZ = (RKN > RNK ? RKN : RNK) * W;
  static constexpr int STAGE = LSZ + RSZ;  // doubles
  static constexpr int SMEM = STAGES * STAGE * 8;
  static constexpr int FM = TM / WM / 8, FN = TN / WN / 8;
};

__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool ok) {
  const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  const int n = ok ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(n));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// ---------------------------------------------------------------------------
// seg_gemm v3: the v2 pipeline with the per-chunk integer work taken out of the
// loop (profiles/r01/ncu_seg_gemm2_8x4_source.txt: v2 issued ~10 integer /
// branch instructions per DMMA — cursor walk, copy-index math, runtime layout
// selects — and the warp scheduler, not the tensor pipe, was the limit).
//  * every inner dimension is a multiple of the k-chunk (all padded dims are
//    multiples of 8), so a chunk never straddles an entry and needs no k test;
//  * rows past M / columns past N are not copied at all: they only feed output
//    rows / columns the epilogue discards, so no zero fill is needed;
//  * the copy sources are per-thread pointers set once per entry and bumped by
//    a constant per chunk;
//  * the fragment loads run in a body specialised per operand layout (N/C vs
//    T/H on each side), selected once per group, with immediate smem offsets.
// G3 (complex only): 3 real products per complex MAC (Gauss): with s_a = a + i-part, d_b = bi - b,
// s_b = b + bi: P = sum s_a b, R = sum a d_b, Q = sum ai s_b; Re = P - Q, Im = P + R
// (3 DMMAs instead of 4, one more accumulator set).
template <int TM, int TN, bool CPLX, int KC_ = 8, int ST_ = 4, int WM_ = 2, int WN_ = 2, bool G3 = false>
__global__ void __launch_bounds__(32 * WM_ * WN_) seg_gemm3_kernel(const SegParams p) {
  using C = Seg2Cfg<TM, TN, CPLX, KC_, ST_, WM_, WN_>;
  constexpr int NT = C::NT;
  constexpr int KC = C::KC, W = C::W, ST = C::STAGES;
  constexpr int EPS = CPLX ? 1 : 2;  // elements per 16-byte copy
  // row pads (elements) of the [k][m] / [k][n] and [m][k] / [n][k] stage layouts: 4 doubles
  // for 8-byte real fragment loads; for 16-byte complex loads 2 and 0 elements make every
  // quarter-warp hit 8 distinct 4-bank groups (the +4 pads of the real layout gave 2-way
  // conflicts: 1.3e10 bank conflicts in one cfg5 leaf launch).  Both fit Seg2Cfg's sizes.
  constexpr int PM = CPLX ? 2 : 4, PK = CPLX ? 0 : 4;
  constexpr int LSEG = TM * KC / EPS, RSEG = TN * KC / EPS;
  constexpr int LPT = (LSEG + NT - 1) / NT, RPT = (RSEG + NT - 1) / NT;
  extern __shared__ __align__(16) double smem[];

  const int t = blockIdx.x;
  int m0, n0;
  if (p.sym) {
    const int y = blockIdx.y;
    int tm = (int)((sqrt(8.0 * y + 1.0) - 1.0) * 0.5);
    while ((tm + 1) * (tm + 2) / 2 <= y) ++tm;
    while (tm * (tm + 1) / 2 > y) --tm;
    m0 = tm * TM;
    n0 = (y - tm * (tm + 1) / 2) * TN;
  } else {
    const int tilesM = (p.M + TM - 1) / TM;
    m0 = (blockIdx.y % tilesM) * TM;
    n0 = (blockIdx.y / tilesM) * TN;
  }
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  const int wm = (warp % C::WM) * (TM / C::WM), wn = (warp / C::WM) * (TN / C::WN);

  double acc[C::FM][C::FN][2];
  double acci[CPLX ? C::FM : 1][CPLX ? C::FN : 1][2];
  double accq[(CPLX && G3) ? C::FM : 1][(CPLX && G3) ? C::FN : 1][2];
  if constexpr (CPLX && G3) {
#pragma unroll
    for (int i = 0; i < C::FM; ++i)
#pragma unroll
      for (int j = 0; j < C::FN; ++j) accq[i][j][0] = accq[i][j][1] = 0.0;
  }
#pragma unroll
  for (int i = 0; i < C::FM; ++i)
#pragma unroll
    for (int j = 0; j < C::FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  if constexpr (CPLX) {
#pragma unroll
    for (int i = 0; i < C::FM; ++i)
#pragma unroll
      for (int j = 0; j < C::FN; ++j) acci[i][j][0] = acci[i][j][1] = 0.0;
  }

  // accumulating launches: the output tile's lines go to L2 now, so the epilogue's read of C
  // overlaps the operand fetches instead of starting a second DRAM round trip after the last DMMA
  if (p.accumulate & 2) {
    const char* Ob = reinterpret_cast<const char*>(seg_out_ptr(p, t, W));
    const int rows = min(TM, p.M - m0), cols = min(TN, p.N - n0);
    const int lpc = (rows * 8 * W + 127) / 128;  // 128-byte lines per column
    for (int x = tid; x < cols * lpc; x += NT) {
      const char* a = Ob + (m0 + (long long)(n0 + x / lpc) * p.Old) * (8 * W) + (x % lpc) * 128;
      asm volatile("prefetch.global.L2 [%0];" ::"l"(a));
    }
  }

  // ---- copy (producer) state: one chunk ahead of the consumer by ST-1 -------
  int ig = 0, ie = 0, ie1 = 0, ikc = 0, inkc = 1;
  bool iv = false;
  const double* lsrc[LPT];
  const double* rsrc[RPT];
  int ldst[LPT], rdst[RPT], loff[LPT], roff[RPT];
  bool lok[LPT], rok[RPT];
  long long lstep = 0, rstep = 0;
  auto range = [&](int g, int& e0, int& e1) {
    const int* ptr = p.g[g].ptr;
    if (ptr) {
      e0 = ptr[t];
      e1 = ptr[t + 1];
    } else {
      e0 = 0;
      e1 = 1;
    }
  };
  auto setup_group = [&](int g) {  // per-thread copy geometry of group g
    const SegGroup& G = p.g[g];
    const bool lt = G.opL == OP_T || G.opL == OP_H;
    const bool rt = G.opR == OP_T || G.opR == OP_H;
#pragma unroll
    for (int j = 0; j < LPT; ++j) {
      const int sgi = tid + j * NT;
      int m, k;
      if (!lt) {
        k = sgi / (TM / EPS);
        m = (sgi % (TM / EPS)) * EPS;
      } else {
        m = sgi / (KC / EPS);
        k = (sgi % (KC / EPS)) * EPS;
      }
      lok[j] = sgi < LSEG && m0 + m < p.M;
      loff[j] = lt ? (k + (m0 + m) * G.Lld) : (m0 + m + k * G.Lld);
      ldst[j] = (lt ? m * (KC + PK) + k : k * (TM + PM) + m) * W;
    }
#pragma unroll
    for (int j = 0; j < RPT; ++j) {
      const int sgi = tid + j * NT;
      int n, k;
      if (rt) {
        k = sgi / (TN / EPS);
        n = (sgi % (TN / EPS)) * EPS;
      } else {
        n = sgi / (KC / EPS);
        k = (sgi % (KC / EPS)) * EPS;
      }
      rok[j] = sgi < RSEG && n0 + n < p.N;
      roff[j] = rt ? (n0 + n + k * G.Rld) : (k + (n0 + n) * G.Rld);
      rdst[j] = (rt ? k * (TN + PM) + n : n * (KC + PK) + k) * W;
    }
    lstep = (lt ? (long long)KC : (long long)KC * G.Lld) * W;
    rstep = (rt ? (long long)KC * G.Rld : (long long)KC) * W;
    inkc = G.K / KC;
  };
  auto setup_entry = [&]() {  // source pointers of entry ie of group ig
    const SegGroup& G = p.g[ig];
    int l, r;
    if (G.ptr) {
      l = G.li[ie];
      r = G.ri[ie];
    } else {
      l = G.li ? G.li[t] : t;
      r = G.ri ? G.ri[t] : t;
    }
    const double* Lp = G.Lch ? G.Lch[l >> G.Lsh] + (G.Ls * (l & ((1 << G.Lsh) - 1)) + G.Loff) * W
                             : G.L + (G.Ls * l + G.Loff) * W;
    const double* Rp = G.Rch ? G.Rch[r >> G.Rsh] + (G.Rs * (r & ((1 << G.Rsh) - 1)) + G.Roff) * W
                             : G.R + (G.Rs * r + G.Roff) * W;
#pragma unroll
    for (int j = 0; j < LPT; ++j) lsrc[j] = Lp + (long long)loff[j] * W;
#pragma unroll
    for (int j = 0; j < RPT; ++j) rsrc[j] = Rp + (long long)roff[j] * W;
    ikc = 0;
  };
  auto next_group = [&](int g) {  // first group >= g with entries for this tile
    for (; g < p.ngroups; ++g) {
      range(g, ie, ie1);
      if (ie < ie1) {
        ig = g;
        setup_group(g);
        setup_entry();
        return true;
      }
    }
    return false;
  };
  auto issue = [&](int stage) {
    if (iv) {
      double* Ls = smem + stage * C::STAGE;
      double* Rs = Ls + C::LSZ;
#pragma unroll
      for (int j = 0; j < LPT; ++j) {
        if (lok[j]) cp_async16(Ls + ldst[j], lsrc[j], true);
        lsrc[j] += lstep;
      }
#pragma unroll
      for (int j = 0; j < RPT; ++j) {
        if (rok[j]) cp_async16(Rs + rdst[j], rsrc[j], true);
        rsrc[j] += rstep;
      }
      if (++ikc == inkc) {
        if (++ie < ie1) setup_entry();
        else iv = next_group(ig + 1);
      }
    }
    cp_async_commit();
  };

  iv = next_group(0);
#pragma unroll 1
  for (int s = 0; s < ST - 1; ++s) issue(s);

  // ---- consumer: groups in order, a layout-specialised body per group -------
  int stage = 0, istage = ST - 1;
  auto run = [&](auto LT, auto RT, int nch, double cl, double cr) {
    constexpr bool lt = decltype(LT)::value, rt = decltype(RT)::value;
    const int abase = (lt ? (wm + gq) * (KC + PK) + tq : tq * (TM + PM) + wm + gq) * W;
    const int bbase = (rt ? tq * (TN + PM) + wn + gq : (wn + gq) * (KC + PK) + tq) * W;
#pragma unroll 1
    for (int c = 0; c < nch; ++c) {
      cp_async_wait<ST - 2>();
      __syncthreads();
      issue(istage);
      istage = istage + 1 == ST ? 0 : istage + 1;
      const double* Ls = smem + stage * C::STAGE + abase;
      const double* Rs = smem + stage * C::STAGE + C::LSZ + bbase;
#pragma unroll
      for (int kk = 0; kk < KC; kk += 4) {
        constexpr int ami = (lt ? 8 * (KC + PK) : 8) * W, amk = (lt ? 1 : TM + PM) * W;
        constexpr int bnj = (rt ? 8 : 8 * (KC + PK)) * W, bnk = (rt ? TN + PM : 1) * W;
        if constexpr (CPLX) {
          double a[C::FM], ai[C::FM], b[C::FN], bi[C::FN];
#pragma unroll
          for (int i = 0; i < C::FM; ++i) {
            const double2 v = *reinterpret_cast<const double2*>(Ls + i * ami + kk * amk);
            a[i] = v.x;
            ai[i] = cl * v.y;
          }
#pragma unroll
          for (int j = 0; j < C::FN; ++j) {
            const double2 v = *reinterpret_cast<const double2*>(Rs + j * bnj + kk * bnk);
            b[j] = v.x;
            bi[j] = cr * v.y;
          }
          if constexpr (G3) {
            double sa[C::FM], db[C::FN], sb[C::FN];
#pragma unroll
            for (int i = 0; i < C::FM; ++i) sa[i] = a[i] + ai[i];
#pragma unroll
            for (int j = 0; j < C::FN; ++j) {
              db[j] = bi[j] - b[j];
              sb[j] = b[j] + bi[j];
            }
#pragma unroll
            for (int i = 0; i < C::FM; ++i)
#pragma unroll
              for (int j = 0; j < C::FN; ++j) {
                dmma(acc[i][j][0], acc[i][j][1], sa[i], b[j]);     // P
                dmma(acci[i][j][0], acci[i][j][1], a[i], db[j]);   // R
                dmma(accq[i][j][0], accq[i][j][1], ai[i], sb[j]);  // Q
              }
          } else {
#pragma unroll
            for (int i = 0; i < C::FM; ++i)
#pragma unroll
              for (int j = 0; j < C::FN; ++j) {
                dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
                dmma(acc[i][j][0], acc[i][j][1], -ai[i], bi[j]);
                dmma(acci[i][j][0], acci[i][j][1], a[i], bi[j]);
                dmma(acci[i][j][0], acci[i][j][1], ai[i], b[j]);
              }
          }
        } else {
          double a[C::FM], b[C::FN];
#pragma unroll
          for (int i = 0; i < C::FM; ++i) a[i] = Ls[i * ami + kk * amk];
#pragma unroll
          for (int j = 0; j < C::FN; ++j) b[j] = Rs[j * bnj + kk * bnk];
#pragma unroll
          for (int i = 0; i < C::FM; ++i)
#pragma unroll
            for (int j = 0; j < C::FN; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
        }
      }
      stage = stage + 1 == ST ? 0 : stage + 1;
    }
  };
  using F_ = std::false_type;
  using T_ = std::true_type;
#pragma unroll 1
  for (int g = 0; g < p.ngroups; ++g) {
    int e0, e1;
    range(g, e0, e1);
    if (e0 >= e1) continue;
    const SegGroup& G = p.g[g];
    const int nch = (e1 - e0) * (G.K / KC);
    const bool lt = G.opL == OP_T || G.opL == OP_H;
    const bool rt = G.opR == OP_T || G.opR == OP_H;
    const double cl = (G.opL == OP_H || G.opL == OP_C) ? -1.0 : 1.0;
    const double cr = (G.opR == OP_H || G.opR == OP_C) ? -1.0 : 1.0;
    if (lt) {
      if (rt) run(T_{}, T_{}, nch, cl, cr);
      else run(T_{}, F_{}, nch, cl, cr);
    } else {
      if (rt) run(F_{}, T_{}, nch, cl, cr);
      else run(F_{}, F_{}, nch, cl, cr);
    }
  }
  cp_async_wait<0>();

  double* Op = seg_out_ptr(p, t, W);
#pragma unroll
  for (int i = 0; i < C::FM; ++i)
#pragma unroll
    for (int j = 0; j < C::FN; ++j)
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int m = m0 + wm + 8 * i + gq;
        const int n = n0 + wn + 8 * j + 2 * tq + q;
        if (m < p.M && n < p.N) {
          const long long off = m + (long long)n * p.Old;
          const long long offt = n + (long long)m * p.Old;
          const bool mirror = p.sym && m0 != n0;
          if constexpr (CPLX) {
            double re = acc[i][j][q], im = acci[i][j][q];
            if constexpr (G3) {
              re = acc[i][j][q] - accq[i][j][q];
              im = acc[i][j][q] + acci[i][j][q];
            }
            if (p.accumulate) {
              re += Op[2 * off];
              im += Op[2 * off + 1];
            }
            Op[2 * off] = re;
            Op[2 * off + 1] = im;
            if (mirror) {
              Op[2 * offt] = re;
              Op[2 * offt + 1] = -im;
            }
          } else {
            double v = acc[i][j][q];
            if (p.accumulate) v += Op[off];
            Op[off] = v;
            if (mirror) Op[offt] = v;
          }
        }
      }
}

// ---------------------------------------------------------------------------
// seg_small: the same segmented product for outputs of at most 32 x 32 with few k-chunks (the
// small-rank target sums, projections and split products of configs[2] / configs[4]).  ncu of
// seg_gemm3 on those launches (profiles/r02/ncu/l12_targets_cfg3_*): ~940 warp instructions per
// warp around 16 DMMAs - the CTA-wide cp.async pipeline, its barriers and the copy geometry are
// all overhead there, and the launch is instruction-issue bound at ~50 % of the HBM rate.  Here
// ONE WARP owns one output (4 outputs per CTA, no shared memory, no barriers): every lane loads
// its m8n8k4 fragment elements straight from global memory (element (m, k) of op(L) at
// m * sm + k * sk, so all four operand layouts share one body; a quarter-warp reads 32-64
// contiguous bytes: whole sectors), 8 k per step so 2 (FM + FN) loads are in flight before the
// DMMAs.  M = 8 FM and N = 8 FN exactly (all padded dimensions are multiples of 8).  Complex
// products in the 4-product form (two accumulator sets: these launches are not DMMA bound).
template <int FM, int FN, bool CPLX>
__global__ void __launch_bounds__(128) seg_small_kernel(const SegParams p) {
  constexpr int W = CPLX ? 2 : 1;
  constexpr unsigned kFull = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int gq = lane >> 2, tq = lane & 3;
  const int t = blockIdx.x * 4 + (threadIdx.x >> 5);
  if (t >= p.n_out) return;

  // Lane g fetches group g's CSR range and the operand indices of its first entry, all groups at
  // once (two parallel rounds instead of a dependent range -> index pair per group inside the
  // loop); the values reach the other lanes by shuffle.
  int me0 = 0, me1 = 0, ml = 0, mr = 0;
  if (lane < p.ngroups) {
    const SegGroup& G = p.g[lane];
    me0 = G.ptr ? G.ptr[t] : 0;
    me1 = G.ptr ? G.ptr[t + 1] : 1;
    if (me0 < me1) {
      ml = G.ptr ? G.li[me0] : (G.li ? G.li[t] : t);
      mr = G.ptr ? G.ri[me0] : (G.ri ? G.ri[t] : t);
    }
  }
  double* Op = seg_out_ptr(p, t, W);

  // the accumulators start from C when the launch accumulates: the read overlaps the operand
  // fetches and the epilogue only stores
  double acc[FM][FN][2];
  double acci[CPLX ? FM : 1][CPLX ? FN : 1][2];
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j)
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const long long off = (8 * i + gq) + (long long)(8 * j + 2 * tq + q) * p.Old;
        if constexpr (CPLX) {
          double2 c = make_double2(0.0, 0.0);
          if (p.accumulate) c = *reinterpret_cast<const double2*>(Op + 2 * off);
          acc[i][j][q] = c.x;
          acci[i][j][q] = c.y;
        } else {
          acc[i][j][q] = p.accumulate ? Op[off] : 0.0;
        }
      }

#pragma unroll 1
  for (int g = 0; g < p.ngroups; ++g) {
    const int e0 = __shfl_sync(kFull, me0, g), e1 = __shfl_sync(kFull, me1, g);
    int l = __shfl_sync(kFull, ml, g), r = __shfl_sync(kFull, mr, g);
    if (e0 >= e1) continue;
    const SegGroup& G = p.g[g];
    const bool lt = G.opL == OP_T || G.opL == OP_H;
    const bool rt = G.opR == OP_T || G.opR == OP_H;
    const double cl = (G.opL == OP_H || G.opL == OP_C) ? -1.0 : 1.0;
    const double cr = (G.opR == OP_H || G.opR == OP_C) ? -1.0 : 1.0;
    // element strides (in scalars): op(L)(m, k) at m * lsm + k * lsk, op(R)(k, n) at k * rsk + n * rsn
    // (ints: a matrix of the product has far fewer than 2^31 scalars)
    const int lsm = (lt ? G.Lld : 1) * W, lsk = (lt ? 1 : G.Lld) * W;
    const int rsk = (rt ? G.Rld : 1) * W, rsn = (rt ? 1 : G.Rld) * W;
    const int aoff = gq * lsm + tq * lsk, boff = tq * rsk + gq * rsn;
#pragma unroll 1
    for (int e = e0; e < e1; ++e) {
      const double* Lp = (G.Lch ? G.Lch[l >> G.Lsh] + (G.Ls * (l & ((1 << G.Lsh) - 1)) + G.Loff) * W
                                : G.L + (G.Ls * l + G.Loff) * W) + aoff;
      const double* Rp = (G.Rch ? G.Rch[r >> G.Rsh] + (G.Rs * (r & ((1 << G.Rsh) - 1)) + G.Roff) * W
                                : G.R + (G.Rs * r + G.Roff) * W) + boff;
      if (e + 1 < e1) {  // next entry's indices while this entry's operands are fetched
        l = G.li[e + 1];
        r = G.ri[e + 1];
      }
#pragma unroll 1
      for (int kk = 0; kk < G.K; kk += 8) {
        if constexpr (CPLX) {
          double2 a[2][FM], b[2][FN];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
#pragma unroll
            for (int i = 0; i < FM; ++i)
              a[h][i] = __ldg(reinterpret_cast<const double2*>(Lp + 8 * i * lsm + (kk + 4 * h) * lsk));
#pragma unroll
            for (int j = 0; j < FN; ++j)
              b[h][j] = __ldg(reinterpret_cast<const double2*>(Rp + (kk + 4 * h) * rsk + 8 * j * rsn));
          }
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int i = 0; i < FM; ++i)
#pragma unroll
              for (int j = 0; j < FN; ++j) {
                const double ar = a[h][i].x, ai = cl * a[h][i].y, br = b[h][j].x, bi = cr * b[h][j].y;
                dmma(acc[i][j][0], acc[i][j][1], ar, br);
                dmma(acc[i][j][0], acc[i][j][1], -ai, bi);
                dmma(acci[i][j][0], acci[i][j][1], ar, bi);
                dmma(acci[i][j][0], acci[i][j][1], ai, br);
              }
        } else {
          double a[2][FM], b[2][FN];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
#pragma unroll
            for (int i = 0; i < FM; ++i) a[h][i] = __ldg(Lp + 8 * i * lsm + (kk + 4 * h) * lsk);
#pragma unroll
            for (int j = 0; j < FN; ++j) b[h][j] = __ldg(Rp + (kk + 4 * h) * rsk + 8 * j * rsn);
          }
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (int i = 0; i < FM; ++i)
#pragma unroll
              for (int j = 0; j < FN; ++j) dmma(acc[i][j][0], acc[i][j][1], a[h][i], b[h][j]);
        }
      }
    }
  }

#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j)
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const long long off = (8 * i + gq) + (long long)(8 * j + 2 * tq + q) * p.Old;
        if constexpr (CPLX) *reinterpret_cast<double2*>(Op + 2 * off) = make_double2(acc[i][j][q], acci[i][j][q]);
        else Op[off] = acc[i][j][q];
      }
}

// ---------------------------------------------------------------------------
// seg_add: out_t = sum_{e in seg(t)} in[idx_e]   (elements = matrix size in doubles)
static __global__ void seg_add_kernel(double* out, long long Os, const double* in, long long Is,
                               const int* ptr, const int* idx, long long elems, int accumulate) {
  const int t = blockIdx.x;
  const int e0 = ptr[t], e1 = ptr[t + 1];
  for (long long x = (blockIdx.y * (long long)blockDim.x + threadIdx.x) * 2; x < elems;
       x += (long long)gridDim.y * blockDim.x * 2) {
    double2 s = make_double2(0.0, 0.0);
    if (accumulate) s = *reinterpret_cast<const double2*>(out + Os * t + x);
    for (int e = e0; e < e1; ++e) {
      const double2 v = *reinterpret_cast<const double2*>(in + Is * idx[e] + x);
      s.x += v.x;
      s.y += v.y;
    }
    *reinterpret_cast<double2*>(out + Os * t + x) = s;
  }
}

// ---------------------------------------------------------------------------
// gram_combine (mmp.cpp:82-85,192-198): G = sum_i g_i/||g_i||_F (zero terms
// skipped); pre_degenerate = ||g1|| == 0 && ||g2|| == 0 && operand flag.
template <bool CPLX>
__global__ void gram_combine_kernel(const double* g1, const double* g2, const double* g3, double* G,
                                    long long stride, int elems, const uint8_t* op_degen,
                                    const int* op_map, uint8_t* pre_degen) {
  constexpr int W = CPLX ? 2 : 1;
  const int t = blockIdx.x;
  const double* src[3] = {g1 + stride * t * W, g2 + stride * t * W, g3 + stride * t * W};
  __shared__ double red[3][32];
  double s[3] = {0, 0, 0};
  for (int x = threadIdx.x; x < elems * W; x += blockDim.x)
    for (int q = 0; q < 3; ++q) s[q] += src[q][x] * src[q][x];
  for (int q = 0; q < 3; ++q)
    for (int o = 16; o > 0; o >>= 1) s[q] += __shfl_xor_sync(0xffffffffu, s[q], o);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0)
    for (int q = 0; q < 3; ++q) red[q][warp] = s[q];
  __syncthreads();
  __shared__ double nrm[3];
  if (threadIdx.x < 3) {
    double v = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v += red[threadIdx.x][w];
    nrm[threadIdx.x] = sqrt(v);
  }
  __syncthreads();
  double* out = G + stride * t * W;
  for (int x = threadIdx.x; x < elems * W; x += blockDim.x) {
    double v = 0.0;
    for (int q = 0; q < 3; ++q)
      if (nrm[q] > 0.0) v += src[q][x] / nrm[q];
    out[x] = v;
  }
  if (threadIdx.x == 0) {
    const int c = op_map ? op_map[t] : t;
    pre_degen[t] = (nrm[0] == 0.0 && nrm[1] == 0.0 && op_degen[c]) ? 1 : 0;
  }
}

// Grid-wide form of gram_combine for few large Grams (upper levels): grid
// (count, P); pass 1 writes per-chunk sums of squares, pass 2 reads the P
// partials of its Gram in a fixed order (deterministic) and combines its chunk.
__device__ __forceinline__ void chunk_range(long long total, int P, int p, long long& x0, long long& x1) {
  const long long per = (total + P - 1) / P;
  x0 = min(total, per * p);
  x1 = min(total, x0 + per);
}
template <bool CPLX>
__global__ void __launch_bounds__(256) gram_norm_partial_kernel(const double* g1, const double* g2, const double* g3,
                                                                long long stride, int elems, double* partial) {
  constexpr int W = CPLX ? 2 : 1;
  const int t = blockIdx.x, P = gridDim.y, p = blockIdx.y;
  const double* src[3] = {g1 + stride * t * W, g2 + stride * t * W, g3 + stride * t * W};
  long long x0, x1;
  chunk_range((long long)elems * W, P, p, x0, x1);
  double s[3] = {0, 0, 0};
  for (long long x = x0 + threadIdx.x; x < x1; x += blockDim.x)
    for (int q = 0; q < 3; ++q) s[q] += src[q][x] * src[q][x];
  __shared__ double red[3][8];
  for (int q = 0; q < 3; ++q)
    for (int o = 16; o > 0; o >>= 1) s[q] += __shfl_xor_sync(0xffffffffu, s[q], o);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0)
    for (int q = 0; q < 3; ++q) red[q][warp] = s[q];
  __syncthreads();
  if (threadIdx.x < 3) {
    double v = 0;
    for (int w = 0; w < 8; ++w) v += red[threadIdx.x][w];
    partial[(size_t(t) * P + p) * 3 + threadIdx.x] = v;
  }
}
template <bool CPLX>
__global__ void __launch_bounds__(256) gram_combine_grid_kernel(const double* g1, const double* g2, const double* g3,
                                                                double* G, long long stride, int elems,
                                                                const double* partial, const uint8_t* op_degen,
                                                                uint8_t* pre_degen) {
  constexpr int W = CPLX ? 2 : 1;
  const int t = blockIdx.x, P = gridDim.y, p = blockIdx.y;
  __shared__ double nrm[3];
  if (threadIdx.x < 3) {
    double v = 0;
    for (int k = 0; k < P; ++k) v += partial[(size_t(t) * P + k) * 3 + threadIdx.x];
    nrm[threadIdx.x] = sqrt(v);
  }
  __syncthreads();
  const double* src[3] = {g1 + stride * t * W, g2 + stride * t * W, g3 + stride * t * W};
  double* out = G + stride * t * W;
  long long x0, x1;
  chunk_range((long long)elems * W, P, p, x0, x1);
  for (long long x = x0 + threadIdx.x; x < x1; x += blockDim.x) {
    double v = 0.0;
    for (int q = 0; q < 3; ++q)
      if (nrm[q] > 0.0) v += src[q][x] / nrm[q];
    out[x] = v;
  }
  if (p == 0 && threadIdx.x == 0) pre_degen[t] = (nrm[0] == 0.0 && nrm[1] == 0.0 && op_degen[t]) ? 1 : 0;
}

// ---------------------------------------------------------------------------
// pack sorted eigenvectors (n x n) into a padded basis (rows x KC), zeroing
// columns at and beyond the rank
static __global__ void pack_basis_kernel(const double* vec, int n, double* out, int rows, int kc,
                                  const int* rank, int W) {
  const int b = blockIdx.x;
  const int r = rank[b];
  const double* src = vec + (size_t)b * n * n * W;
  double* dst = out + (size_t)b * rows * kc * W;
  for (int x = threadIdx.x; x < rows * kc * W; x += blockDim.x) {
    const int e = x / W, w = x % W;
    const int row = e % rows, col = e / rows;
    dst[x] = (col < r && row < n) ? src[(row + (size_t)col * n) * W + w] : 0.0;
  }
}

// ---------------------------------------------------------------------------
// copy compact R x C blocks cp[e] into quadrant oquad[e] & 3 of the 2R x 2C block
// oquad[e] >> 2 of `out` (the parents' merged blocks, mmp.cpp:344-365)
static __global__ void scatter_quad_kernel(double* const* och, int osh, const double* const* cpch, int cpsh,
                                    const int* oquad, int R, int Cc, int W) {
  const int e = blockIdx.x;
  const int v = oquad[e];
  const int q = v & 3;
  const long long blk = v >> 2;
  double* o = och[blk >> osh] + ((size_t)4 * R * Cc * (blk & ((1LL << osh) - 1)) + (q >> 1) * R +
                                 (size_t)(q & 1) * Cc * 2 * R) * W;
  const double* c = cpch[e >> cpsh] + (size_t)(e & ((1 << cpsh) - 1)) * R * Cc * W;
  for (int x = threadIdx.x; x < R * Cc * W; x += blockDim.x) {
    const int el = x / W, w = x % W;
    const int r = el % R, col = el / R;
    o[((size_t)r + (size_t)col * 2 * R) * W + w] = c[x];
  }
}

// ---------------------------------------------------------------------------
// strided matrix copy jobs (input unpack / output pack)
struct CopyJob {
  const double* src;
  double* dst;
  int rows, cols, sld, dld;
};
static __global__ void copy_jobs_kernel(const CopyJob* jobs, int W) {
  const CopyJob j = jobs[blockIdx.x];
  const long long total = (long long)j.rows * j.cols * W;
  for (long long x = threadIdx.x; x < total; x += blockDim.x) {
    const long long e = x / W;
    const int w = (int)(x % W);
    const int r = (int)(e % j.rows), c = (int)(e / j.rows);
    j.dst[(r + (long long)c * j.dld) * W + w] = j.src[(r + (long long)c * j.sld) * W + w];
  }
}

// MVP: original-order vectors <-> leaf blocks in tree order (padded)
static __global__ void mvp_gather_kernel(const double* X, int N, int nv, const int* perm, const int* beg, const int* size,
                                  double* XL, int NL, int NV, int W) {
  const int p = blockIdx.x;
  double* o = XL + (size_t)p * NL * NV * W;
  for (int x = threadIdx.x; x < size[p] * nv * W; x += blockDim.x) {
    const int e = x / W, w = x % W;
    const int r = e % size[p], v = e / size[p];
    o[(r + (size_t)v * NL) * W + w] = X[(perm[beg[p] + r] + (size_t)v * N) * W + w];
  }
}
static __global__ void mvp_scatter_kernel(const double* YL, int NL, int NV, const int* perm, const int* beg, const int* size,
                                   double* Y, int N, int nv, int W) {
  const int p = blockIdx.x;
  const double* i_ = YL + (size_t)p * NL * NV * W;
  for (int x = threadIdx.x; x < size[p] * nv * W; x += blockDim.x) {
    const int e = x / W, w = x % W;
    const int r = e % size[p], v = e / size[p];
    Y[(perm[beg[p] + r] + (size_t)v * N) * W + w] = i_[(r + (size_t)v * NL) * W + w];
  }
}

// identity matrices (formatted product: P = I, mmp.cpp:280-283)
// columns c0 .. c0+cw-1 of the N x N identity into a zeroed N x cw panel
static __global__ void unit_columns_kernel(double* X, int N, int c0, int cw, int W) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < cw) X[(size_t(c0 + j) + size_t(j) * N) * W] = 1.0;
}

static __global__ void set_identity_kernel(double* out, int n, int ld, const int* rank, int W) {
  const int b = blockIdx.x;
  double* o = out + (size_t)b * n * ld * W;
  for (int x = threadIdx.x; x < n * ld * W; x += blockDim.x) {
    const int e = x / W, w = x % W;
    const int r = e % ld, c = e / ld;
    o[x] = (w == 0 && r == c && r < rank[b]) ? 1.0 : 0.0;
  }
}

}  // namespace h2b
