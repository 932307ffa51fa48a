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
};

constexpr int kMaxGroups = 4;

struct SegParams {
  double* out;
  long long Os, Ooff;
  int Old;
  const int* omap;     // storage index of output t (nullptr = t)
  int M, N;            // output dims (padded)
  int n_out;
  int accumulate;      // out (+)= sum
  int sym;             // Hermitian output (Gram): only tiles m0 >= n0 are computed, mirrored
  int ngroups;
  // optional quadrant scatter (children targets written straight into their
  // parents' merged 2x2 blocks): output t -> block oquad[t] >> 2, quadrant
  // q = oquad[t] & 3 at row offset (q >> 1) * qm and column offset (q & 1) * qn
  const int* oquad;
  int qm, qn;
  SegGroup g[kMaxGroups];
};

__device__ __forceinline__ long long seg_out_offset(const SegParams& p, int t) {
  if (p.oquad) {
    const int v = p.oquad[t];
    const int q = v & 3;
    return p.Os * (v >> 2) + p.Ooff + (q >> 1) * p.qm + (long long)((q & 1) * p.qn) * p.Old;
  }
  return p.Os * (p.omap ? p.omap[t] : t) + p.Ooff;
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
// seg_gemm: CTA = 4 warps (2x2), CTA tile TM x TN, k-chunk KC staged in smem
// as [k][m] / [k][n] (leading dim T+4 -> conflict-free fragment loads), next
// chunk prefetched into registers while the current one is multiplied.
template <int TM, int TN, bool CPLX>
struct SegCfg {
  static constexpr int KC = CPLX ? 16 : 32;
  static constexpr int LDL = TM + 4;
  static constexpr int LDR = TN + 4;
  static constexpr int PL = (TM * KC) / 128;  // L elements per thread per chunk
  static constexpr int PR = (TN * KC) / 128;
  static constexpr int FM = TM / 16;          // 8x8 fragments per warp along m
  static constexpr int FN = TN / 16;
  static constexpr int W = CPLX ? 2 : 1;
  static constexpr int SMEM = (KC * LDL + KC * LDR) * W * 8;
};

struct Cursor {
  int g, e, e1, k0;
  int l, r;
};

template <int TM, int TN, bool CPLX>
__global__ void __launch_bounds__(128) seg_gemm_kernel(const SegParams p) {
  using C = SegCfg<TM, TN, CPLX>;
  constexpr int KC = C::KC;
  extern __shared__ __align__(16) double smem[];
  double* Ls = smem;                          // [W][KC][LDL]
  double* Rs = smem + C::W * KC * C::LDL;     // [W][KC][LDR]

  const int t = blockIdx.x;
  const int tilesM = (p.M + TM - 1) / TM;
  int m0, n0;
  if (p.sym) {  // lower-triangular tile enumeration
    const int y = blockIdx.y;
    int tm = (int)((sqrt(8.0 * y + 1.0) - 1.0) * 0.5);
    while ((tm + 1) * (tm + 2) / 2 <= y) ++tm;
    while (tm * (tm + 1) / 2 > y) --tm;
    m0 = tm * TM;
    n0 = (y - tm * (tm + 1) / 2) * TN;
  } else {
    m0 = (blockIdx.y % tilesM) * TM;
    n0 = (blockIdx.y / tilesM) * TN;
  }
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  const int wm = (warp & 1) * (TM / 2), wn = (warp >> 1) * (TN / 2);

  double acc[C::FM][C::FN][2];
  double acci[CPLX ? C::FM : 1][CPLX ? C::FN : 1][2];
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

  // ---- iteration cursor over (group, entry, k-chunk)
  auto entry_range = [&](int g, int& e0, int& e1) {
    const SegGroup& G = p.g[g];
    if (G.ptr) {
      e0 = G.ptr[t];
      e1 = G.ptr[t + 1];
    } else {
      e0 = 0;
      e1 = 1;
    }
  };
  auto load_entry = [&](Cursor& c) {
    const SegGroup& G = p.g[c.g];
    if (G.ptr) {
      c.l = G.li[c.e];
      c.r = G.ri[c.e];
    } else {
      c.l = G.li ? G.li[t] : t;
      c.r = G.ri ? G.ri[t] : t;
    }
  };
  // advance to the first valid position at or after c (returns false at end)
  auto settle = [&](Cursor& c) -> bool {
    while (c.g < p.ngroups) {
      if (c.e < c.e1 && c.k0 < p.g[c.g].K) return true;
      if (c.e < c.e1) {  // next entry
        c.e++;
        c.k0 = 0;
        if (c.e < c.e1) {
          load_entry(c);
          continue;
        }
      }
      c.g++;
      if (c.g < p.ngroups) {
        entry_range(c.g, c.e, c.e1);
        c.k0 = 0;
        if (c.e < c.e1) load_entry(c);
      }
    }
    return false;
  };

  double rl[C::PL * C::W], rr[C::PR * C::W];
  auto fetch = [&](const Cursor& c) {
    const SegGroup& G = p.g[c.g];
    const double* Lp = G.L + (G.Ls * c.l + G.Loff) * C::W;
    const double* Rp = G.R + (G.Rs * c.r + G.Roff) * C::W;
    const bool lt = G.opL == OP_T || G.opL == OP_H;
    const bool rt = G.opR == OP_T || G.opR == OP_H;
#pragma unroll
    for (int u = 0; u < C::PL; ++u) {
      const int e = tid + u * 128;
      int m, k;
      if (!lt) { m = e % TM; k = e / TM; }
      else { k = e % KC; m = e / KC; }
      const int gm = m0 + m, gk = c.k0 + k;
      const bool ok = gm < p.M && gk < G.K;
      const long long off = lt ? (gk + (long long)gm * G.Lld) : (gm + (long long)gk * G.Lld);
      if constexpr (CPLX) {
        double2 v = ok ? *reinterpret_cast<const double2*>(Lp + 2 * off) : make_double2(0.0, 0.0);
        rl[2 * u] = v.x;
        rl[2 * u + 1] = (G.opL == OP_H || G.opL == OP_C) ? -v.y : v.y;
      } else {
        rl[u] = ok ? Lp[off] : 0.0;
      }
    }
#pragma unroll
    for (int u = 0; u < C::PR; ++u) {
      const int e = tid + u * 128;
      int n, k;
      if (rt) { n = e % TN; k = e / TN; }
      else { k = e % KC; n = e / KC; }
      const int gn = n0 + n, gk = c.k0 + k;
      const bool ok = gn < p.N && gk < G.K;
      const long long off = rt ? (gn + (long long)gk * G.Rld) : (gk + (long long)gn * G.Rld);
      if constexpr (CPLX) {
        double2 v = ok ? *reinterpret_cast<const double2*>(Rp + 2 * off) : make_double2(0.0, 0.0);
        rr[2 * u] = v.x;
        rr[2 * u + 1] = (G.opR == OP_H || G.opR == OP_C) ? -v.y : v.y;
      } else {
        rr[u] = ok ? Rp[off] : 0.0;
      }
    }
  };
  auto stash = [&](const Cursor& c) {
    const SegGroup& G = p.g[c.g];
    const bool lt = G.opL == OP_T || G.opL == OP_H;
    const bool rt = G.opR == OP_T || G.opR == OP_H;
#pragma unroll
    for (int u = 0; u < C::PL; ++u) {
      const int e = tid + u * 128;
      int m, k;
      if (!lt) { m = e % TM; k = e / TM; }
      else { k = e % KC; m = e / KC; }
      if constexpr (CPLX) {
        Ls[k * C::LDL + m] = rl[2 * u];
        Ls[KC * C::LDL + k * C::LDL + m] = rl[2 * u + 1];
      } else {
        Ls[k * C::LDL + m] = rl[u];
      }
    }
#pragma unroll
    for (int u = 0; u < C::PR; ++u) {
      const int e = tid + u * 128;
      int n, k;
      if (rt) { n = e % TN; k = e / TN; }
      else { k = e % KC; n = e / KC; }
      if constexpr (CPLX) {
        Rs[k * C::LDR + n] = rr[2 * u];
        Rs[KC * C::LDR + k * C::LDR + n] = rr[2 * u + 1];
      } else {
        Rs[k * C::LDR + n] = rr[u];
      }
    }
  };

  Cursor cur;
  cur.g = 0;
  cur.k0 = 0;
  entry_range(0, cur.e, cur.e1);
  if (cur.e < cur.e1) load_entry(cur);
  bool have = settle(cur);
  if (have) fetch(cur);
  while (have) {
    __syncthreads();
    stash(cur);
    __syncthreads();
    Cursor nxt = cur;
    nxt.k0 += KC;
    const bool more = settle(nxt);
    if (more) fetch(nxt);  // global loads in flight during the MMAs below
#pragma unroll
    for (int kk = 0; kk < KC; kk += 4) {
      double a[C::FM], b[C::FN];
#pragma unroll
      for (int i = 0; i < C::FM; ++i) a[i] = Ls[(kk + tq) * C::LDL + wm + 8 * i + gq];
#pragma unroll
      for (int j = 0; j < C::FN; ++j) b[j] = Rs[(kk + tq) * C::LDR + wn + 8 * j + gq];
      if constexpr (CPLX) {
        double ai[C::FM], bi[C::FN];
#pragma unroll
        for (int i = 0; i < C::FM; ++i) ai[i] = Ls[KC * C::LDL + (kk + tq) * C::LDL + wm + 8 * i + gq];
#pragma unroll
        for (int j = 0; j < C::FN; ++j) bi[j] = Rs[KC * C::LDR + (kk + tq) * C::LDR + wn + 8 * j + gq];
#pragma unroll
        for (int i = 0; i < C::FM; ++i)
#pragma unroll
          for (int j = 0; j < C::FN; ++j) {
            dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
            dmma(acc[i][j][0], acc[i][j][1], -ai[i], bi[j]);
            dmma(acci[i][j][0], acci[i][j][1], a[i], bi[j]);
            dmma(acci[i][j][0], acci[i][j][1], ai[i], b[j]);
          }
      } else {
#pragma unroll
        for (int i = 0; i < C::FM; ++i)
#pragma unroll
          for (int j = 0; j < C::FN; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
      }
    }
    cur = nxt;
    have = more;
  }

  // ---- epilogue: out (+)= acc
  double* Op = p.out + seg_out_offset(p, t) * C::W;
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
          const long long offt = n + (long long)m * p.Old;  // mirrored position
          const bool mirror = p.sym && m0 != n0;
          if constexpr (CPLX) {
            double re = acc[i][j][q], im = acci[i][j][q];
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
// seg_gemm v2: STAGES-deep cp.async pipeline of raw (untransformed) tiles.
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

template <int TM, int TN, bool CPLX, int KC_ = 16, int ST_ = 3, int WM_ = 2, int WN_ = 2>
__global__ void __launch_bounds__(32 * WM_ * WN_) seg_gemm2_kernel(const SegParams p) {
  using C = Seg2Cfg<TM, TN, CPLX, KC_, ST_, WM_, WN_>;
  constexpr int NT = C::NT;
  constexpr int KC = C::KC, W = C::W, ST = C::STAGES;
  extern __shared__ __align__(16) double smem[];

  const int t = blockIdx.x;
  const int tilesM = (p.M + TM - 1) / TM;
  int m0, n0;
  if (p.sym) {
    const int y = blockIdx.y;
    int tm = (int)((sqrt(8.0 * y + 1.0) - 1.0) * 0.5);
    while ((tm + 1) * (tm + 2) / 2 <= y) ++tm;
    while (tm * (tm + 1) / 2 > y) --tm;
    m0 = tm * TM;
    n0 = (y - tm * (tm + 1) / 2) * TN;
  } else {
    m0 = (blockIdx.y % tilesM) * TM;
    n0 = (blockIdx.y / tilesM) * TN;
  }
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  const int wm = (warp % C::WM) * (TM / C::WM), wn = (warp / C::WM) * (TN / C::WN);

  double acc[C::FM][C::FN][2];
  double acci[CPLX ? C::FM : 1][CPLX ? C::FN : 1][2];
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

  auto entry_range = [&](int g, int& e0, int& e1) {
    const SegGroup& G = p.g[g];
    if (G.ptr) {
      e0 = G.ptr[t];
      e1 = G.ptr[t + 1];
    } else {
      e0 = 0;
      e1 = 1;
    }
  };
  auto load_entry = [&](Cursor& c) {
    const SegGroup& G = p.g[c.g];
    if (G.ptr) {
      c.l = G.li[c.e];
      c.r = G.ri[c.e];
    } else {
      c.l = G.li ? G.li[t] : t;
      c.r = G.ri ? G.ri[t] : t;
    }
  };
  auto settle = [&](Cursor& c) -> bool {
    while (c.g < p.ngroups) {
      if (c.e < c.e1 && c.k0 < p.g[c.g].K) return true;
      if (c.e < c.e1) {
        c.e++;
        c.k0 = 0;
        if (c.e < c.e1) {
          load_entry(c);
          continue;
        }
      }
      c.g++;
      if (c.g < p.ngroups) {
        entry_range(c.g, c.e, c.e1);
        c.k0 = 0;
        if (c.e < c.e1) load_entry(c);
      }
    }
    return false;
  };
  auto init = [&](Cursor& c) -> bool {
    c.g = 0;
    c.k0 = 0;
    if (p.ngroups == 0) return false;
    entry_range(0, c.e, c.e1);
    if (c.e < c.e1) load_entry(c);
    return settle(c);
  };

  // issue the cp.async copies of one chunk into `stage`
  auto issue = [&](const Cursor& c, int stage) {
    const SegGroup& G = p.g[c.g];
    double* Ls = smem + stage * C::STAGE;
    double* Rs = Ls + C::LSZ;
    const double* Lp = G.L + (G.Ls * c.l + G.Loff) * W;
    const double* Rp = G.R + (G.Rs * c.r + G.Roff) * W;
    const bool lt = G.opL == OP_T || G.opL == OP_H;
    const bool rt = G.opR == OP_T || G.opR == OP_H;
    constexpr int EPS = CPLX ? 1 : 2;  // elements per 16-byte segment
    // L chunk: TM x KC elements
    constexpr int LSEG = TM * KC / EPS;
    for (int sgi = tid; sgi < LSEG; sgi += NT) {
      int m, k;
      if (!lt) {  // [k][m], contiguous in m
        k = sgi / (TM / EPS);
        m = (sgi % (TM / EPS)) * EPS;
      } else {  // [m][k], contiguous in k
        m = sgi / (KC / EPS);
        k = (sgi % (KC / EPS)) * EPS;
      }
      const int gm = m0 + m, gk = c.k0 + k;
      const bool ok = gm < p.M && gk < G.K;
      const long long off = lt ? (gk + (long long)gm * G.Lld) : (gm + (long long)gk * G.Lld);
      double* dst = lt ? Ls + (m * (KC + 4) + k) * W : Ls + (k * (TM + 4) + m) * W;
      cp_async16(dst, ok ? Lp + off * W : Lp, ok);
    }
    constexpr int RSEG = TN * KC / EPS;
    for (int sgi = tid; sgi < RSEG; sgi += NT) {
      int n, k;
      if (rt) {  // [k][n], contiguous in n
        k = sgi / (TN / EPS);
        n = (sgi % (TN / EPS)) * EPS;
      } else {  // [n][k], contiguous in k
        n = sgi / (KC / EPS);
        k = (sgi % (KC / EPS)) * EPS;
      }
      const int gn = n0 + n, gk = c.k0 + k;
      const bool ok = gn < p.N && gk < G.K;
      const long long off = rt ? (gn + (long long)gk * G.Rld) : (gk + (long long)gn * G.Rld);
      double* dst = rt ? Rs + (k * (TN + 4) + n) * W : Rs + (n * (KC + 4) + k) * W;
      cp_async16(dst, ok ? Rp + off * W : Rp, ok);
    }
  };

  Cursor ci, cc;
  bool vi = init(ci);
  bool vc = init(cc);
#pragma unroll 1
  for (int s = 0; s < ST - 1; ++s) {
    if (vi) {
      issue(ci, s);
      ci.k0 += KC;
      vi = settle(ci);
    }
    cp_async_commit();
  }
  int stage = 0, istage = ST - 1;
#pragma unroll 1
  while (vc) {
    cp_async_wait<ST - 2>();
    __syncthreads();
    if (vi) {
      issue(ci, istage);
      ci.k0 += KC;
      vi = settle(ci);
    }
    cp_async_commit();
    istage = istage + 1 == ST ? 0 : istage + 1;

    const SegGroup& G = p.g[cc.g];
    const bool lt = G.opL == OP_T || G.opL == OP_H;
    const bool rt = G.opR == OP_T || G.opR == OP_H;
    const double* Ls = smem + stage * C::STAGE;
    const double* Rs = Ls + C::LSZ;
#pragma unroll
    for (int kk = 0; kk < KC; kk += 4) {
      const int k = kk + tq;
      if constexpr (CPLX) {
        const double cl = (G.opL == OP_H || G.opL == OP_C) ? -1.0 : 1.0;
        const double cr = (G.opR == OP_H || G.opR == OP_C) ? -1.0 : 1.0;
        double a[C::FM], ai[C::FM], b[C::FN], bi[C::FN];
#pragma unroll
        for (int i = 0; i < C::FM; ++i) {
          const int m = wm + 8 * i + gq;
          const double2 v = *reinterpret_cast<const double2*>(Ls + 2 * (lt ? m * (KC + 4) + k : k * (TM + 4) + m));
          a[i] = v.x;
          ai[i] = cl * v.y;
        }
#pragma unroll
        for (int j = 0; j < C::FN; ++j) {
          const int n = wn + 8 * j + gq;
          const double2 v = *reinterpret_cast<const double2*>(Rs + 2 * (rt ? k * (TN + 4) + n : n * (KC + 4) + k));
          b[j] = v.x;
          bi[j] = cr * v.y;
        }
#pragma unroll
        for (int i = 0; i < C::FM; ++i)
#pragma unroll
          for (int j = 0; j < C::FN; ++j) {
            dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
            dmma(acc[i][j][0], acc[i][j][1], -ai[i], bi[j]);
            dmma(acci[i][j][0], acci[i][j][1], a[i], bi[j]);
            dmma(acci[i][j][0], acci[i][j][1], ai[i], b[j]);
          }
      } else {
        double a[C::FM], b[C::FN];
#pragma unroll
        for (int i = 0; i < C::FM; ++i) {
          const int m = wm + 8 * i + gq;
          a[i] = Ls[lt ? m * (KC + 4) + k : k * (TM + 4) + m];
        }
#pragma unroll
        for (int j = 0; j < C::FN; ++j) {
          const int n = wn + 8 * j + gq;
          b[j] = Rs[rt ? k * (TN + 4) + n : n * (KC + 4) + k];
        }
#pragma unroll
        for (int i = 0; i < C::FM; ++i)
#pragma unroll
          for (int j = 0; j < C::FN; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
      }
    }
    stage = stage + 1 == ST ? 0 : stage + 1;
    cc.k0 += KC;
    vc = settle(cc);
  }
  cp_async_wait<0>();

  double* Op = p.out + seg_out_offset(p, t) * W;
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
    const double* Lp = G.L + (G.Ls * l + G.Loff) * W;
    const double* Rp = G.R + (G.Rs * r + G.Roff) * W;
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

  double* Op = p.out + seg_out_offset(p, t) * W;
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
// seg_gemm v5 = v3 with several outputs per CTA (grid-stride over outputs): the copy
// pipeline runs on across output boundaries, so the next output's operand chunks are in
// flight while the current output finishes and is written.  For many small outputs with
// a few short entries each (e.g. 24 x 24 targets from 1-3 entries of K = 8), where v3's
// one-output CTAs are dominated by their prologue / epilogue.
template <int TM, int TN, bool CPLX, int KC_ = 8, int ST_ = 4, int WM_ = 2, int WN_ = 2>
__global__ void __launch_bounds__(32 * WM_ * WN_) seg_gemm5_kernel(const SegParams p) {
  using C = Seg2Cfg<TM, TN, CPLX, KC_, ST_, WM_, WN_>;
  constexpr int NT = C::NT;
  constexpr int KC = C::KC, W = C::W, ST = C::STAGES;
  constexpr int EPS = CPLX ? 1 : 2;  // elements per 16-byte copy
  constexpr int LSEG = TM * KC / EPS, RSEG = TN * KC / EPS;
  constexpr int LPT = (LSEG + NT - 1) / NT, RPT = (RSEG + NT - 1) / NT;
  extern __shared__ __align__(16) double smem[];

  int t = blockIdx.x, tp = blockIdx.x;  // consumer / producer output
  const int tstride = gridDim.x;
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

  // ---- copy (producer) state: one chunk ahead of the consumer by ST-1 -------
  int ig = 0, ie = 0, ie1 = 0, ikc = 0, inkc = 1;
  bool iv = false;
  const double* lsrc[LPT];
  const double* rsrc[RPT];
  int ldst[LPT], rdst[RPT], loff[LPT], roff[RPT];
  bool lok[LPT], rok[RPT];
  long long lstep = 0, rstep = 0;
  auto range = [&](int g, int tt, int& e0, int& e1) {
    const int* ptr = p.g[g].ptr;
    if (ptr) {
      e0 = ptr[tt];
      e1 = ptr[tt + 1];
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
      ldst[j] = (lt ? m * (KC + 4) + k : k * (TM + 4) + m) * W;
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
      rdst[j] = (rt ? k * (TN + 4) + n : n * (KC + 4) + k) * W;
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
      l = G.li ? G.li[tp] : tp;
      r = G.ri ? G.ri[tp] : tp;
    }
    const double* Lp = G.L + (G.Ls * l + G.Loff) * W;
    const double* Rp = G.R + (G.Rs * r + G.Roff) * W;
#pragma unroll
    for (int j = 0; j < LPT; ++j) lsrc[j] = Lp + (long long)loff[j] * W;
#pragma unroll
    for (int j = 0; j < RPT; ++j) rsrc[j] = Rp + (long long)roff[j] * W;
    ikc = 0;
  };
  auto next_group = [&](int g) {  // first group >= g with entries, this output or the next ones
    for (;;) {
      for (; g < p.ngroups; ++g) {
        range(g, tp, ie, ie1);
        if (ie < ie1) {
          ig = g;
          setup_group(g);
          setup_entry();
          return true;
        }
      }
      tp += tstride;
      if (tp >= p.n_out) return false;
      g = 0;
    }
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
    const int abase = (lt ? (wm + gq) * (KC + 4) + tq : tq * (TM + 4) + wm + gq) * W;
    const int bbase = (rt ? tq * (TN + 4) + wn + gq : (wn + gq) * (KC + 4) + tq) * W;
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
        constexpr int ami = (lt ? 8 * (KC + 4) : 8) * W, amk = (lt ? 1 : TM + 4) * W;
        constexpr int bnj = (rt ? 8 : 8 * (KC + 4)) * W, bnk = (rt ? TN + 4 : 1) * W;
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
#pragma unroll
          for (int i = 0; i < C::FM; ++i)
#pragma unroll
            for (int j = 0; j < C::FN; ++j) {
              dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
              dmma(acc[i][j][0], acc[i][j][1], -ai[i], bi[j]);
              dmma(acci[i][j][0], acci[i][j][1], a[i], bi[j]);
              dmma(acci[i][j][0], acci[i][j][1], ai[i], b[j]);
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
  for (; t < p.n_out; t += tstride) {
#pragma unroll 1
  for (int g = 0; g < p.ngroups; ++g) {
    int e0, e1;
    range(g, t, e0, e1);
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
  {
  double* Op = p.out + seg_out_offset(p, t) * W;
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
#pragma unroll
  for (int i = 0; i < C::FM; ++i)
#pragma unroll
    for (int j = 0; j < C::FN; ++j) {
      acc[i][j][0] = acc[i][j][1] = 0.0;
      if constexpr (CPLX) acci[i][j][0] = acci[i][j][1] = 0.0;
    }
  }
  cp_async_wait<0>();
}


// ---------------------------------------------------------------------------
// seg_gemm v4 (small output tiles, TM, TN <= 32): the NW warps of the CTA split the
// k-CHUNKS of the segment instead of the output tile.  A pipeline stage holds NW
// consecutive chunks of one group; warp w multiplies chunk w of the stage into its own
// copy of the whole TM x TN accumulator, so one barrier covers NW chunks of MMA work
// (v3 with 2x2 warps on a 16 x 16 tile issues 2 DMMAs per warp per barrier).  The NW
// partial tiles are summed in a fixed order at the end (deterministic).  Copy geometry
// and layout-specialised fragment loads are v3's.
template <int TM, int TN, bool CPLX, int NW = 4, int ST_ = 3>
struct Seg4Cfg {
  using B = Seg2Cfg<TM, TN, CPLX, 8, ST_, 1, 1>;
  static constexpr int NT = 32 * NW;
  static constexpr int CH = B::STAGE;       // doubles per chunk slot
  static constexpr int STG = NW * CH;       // doubles per stage
  static constexpr int PIPE = ST_ * STG;
  static constexpr int RED = NW * TM * TN * B::W;
  static constexpr int SMEM = (PIPE > RED ? PIPE : RED) * 8;
};

template <int TM, int TN, bool CPLX, int NW = 4, int ST_ = 3>
__global__ void __launch_bounds__(32 * NW) seg_gemm4_kernel(const SegParams p) {
  using Q = Seg4Cfg<TM, TN, CPLX, NW, ST_>;
  using C = typename Q::B;
  constexpr int NT = Q::NT, ST = ST_;
  constexpr int KC = C::KC, W = C::W;
  constexpr int EPS = CPLX ? 1 : 2;  // elements per 16-byte copy
  constexpr int LSEG = TM * KC / EPS, RSEG = TN * KC / EPS;
  constexpr int LPT = (LSEG + NT - 1) / NT, RPT = (RSEG + NT - 1) / NT;
  constexpr int FM = TM / 8, FN = TN / 8;
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

  double acc[FM][FN][2];
  double acci[CPLX ? FM : 1][CPLX ? FN : 1][2];
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  if constexpr (CPLX) {
#pragma unroll
    for (int i = 0; i < FM; ++i)
#pragma unroll
      for (int j = 0; j < FN; ++j) acci[i][j][0] = acci[i][j][1] = 0.0;
  }

  // ---- producer state (v3's) ----------------------------------------------
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
  auto setup_group = [&](int g) {
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
      ldst[j] = (lt ? m * (KC + 4) + k : k * (TM + 4) + m) * W;
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
      rdst[j] = (rt ? k * (TN + 4) + n : n * (KC + 4) + k) * W;
    }
    lstep = (lt ? (long long)KC : (long long)KC * G.Lld) * W;
    rstep = (rt ? (long long)KC * G.Rld : (long long)KC) * W;
    inkc = G.K / KC;
  };
  auto setup_entry = [&]() {
    const SegGroup& G = p.g[ig];
    int l, r;
    if (G.ptr) {
      l = G.li[ie];
      r = G.ri[ie];
    } else {
      l = G.li ? G.li[t] : t;
      r = G.ri ? G.ri[t] : t;
    }
    const double* Lp = G.L + (G.Ls * l + G.Loff) * W;
    const double* Rp = G.R + (G.Rs * r + G.Roff) * W;
#pragma unroll
    for (int j = 0; j < LPT; ++j) lsrc[j] = Lp + (long long)loff[j] * W;
#pragma unroll
    for (int j = 0; j < RPT; ++j) rsrc[j] = Rp + (long long)roff[j] * W;
    ikc = 0;
  };
  auto next_group = [&](int g) {
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
  // one stage = up to NW consecutive chunks of ONE group (a group's first chunk always
  // opens a fresh stage, so producer and consumer partition every group identically)
  auto issue = [&](int stage) {
    if (iv) {
      const int g0 = ig;
#pragma unroll 1
      for (int q = 0; q < NW; ++q) {
        if (!iv || ig != g0) break;
        double* Ls = smem + stage * Q::STG + q * Q::CH;
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
    }
    cp_async_commit();
  };

  iv = next_group(0);
#pragma unroll 1
  for (int s = 0; s < ST - 1; ++s) issue(s);

  int stage = 0, istage = ST - 1;
  auto run = [&](auto LT, auto RT, int nch, double cl, double cr) {
    constexpr bool lt = decltype(LT)::value, rt = decltype(RT)::value;
    const int abase = (lt ? gq * (KC + 4) + tq : tq * (TM + 4) + gq) * W;
    const int bbase = (rt ? tq * (TN + 4) + gq : gq * (KC + 4) + tq) * W;
    const int nst = (nch + NW - 1) / NW;
#pragma unroll 1
    for (int c = 0; c < nst; ++c) {
      cp_async_wait<ST - 2>();
      __syncthreads();
      issue(istage);
      istage = istage + 1 == ST ? 0 : istage + 1;
      if (c * NW + warp < nch) {
        const double* Ls = smem + stage * Q::STG + warp * Q::CH + abase;
        const double* Rs = smem + stage * Q::STG + warp * Q::CH + C::LSZ + bbase;
#pragma unroll
        for (int kk = 0; kk < KC; kk += 4) {
          constexpr int ami = (lt ? 8 * (KC + 4) : 8) * W, amk = (lt ? 1 : TM + 4) * W;
          constexpr int bnj = (rt ? 8 : 8 * (KC + 4)) * W, bnk = (rt ? TN + 4 : 1) * W;
          if constexpr (CPLX) {
            double a[FM], ai[FM], b[FN], bi[FN];
#pragma unroll
            for (int i = 0; i < FM; ++i) {
              const double2 v = *reinterpret_cast<const double2*>(Ls + i * ami + kk * amk);
              a[i] = v.x;
              ai[i] = cl * v.y;
            }
#pragma unroll
            for (int j = 0; j < FN; ++j) {
              const double2 v = *reinterpret_cast<const double2*>(Rs + j * bnj + kk * bnk);
              b[j] = v.x;
              bi[j] = cr * v.y;
            }
#pragma unroll
            for (int i = 0; i < FM; ++i)
#pragma unroll
              for (int j = 0; j < FN; ++j) {
                dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
                dmma(acc[i][j][0], acc[i][j][1], -ai[i], bi[j]);
                dmma(acci[i][j][0], acci[i][j][1], a[i], bi[j]);
                dmma(acci[i][j][0], acci[i][j][1], ai[i], b[j]);
              }
          } else {
            double a[FM], b[FN];
#pragma unroll
            for (int i = 0; i < FM; ++i) a[i] = Ls[i * ami + kk * amk];
#pragma unroll
            for (int j = 0; j < FN; ++j) b[j] = Rs[j * bnj + kk * bnk];
#pragma unroll
            for (int i = 0; i < FM; ++i)
#pragma unroll
              for (int j = 0; j < FN; ++j) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
          }
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
  __syncthreads();  // the pipeline buffers become the reduction buffer

  // ---- fixed-order reduction of the NW partial tiles, then the v3 epilogue ----
  double* red = smem + warp * TM * TN * W;
#pragma unroll
  for (int i = 0; i < FM; ++i)
#pragma unroll
    for (int j = 0; j < FN; ++j)
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        const int x = (8 * i + gq) + (8 * j + 2 * tq + q) * TM;
        red[x * W] = acc[i][j][q];
        if constexpr (CPLX) red[x * W + 1] = acci[i][j][q];
      }
  __syncthreads();
  double* Op = p.out + seg_out_offset(p, t) * W;
  const bool mirror = p.sym && m0 != n0;
  for (int x = tid; x < TM * TN; x += NT) {
    const int m = m0 + x % TM, n = n0 + x / TM;
    if (m >= p.M || n >= p.N) continue;
    double re = 0.0, im = 0.0;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      re += smem[(w * TM * TN + x) * W];
      if constexpr (CPLX) im += smem[(w * TM * TN + x) * W + 1];
    }
    const long long off = m + (long long)n * p.Old;
    const long long offt = n + (long long)m * p.Old;
    if constexpr (CPLX) {
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
      if (p.accumulate) re += Op[off];
      Op[off] = re;
      if (mirror) Op[offt] = re;
    }
  }
}

// ---------------------------------------------------------------------------
// seg_add: out_t = sum_{e in seg(t)} in[idx_e]   (elements = matrix size in doubles)
__global__ void seg_add_kernel(double* out, long long Os, const double* in, long long Is,
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
// Batched Hermitian eigensolver for the truncation (truncation.cpp:9-47):
// two-sided cyclic Jacobi, round-robin parallel ordering (n/2 disjoint
// rotations per step), one CTA per Gram.  Storage in shared memory when it
// fits, else in a global scratch (L2-resident).  Output: eigenvectors sorted
// by descending eigenvalue, rank = #{lambda_i > eps*lambda_max} (>= 1), and
// the e_1 / degenerate rule for zero Grams.
struct JacobiParams {
  const double* G;      // [batch][n*n]
  double* scratch;      // global storage when !SMEM: [batch][2][n*(n+1)]
  double* vec_out;      // [batch][n*n] sorted eigenvectors
  double* val_out;      // [batch][n] sorted clamped eigenvalues
  int* rank_out;
  uint8_t* degen_io;    // in: pre-degenerate flag, out: final degenerate flag
  int n;
  double eps;
  int max_sweeps;
};

// MODE 1: A and V in shared memory; 2: A in shared memory, V in global scratch (half the
// shared memory -> more CTAs per SM); 0: both in global scratch
template <bool CPLX, int MODE>
__global__ void __launch_bounds__(256) jacobi_kernel(const JacobiParams p) {
  constexpr int W = CPLX ? 2 : 1;
  const int n = p.n, ld = n + 1;
  const int b = blockIdx.x;
  extern __shared__ __align__(16) double jsm[];
  double* A;
  double* V;
  if constexpr (MODE == 1) {
    A = jsm;
    V = jsm + (size_t)n * ld * W;
  } else if constexpr (MODE == 2) {
    A = jsm;
    V = p.scratch + (size_t)b * n * ld * W;
  } else {
    A = p.scratch + (size_t)b * 2 * n * ld * W;
    V = A + (size_t)n * ld * W;
  }
  __shared__ double cs_c[256], cs_s[256], cs_pr[256], cs_pi[256];
  __shared__ int pp[256], qq[256];
  __shared__ int any_rot, nonzero;
  __shared__ double fro;
  const double* G = p.G + (size_t)b * n * n * W;
  const int tid = threadIdx.x, nt = blockDim.x;
  if (tid == 0) { any_rot = 0; nonzero = 0; fro = 0.0; }
  __syncthreads();
  double ss = 0.0;
  int nz = 0;
  for (int x = tid; x < n * n; x += nt) {
    const int r = x % n, c = x / n;
    // Hermitian: use the lower triangle like Eigen's SelfAdjointEigenSolver
    const int rr = r >= c ? r : c, cc = r >= c ? c : r;
    const double re = G[(rr + cc * n) * W];
    const double im = CPLX ? (r >= c ? G[(rr + cc * n) * W + 1] : -G[(rr + cc * n) * W + 1]) : 0.0;
    if (G[x * W] != 0.0 || (CPLX && G[x * W + 1] != 0.0)) nz = 1;
    A[(r * ld + c) * W] = re;
    if (CPLX) A[(r * ld + c) * W + 1] = (r == c) ? 0.0 : im;
    V[(r * ld + c) * W] = r == c ? 1.0 : 0.0;
    if (CPLX) V[(r * ld + c) * W + 1] = 0.0;
    ss += re * re + im * im;
  }
  // A is stored row-major A[r*ld + c] = a_rc
  for (int o = 16; o > 0; o >>= 1) {
    ss += __shfl_xor_sync(0xffffffffu, ss, o);
    nz |= __shfl_xor_sync(0xffffffffu, nz, o);
  }
  // deterministic block reduction (fixed order) of the Frobenius norm
  __shared__ double warp_ss[32];
  if ((tid & 31) == 0) {
    warp_ss[tid >> 5] = ss;
    if (nz) nonzero = 1;
  }
  __syncthreads();
  if (tid == 0) {
    double f = 0.0;
    for (int w = 0; w < nt / 32; ++w) f += warp_ss[w];
    fro = f;
  }
  __syncthreads();
  // rotation threshold a few ulps of ||G||_F (LAPACK-level backward error):
  // below it rotations only reshuffle round-off in the null space of the PSD
  // Gram and never converge
  const double tol_abs = 2e-15 * sqrt(fro);
  const int half = n / 2;
  if (nonzero) {
    for (int sweep = 0; sweep < p.max_sweeps; ++sweep) {
      __syncthreads();  // every thread has read the previous sweep's flag
      if (tid == 0) any_rot = 0;
      __syncthreads();
      for (int step = 0; step < n - 1; ++step) {
        for (int i = tid; i < half; i += nt) {
          auto idx = [&](int x) { return x == 0 ? 0 : 1 + ((x - 1 + step) % (n - 1)); };
          int a = idx(i), c = idx(n - 1 - i);
          const int pq = a < c ? a : c, qv = a < c ? c : a;
          pp[i] = pq;
          qq[i] = qv;
          const double app = A[(pq * ld + pq) * W], aqq = A[(qv * ld + qv) * W];
          const double br = A[(pq * ld + qv) * W], bi = CPLX ? A[(pq * ld + qv) * W + 1] : 0.0;
          const double babs = CPLX ? hypot(br, bi) : fabs(br);
          double c_ = 1.0, s_ = 0.0, pr = 1.0, pi = 0.0;
          if (babs > tol_abs && babs > 1e-15 * sqrt(fabs(app) * fabs(aqq))) {
            const double tau = (aqq - app) / (2.0 * babs);
            const double tt = (tau >= 0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
            c_ = 1.0 / sqrt(1.0 + tt * tt);
            s_ = tt * c_;
            if (CPLX) { pr = br / babs; pi = bi / babs; }  // e^{i phi}
            else pr = br >= 0 ? 1.0 : -1.0;
            any_rot = 1;
          }
          cs_c[i] = c_;
          cs_s[i] = s_;
          cs_pr[i] = pr;
          cs_pi[i] = pi;
        }
        __syncthreads();
        // rows: row_p <- c row_p - s e^{i phi} row_q ; row_q <- s row_p + c e^{i phi} row_q
        for (int x = tid; x < half * n; x += nt) {
          const int i = x / n, k = x % n;
          const int pq = pp[i], qv = qq[i];
          const double c_ = cs_c[i], s_ = cs_s[i];
          if (s_ == 0.0) continue;
          if constexpr (CPLX) {
            const double pr = cs_pr[i], pi = cs_pi[i];
            const double apr = A[(pq * ld + k) * 2], api = A[(pq * ld + k) * 2 + 1];
            const double aqr = A[(qv * ld + k) * 2], aqi = A[(qv * ld + k) * 2 + 1];
            const double er = pr * aqr - pi * aqi, ei = pr * aqi + pi * aqr;  // e^{i phi} a_q
            A[(pq * ld + k) * 2] = c_ * apr - s_ * er;
            A[(pq * ld + k) * 2 + 1] = c_ * api - s_ * ei;
            A[(qv * ld + k) * 2] = s_ * apr + c_ * er;
            A[(qv * ld + k) * 2 + 1] = s_ * api + c_ * ei;
          } else {
            const double sg = cs_pr[i];
            const double ap = A[pq * ld + k], aq = sg * A[qv * ld + k];
            A[pq * ld + k] = c_ * ap - s_ * aq;
            A[qv * ld + k] = s_ * ap + c_ * aq;
          }
        }
        __syncthreads();
        // columns (and V): col_p <- c col_p - s e^{-i phi} col_q ; col_q <- s col_p + c e^{-i phi} col_q
        for (int x = tid; x < half * n * 2; x += nt) {
          const int which = x / (half * n);
          const int y = x % (half * n);
          const int i = y / n, k = y % n;
          const int pq = pp[i], qv = qq[i];
          const double c_ = cs_c[i], s_ = cs_s[i];
          if (s_ == 0.0) continue;
          double* M = which == 0 ? A : V;
          if constexpr (CPLX) {
            const double pr = cs_pr[i], pi = -cs_pi[i];  // e^{-i phi}
            const double apr = M[(k * ld + pq) * 2], api = M[(k * ld + pq) * 2 + 1];
            const double aqr = M[(k * ld + qv) * 2], aqi = M[(k * ld + qv) * 2 + 1];
            const double er = pr * aqr - pi * aqi, ei = pr * aqi + pi * aqr;
            M[(k * ld + pq) * 2] = c_ * apr - s_ * er;
            M[(k * ld + pq) * 2 + 1] = c_ * api - s_ * ei;
            M[(k * ld + qv) * 2] = s_ * apr + c_ * er;
            M[(k * ld + qv) * 2 + 1] = s_ * api + c_ * ei;
          } else {
            const double sg = cs_pr[i];
            const double ap = M[k * ld + pq], aq = sg * M[k * ld + qv];
            M[k * ld + pq] = c_ * ap - s_ * aq;
            M[k * ld + qv] = s_ * ap + c_ * aq;
          }
        }
        __syncthreads();
      }
      const int rotated = any_rot;
      if (!rotated) break;
    }
  }
  __syncthreads();
  // eigenvalues, descending stable order, rank (truncation.cpp:29-45)
  __shared__ double top_s;
  double* vals = p.val_out + (size_t)b * n;
  if (tid == 0) {
    double top = 0.0;
    for (int i = 0; i < n; ++i) top = fmax(top, fmax(A[(i * ld + i) * W], 0.0));
    top_s = top;
  }
  __syncthreads();
  const double top = top_s;
  const bool unit = !nonzero || !(top > 0.0);
  double* vo = p.vec_out + (size_t)b * n * n * W;
  __shared__ int rank_s;
  if (tid == 0) rank_s = 0;
  __syncthreads();
  for (int i = tid; i < n; i += nt) {
    const double li = fmax(A[(i * ld + i) * W], 0.0);
    int pos = 0;
    for (int j = 0; j < n; ++j) {
      const double lj = fmax(A[(j * ld + j) * W], 0.0);
      pos += (lj > li) || (lj == li && j < i);
    }
    vals[pos] = li;
    if (li > p.eps * top) atomicAdd(&rank_s, 1);
    for (int r = 0; r < n; ++r) {
      vo[(r + (size_t)pos * n) * W] = unit ? (r == 0 && pos == 0 ? 1.0 : 0.0) : V[(r * ld + i) * W];
      if (CPLX) vo[(r + (size_t)pos * n) * W + 1] = unit ? 0.0 : V[(r * ld + i) * W + 1];
    }
  }
  __syncthreads();
  if (tid == 0) {
    // the count of eigenvalues above the threshold equals the leading run in
    // descending order, as in the reference's early-exit loop
    p.rank_out[b] = unit ? 1 : (rank_s < 1 ? 1 : rank_s);
    p.degen_io[b] = (unit ? 1 : 0) | p.degen_io[b];
  }
}

// ---------------------------------------------------------------------------
// Medium Gram dimensions (64 < n <= 224, real): two-sided cyclic Jacobi on the
// packed lower triangle in shared memory (n(n+1)/2 doubles <= 200 KB).  With
// disjoint rotation pairs, every unordered 2x2 block (i, j) of the current
// pairing is updated exactly once per step as B' = G_i B G_j^T (one phase, two
// barriers per step).  The rotations are logged to global memory and V is
// rebuilt afterwards by jacobi_replay_kernel, whose rows are independent
// (V <- V G^T), so the eigenvector accumulation neither needs shared memory
// nor serialises the sweep.
struct JacobiPackedParams {
  const double* G;     // [batch][n*n] (lower triangle read)
  double* log;         // [batch][max_steps][n/2][3]  (c, s, sign)
  int* steps_out;      // [batch] rotation steps taken
  int* order_out;      // [batch][n] position of eigenvalue i in descending order
  double* val_out;     // [batch][n]
  double* vec_out;     // VSM: [batch][n*n] sorted eigenvectors
  int* rank_out;
  uint8_t* degen_io;
  int n;
  double eps;
  int max_sweeps;
};

__device__ __forceinline__ int pk(int r, int c) { return r >= c ? r * (r + 1) / 2 + c : c * (c + 1) / 2 + r; }

template <bool VSM>
__global__ void __launch_bounds__(512) jacobi_packed_kernel(const JacobiPackedParams p) {
  extern __shared__ __align__(16) double Ap[];
  const int n = p.n, h = n / 2, b = blockIdx.x;
  double* Vs = Ap + n * (n + 1) / 2;  // VSM: V in shared memory, ld n + 1
  const int vld = n + 1;
  const int tid = threadIdx.x, nt = blockDim.x;
  __shared__ double cs_c[128], cs_s[128], cs_g[128];
  __shared__ int pp[128], qq[128];
  __shared__ int any_rot, nonzero, steps;
  __shared__ double warp_ss[16], fro;
  const double* G = p.G + (size_t)b * n * n;
  if (tid == 0) { any_rot = 0; nonzero = 0; steps = 0; }
  __syncthreads();
  double ss = 0.0;
  int nz = 0;
  for (int x = tid; x < n * (n + 1) / 2; x += nt) {
    // packed index x -> (r, c), r >= c
    int r = (int)((sqrt(8.0 * x + 1.0) - 1.0) * 0.5);
    while ((r + 1) * (r + 2) / 2 <= x) ++r;
    while (r * (r + 1) / 2 > x) --r;
    const int c = x - r * (r + 1) / 2;
    const double v = G[r + (size_t)c * n];
    Ap[x] = v;
    nz |= v != 0.0;
    ss += (r == c ? 1.0 : 2.0) * v * v;
  }
  for (int o = 16; o > 0; o >>= 1) {
    ss += __shfl_xor_sync(0xffffffffu, ss, o);
    nz |= __shfl_xor_sync(0xffffffffu, nz, o);
  }
  if ((tid & 31) == 0) {
    warp_ss[tid >> 5] = ss;
    if (nz) nonzero = 1;
  }
  __syncthreads();
  if (tid == 0) {
    double f = 0.0;
    for (int w = 0; w < nt / 32; ++w) f += warp_ss[w];
    fro = f;
  }
  __syncthreads();
  // rotation threshold a few ulps of ||G||_F (LAPACK-level backward error):
  // below it rotations only reshuffle round-off in the null space of the PSD
  // Gram and never converge
  const double tol_abs = 2e-15 * sqrt(fro);
  double* log = VSM ? nullptr : p.log + (size_t)b * (size_t)p.max_sweeps * (n - 1) * h * 3;
  int nsteps = 0;
  const int nblk = h * (h + 1) / 2;
  if (VSM)
    for (int x = tid; x < n * vld; x += nt) Vs[x] = (x % vld == x / vld) ? 1.0 : 0.0;
  // this thread's 2x2 blocks (i, j), j <= i, decoded once
  constexpr int kMaxBlk = 13;  // ceil(112 * 113 / 2 / 512)
  int bi_[kMaxBlk], bj_[kMaxBlk], nmine = 0;
  for (int t = tid; t < nblk && nmine < kMaxBlk; t += nt) {
    int i = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
    while ((i + 1) * (i + 2) / 2 <= t) ++i;
    while (i * (i + 1) / 2 > t) --i;
    bi_[nmine] = i;
    bj_[nmine] = t - i * (i + 1) / 2;
    ++nmine;
  }
  __syncthreads();
  if (nonzero) {
    for (int sweep = 0; sweep < p.max_sweeps; ++sweep) {
      __syncthreads();
      if (tid == 0) any_rot = 0;
      __syncthreads();
      for (int step = 0; step < n - 1; ++step) {
        for (int i = tid; i < h; i += nt) {
          auto idx = [&](int x) { return x == 0 ? 0 : 1 + ((x - 1 + step) % (n - 1)); };
          const int a = idx(i), c = idx(n - 1 - i);
          const int pq = a < c ? a : c, qv = a < c ? c : a;
          pp[i] = pq;
          qq[i] = qv;
          const double app = Ap[pk(pq, pq)], aqq = Ap[pk(qv, qv)], br = Ap[pk(qv, pq)];
          const double babs = fabs(br);
          double c_ = 1.0, s_ = 0.0, g_ = 1.0;
          if (babs > tol_abs && babs > 1e-15 * sqrt(fabs(app) * fabs(aqq))) {
            const double tau = (aqq - app) / (2.0 * babs);
            const double tt = (tau >= 0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
            c_ = 1.0 / sqrt(1.0 + tt * tt);
            s_ = tt * c_;
            g_ = br >= 0 ? 1.0 : -1.0;
            any_rot = 1;
          }
          cs_c[i] = c_;
          cs_s[i] = s_;
          cs_g[i] = g_;
          if (!VSM) {
            double* lg = log + ((size_t)nsteps * h + i) * 3;
            lg[0] = c_;
            lg[1] = s_;
            lg[2] = g_;
          }
        }
        __syncthreads();
        // rotation G = [[c, -s g], [s, c g]] on the (p, q) plane: B' = G_i B G_j^T
        if (VSM)  // V <- V G^T on the pair columns (rows independent)
          for (int x = tid; x < n * h; x += nt) {
            const int r = x / h, i = x % h;
            const double c_ = cs_c[i], s_ = cs_s[i], g_ = cs_g[i];
            if (s_ == 0.0) continue;
            double* v = Vs + r * vld;
            const double vp = v[pp[i]], vq = v[qq[i]];
            v[pp[i]] = c_ * vp - s_ * g_ * vq;
            v[qq[i]] = s_ * vp + c_ * g_ * vq;
          }
        for (int u = 0; u < nmine; ++u) {
          const int i = bi_[u], j = bj_[u];  // j <= i
          const double ci = cs_c[i], si = cs_s[i], gi = cs_g[i];
          const double cj = cs_c[j], sj = cs_s[j], gj = cs_g[j];
          if (si == 0.0 && sj == 0.0) continue;
          const int pi_ = pp[i], qi = qq[i], pj = pp[j], qj = qq[j];
          if (i == j) {
            const double x = Ap[pk(pi_, pi_)], y = Ap[pk(qi, pi_)], w = Ap[pk(qi, qi)];
            // rows then columns: B' = G B G^T with B symmetric
            const double r00 = ci * x - si * gi * y, r01 = ci * y - si * gi * w;
            const double r10 = si * x + ci * gi * y, r11 = si * y + ci * gi * w;
            Ap[pk(pi_, pi_)] = r00 * ci - r01 * si * gi;
            Ap[pk(qi, qi)] = r10 * si + r11 * ci * gi;
            Ap[pk(qi, pi_)] = 0.0;  // annihilated by construction
          } else {
            const double x = Ap[pk(pi_, pj)], y = Ap[pk(pi_, qj)], z = Ap[pk(qi, pj)], w = Ap[pk(qi, qj)];
            const double r00 = ci * x - si * gi * z, r01 = ci * y - si * gi * w;  // G_i B
            const double r10 = si * x + ci * gi * z, r11 = si * y + ci * gi * w;
            Ap[pk(pi_, pj)] = r00 * cj - r01 * sj * gj;  // (G_i B) G_j^T
            Ap[pk(pi_, qj)] = r00 * sj + r01 * cj * gj;
            Ap[pk(qi, pj)] = r10 * cj - r11 * sj * gj;
            Ap[pk(qi, qj)] = r10 * sj + r11 * cj * gj;
          }
        }
        __syncthreads();
        ++nsteps;
      }
      const int rotated = any_rot;
      if (!rotated) break;
    }
  }
  __syncthreads();
  __shared__ double top_s;
  __shared__ int rank_s;
  if (tid == 0) {
    double top = 0.0;
    for (int i = 0; i < n; ++i) top = fmax(top, fmax(Ap[pk(i, i)], 0.0));
    top_s = top;
    rank_s = 0;
  }
  __syncthreads();
  const double top = top_s;
  const bool unit = !nonzero || !(top > 0.0);
  for (int i = tid; i < n; i += nt) {
    const double li = fmax(Ap[pk(i, i)], 0.0);
    int pos = 0;
    for (int j = 0; j < n; ++j) {
      const double lj = fmax(Ap[pk(j, j)], 0.0);
      pos += (lj > li) || (lj == li && j < i);
    }
    p.val_out[(size_t)b * n + pos] = li;
    p.order_out[(size_t)b * n + i] = pos;
    if (li > p.eps * top) atomicAdd(&rank_s, 1);
    if (VSM) {
      double* out = p.vec_out + (size_t)b * n * n;
      for (int r = 0; r < n; ++r)
        out[r + (size_t)pos * n] = unit ? ((r == 0 && pos == 0) ? 1.0 : 0.0) : Vs[r * vld + i];
    }
  }
  __syncthreads();
  if (tid == 0) {
    p.steps_out[b] = unit ? -1 : nsteps;  // -1: e_1 basis
    p.rank_out[b] = unit ? 1 : (rank_s < 1 ? 1 : rank_s);
    p.degen_io[b] = (unit ? 1 : 0) | p.degen_io[b];
  }
}

// V = G_1^T G_2^T ... (rows independent): each CTA rebuilds `rows` rows of V in
// shared memory and writes them as sorted eigenvector columns.
__global__ void __launch_bounds__(256) jacobi_replay_kernel(const double* log, const int* steps, const int* order,
                                                            int n, int max_sweeps, int rows_per_cta, double* vec_out) {
  extern __shared__ __align__(16) double Vs[];  // [rows][n]
  const int b = blockIdx.y, r0 = blockIdx.x * rows_per_cta;
  const int h = n / 2, tid = threadIdx.x, nt = blockDim.x;
  const int nr = min(rows_per_cta, n - r0);
  if (nr <= 0) return;
  const int ns = steps[b];
  for (int x = tid; x < nr * n; x += nt) {
    const int rr = x / n, c = x % n;
    Vs[x] = (r0 + rr == c) ? 1.0 : 0.0;
  }
  __syncthreads();
  const double* lg = log + (size_t)b * (size_t)max_sweeps * (n - 1) * h * 3;
  __shared__ double rot[2][112 * 3];
  if (ns > 0)
    for (int x = tid; x < h * 3; x += nt) rot[0][x] = lg[x];
  __syncthreads();
  for (int st = 0; st < ns; ++st) {
    const int step = st % (n - 1);
    const double* cur = rot[st & 1];
    if (st + 1 < ns)  // stage the next step's rotations
      for (int x = tid; x < h * 3; x += nt) rot[(st + 1) & 1][x] = lg[(size_t)(st + 1) * h * 3 + x];
    for (int x = tid; x < nr * h; x += nt) {
      const int rr = x / h, i = x % h;
      const double c_ = cur[3 * i], s_ = cur[3 * i + 1], g_ = cur[3 * i + 2];
      if (s_ == 0.0) continue;
      auto idx = [&](int y) { return y == 0 ? 0 : 1 + ((y - 1 + step) % (n - 1)); };
      const int a = idx(i), cc = idx(n - 1 - i);
      const int pq = a < cc ? a : cc, qv = a < cc ? cc : a;
      double* v = Vs + rr * n;
      const double vp = v[pq], vq = v[qv];
      v[pq] = c_ * vp - s_ * g_ * vq;
      v[qv] = s_ * vp + c_ * g_ * vq;
    }
    __syncthreads();
  }
  double* out = vec_out + (size_t)b * n * n;
  for (int x = tid; x < nr * n; x += nt) {
    const int rr = x / n, c = x % n;
    const int pos = ns < 0 ? c : order[(size_t)b * n + c];
    double v = Vs[x];
    if (ns < 0) v = (r0 + rr == 0 && c == 0) ? 1.0 : 0.0;  // e_1
    out[(r0 + rr) + (size_t)pos * n] = v;
  }
}

// ---------------------------------------------------------------------------
// Finalize a library eigendecomposition (ascending eigenvalues, eigenvectors
// in columns) into the truncation output of jacobi_kernel: clamp at 0, sort
// descending, strict threshold, >= 1 vector, e_1 for exactly-zero Grams
// (truncation.cpp:23-45).
template <bool CPLX>
__global__ void eig_finalize_kernel(const double* G, const double* V, const double* w, int n, double eps,
                                    double* vec_out, double* val_out, int* rank_out, uint8_t* degen_io) {
  constexpr int W = CPLX ? 2 : 1;
  const int b = blockIdx.x;
  const double* g = G + (size_t)b * n * n * W;
  const double* v = V + (size_t)b * n * n * W;
  const double* wb = w + (size_t)b * n;
  __shared__ int nz;
  if (threadIdx.x == 0) nz = 0;
  __syncthreads();
  int mine = 0;
  for (int x = threadIdx.x; x < n * n * W; x += blockDim.x) mine |= g[x] != 0.0;
  if (__syncthreads_or(mine) && threadIdx.x == 0) nz = 1;
  __syncthreads();
  const double top = fmax(wb[n - 1], 0.0);
  const bool unit = !nz || !(top > 0.0);
  double* vo = vec_out + (size_t)b * n * n * W;
  // descending order = reversed ascending order (ties keep LAPACK's order reversed, as Eigen's reverse())
  for (int x = threadIdx.x; x < n * n * W; x += blockDim.x) {
    const int e = x / W, q = x % W;
    const int r = e % n, c = e / n;
    vo[x] = unit ? ((q == 0 && r == 0 && c == 0) ? 1.0 : 0.0) : v[(r + (size_t)(n - 1 - c) * n) * W + q];
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) val_out[(size_t)b * n + i] = fmax(wb[n - 1 - i], 0.0);
  if (threadIdx.x == 0) {
    int r = 0;
    while (r < n && fmax(wb[n - 1 - r], 0.0) > eps * top) ++r;
    rank_out[b] = unit ? 1 : (r < 1 ? 1 : r);
    degen_io[b] = (unit ? 1 : 0) | degen_io[b];
  }
}

// ---------------------------------------------------------------------------
// pack sorted eigenvectors (n x n) into a padded basis (rows x KC), zeroing
// columns at and beyond the rank
__global__ void pack_basis_kernel(const double* vec, int n, double* out, int rows, int kc,
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
// gather 2x2 quadrants into a dense (2R x 2C) matrix; idx[4*t+q] (q = 2*ri+ci)
__global__ void gather_quad_kernel(double* out, const double* src, long long Ss, int R, int Cc,
                                   const int* idx, const int* remap, int W) {
  const int t = blockIdx.x;
  const int ld = 2 * R;
  double* o = out + (size_t)t * 4 * R * Cc * W;
  for (int x = threadIdx.x; x < 4 * R * Cc * W; x += blockDim.x) {
    const int e = x / W, w = x % W;
    const int row = e % ld, col = e / ld;
    const int q = 2 * (row / R) + (col / Cc);
    int s = idx[4 * t + q];
    if (s >= 0 && remap) s = remap[s];
    o[x] = s < 0 ? 0.0 : src[(Ss * s + (row % R) + (size_t)(col % Cc) * R) * W + w];
  }
}

// ---------------------------------------------------------------------------
// strided matrix copy jobs (input unpack / output pack)
struct CopyJob {
  const double* src;
  double* dst;
  int rows, cols, sld, dld;
};
__global__ void copy_jobs_kernel(const CopyJob* jobs, int W) {
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
__global__ void mvp_gather_kernel(const double* X, int N, int nv, const int* perm, const int* beg, const int* size,
                                  double* XL, int NL, int NV, int W) {
  const int p = blockIdx.x;
  double* o = XL + (size_t)p * NL * NV * W;
  for (int x = threadIdx.x; x < size[p] * nv * W; x += blockDim.x) {
    const int e = x / W, w = x % W;
    const int r = e % size[p], v = e / size[p];
    o[(r + (size_t)v * NL) * W + w] = X[(perm[beg[p] + r] + (size_t)v * N) * W + w];
  }
}
__global__ void mvp_scatter_kernel(const double* YL, int NL, int NV, const int* perm, const int* beg, const int* size,
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
__global__ void unit_columns_kernel(double* X, int N, int c0, int cw, int W) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j < cw) X[(size_t(c0 + j) + size_t(j) * N) * W] = 1.0;
}

__global__ void set_identity_kernel(double* out, int n, int ld, const int* rank, int W) {
  const int b = blockIdx.x;
  double* o = out + (size_t)b * n * ld * W;
  for (int x = threadIdx.x; x < n * ld * W; x += blockDim.x) {
    const int e = x / W, w = x % W;
    const int r = e % ld, c = e / ld;
    o[x] = (w == 0 && r == c && r < rank[b]) ? 1.0 : 0.0;
  }
}

}  // namespace h2b
