// The reference's MmpReport counters (mmp.hpp:16-48), computed from the
// structure plan and the per-cluster ranks of A, B and C.  The reference counts
// rows*cols*inner for every dense product it evaluates (mmp.cpp:67-80), the
// Gram outer products by hand (:176,214,221,242) and 9n^3 per truncation (:78);
// this file reproduces exactly those sums so the B200 report equals the CPU
// oracle's bit for bit (they depend only on structure and ranks).
#include <algorithm>

#include "counters.hpp"

namespace h2b {

void count_report(const Plan& P, const RankSet& r, bool adaptive, CountOut& o) {
  const int D = P.depth;
  o.flops = 0;
  o.case_flops = {0, 0, 0, 0};
  o.levels.assign(D + 1, LevelCount{});
  int64_t& F = o.flops;
  auto cf = [&](int c, int64_t w) {
    F += w;
    o.case_flops[c] += w;
  };
  auto n_of = [&](int l, int p) -> int64_t { return P.lv[l].size[p]; };

  // basis products (mmp.cpp:106-124)
  {
    const LevelPlan& L = P.lv[D];
    for (int p = 0; p < L.n; ++p) F += r.ac[D][p] * n_of(D, p) * r.br[D][p];
    for (int l = D - 1; l >= 1; --l)
      for (int p = 0; p < P.lv[l].n; ++p)
        for (int s = 0; s < 2; ++s) {
          const int c = 2 * p + s;
          F += r.ac[l][p] * r.ac[l + 1][c] * r.br[l + 1][c] + r.ac[l][p] * r.br[l + 1][c] * r.br[l][p];
        }
  }

  // ---- leaf level
  {
    const int l = D;
    const LevelPlan& L = P.lv[l];
    LevelCount& st = o.levels[l];
    for (int c = 0; c < 4; ++c) st.case_products[c] = L.case_products[c];
    if (adaptive) {
      // row bases (mmp.cpp:164-200): per full (i,j): qualifying k (hq), F*V, outer
      std::vector<int> t1r(L.n, 0), t1c(L.n, 0), t2(L.n, 0), t3(L.n, 0);
      for (size_t q = 0; q < L.nearb.size(); ++q) {
        const int b = L.nearb[q];
        const int i = L.brow[b], j = L.bcol[b];
        const int64_t ni = n_of(l, i), nj = n_of(l, j);
        for (int e = L.hq.ptr[q]; e < L.hq.ptr[q + 1]; ++e) {
          const int k = L.bcol[L.nearb[L.hq.li[e]]];
          const int64_t nk = n_of(l, k);
          F += ni * nj * nk;  // F^A F^B, counted once (cache semantics, mmp.cpp:127-133)
          F += ni * ni * nk;  // x x^H
          t1r[i]++;
          t1c[k]++;
        }
        F += ni * nj * r.br[l][j] + ni * ni * r.br[l][j];  // case-2 term (mmp.cpp:182-183)
        t2[i]++;
        // column side of the same block viewed as (j,k) of B (mmp.cpp:218-221)
        F += r.ac[l][i] * ni * nj + nj * nj * r.ac[l][i];
        t3[j]++;
      }
      // x^T conj(x) outer products of the column pass (mmp.cpp:212-214)
      for (size_t q = 0; q < L.nearb.size(); ++q) {
        const int b = L.nearb[q];
        const int k = L.bcol[b];
        for (int e = L.hqc.ptr[q]; e < L.hqc.ptr[q + 1]; ++e) {
          const int i = L.brow[L.nearb[L.hqc.li[e]]];
          F += n_of(l, k) * n_of(l, k) * n_of(l, i);
        }
      }
      for (int p = 0; p < L.n; ++p) {
        const int64_t n = n_of(l, p);
        F += n * r.ar[l][p] * n + 9 * n * n * n;  // g3 + truncation (row)
        F += n * r.bc[l][p] * n + 9 * n * n * n;  // g3 + truncation (col)
        st.max_case1_terms = std::max({st.max_case1_terms, t1r[p], t1c[p]});
        st.max_case2_terms = std::max(st.max_case2_terms, t2[p]);
        st.max_case3_terms = std::max(st.max_case3_terms, t3[p]);
      }
      // projections (mmp.cpp:275-279)
      for (int p = 0; p < L.n; ++p)
        F += r.cr[l][p] * n_of(l, p) * r.ar[l][p] + r.bc[l][p] * n_of(l, p) * r.cc[l][p];
    }
    for (int p = 0; p < L.n; ++p) {
      st.max_row_rank = std::max<int64_t>(st.max_row_rank, r.cr[l][p]);
      st.max_col_rank = std::max<int64_t>(st.max_col_rank, r.cc[l][p]);
    }
    // collected full blocks (mmp.cpp:290-293)
    for (int b : L.nearb) {
      const int i = L.brow[b], j = L.bcol[b];
      F += r.cr[l][i] * n_of(l, i) * n_of(l, j) + r.cr[l][i] * n_of(l, j) * r.br[l][j];
      F += r.ac[l][i] * n_of(l, i) * n_of(l, j) + r.ac[l][i] * n_of(l, j) * r.cc[l][j];
    }
    // full targets (mmp.cpp:310-317): densify R operands, then da*db
    for (size_t c = 0; c < L.nearb.size(); ++c) {
      const int tb = L.nearb[c];
      const int i = L.brow[tb], k = L.bcol[tb];
      const int64_t ni = n_of(l, i), nk = n_of(l, k);
      auto da = [&](int j) { return ni * r.ar[l][i] * r.ac[l][j] + ni * r.ac[l][j] * n_of(l, j); };
      auto db = [&](int j) { return n_of(l, j) * r.br[l][j] * r.bc[l][k] + n_of(l, j) * r.bc[l][k] * nk; };
      for (int e = L.ff.ptr[c]; e < L.ff.ptr[c + 1]; ++e) F += ni * n_of(l, L.bcol[L.nearb[L.ff.li[e]]]) * nk;
      for (int e = L.fr.ptr[c]; e < L.fr.ptr[c + 1]; ++e) {
        const int j = L.bcol[L.nearb[L.fr.li[e]]];
        F += db(j) + ni * n_of(l, j) * nk;
      }
      for (int e = L.rf.ptr[c]; e < L.rf.ptr[c + 1]; ++e) {
        const int j = L.bcol[L.adm[L.rf.li[e]]];
        F += da(j) + ni * n_of(l, j) * nk;
      }
      for (int e = L.rr.ptr[c]; e < L.rr.ptr[c + 1]; ++e) {
        const int j = L.bcol[L.adm[L.rr.li[e]]];
        F += da(j) + db(j) + ni * n_of(l, j) * nk;
      }
    }
    // coupling targets (mmp.cpp:319-333)
    for (int t = 0; t < L.n_targets(); ++t) {
      const int i = L.target_row[t], k = L.target_col[t];
      const int64_t kc = r.cr[l][i], kq = r.cc[l][k];
      for (int e = L.ww.ptr[t]; e < L.ww.ptr[t + 1]; ++e) {
        const int64_t ni = n_of(l, i), nk = n_of(l, k);
        if (!adaptive) cf(0, ni * n_of(l, L.bcol[L.nearb[L.ww.li[e]]]) * nk);  // first touch of ff
        cf(0, kc * ni * nk + kc * nk * kq);
      }
      for (int e = L.ly.ptr[t]; e < L.ly.ptr[t + 1]; ++e) {
        const int ab = L.ly.li[e];
        const int j = L.bcol[ab];
        if (L.bkind[ab] != kAdm) {  // F x R
          cf(1, kc * r.br[l][j] * r.bc[l][k] + kc * r.bc[l][k] * kq);
        } else {  // R x R
          cf(3, kc * r.ar[l][i] * r.ac[l][j] + kc * r.ac[l][j] * r.br[l][j] +
                    kc * r.br[l][j] * r.bc[l][k] + kc * r.bc[l][k] * kq);
        }
      }
      for (int e = L.xr.ptr[t]; e < L.xr.ptr[t + 1]; ++e) {
        const int j = L.bcol[L.adm[L.xr.li[e]]];
        cf(2, kc * r.ar[l][i] * r.ac[l][j] + kc * r.ac[l][j] * kq);
      }
    }
  }

  // ---- non-leaf levels (mmp.cpp:555-613)
  for (int l = D - 1; l >= 1; --l) {
    const LevelPlan& L = P.lv[l];
    LevelCount& st = o.levels[l];
    for (int c = 0; c < 4; ++c) st.case_products[c] = L.case_products[c];
    st.case_products[0] = static_cast<int64_t>(L.merged_row.size());
    auto nr = [&](int p) { return r.cr[l + 1][2 * p] + r.cr[l + 1][2 * p + 1]; };
    auto nq = [&](int p) { return r.cc[l + 1][2 * p] + r.cc[l + 1][2 * p + 1]; };
    // assemble_collected (mmp.cpp:370-404)
    for (size_t s = 0; s < L.nearb.size(); ++s)
      for (int q = 0; q < 4; ++q) {
        const int cb = L.sub_child[4 * s + q];
        const LevelPlan& C = P.lv[l + 1];
        if (C.bkind[cb] != kAdm) continue;
        const int tc = C.brow[cb], sc = C.bcol[cb];
        const int m = l + 1;
        F += r.cr[m][tc] * r.ar[m][tc] * r.ac[m][sc] + r.cr[m][tc] * r.ac[m][sc] * r.br[m][sc];
        F += r.ac[m][tc] * r.br[m][tc] * r.bc[m][sc] + r.ac[m][tc] * r.bc[m][sc] * r.cc[m][sc];
      }
    if (adaptive) {
      for (int p = 0; p < L.n; ++p) {
        const int64_t n = nr(p);
        int t1 = 0, t2 = 0;
        for (int e = L.row_merged.ptr[p]; e < L.row_merged.ptr[p + 1]; ++e) {
          F += n * n * nq(L.merged_col[L.row_merged.li[e]]);
          ++t1;
        }
        for (int e = L.row_near.ptr[p]; e < L.row_near.ptr[p + 1]; ++e) {
          const int j = L.bcol[L.nearb[L.row_near.li[e]]];
          const int64_t nb = r.br[l + 1][2 * j] + r.br[l + 1][2 * j + 1];
          F += n * nb * r.br[l][j] + n * n * r.br[l][j];
          ++t2;
        }
        F += n * (r.ar[l + 1][2 * p] + r.ar[l + 1][2 * p + 1]) * r.ar[l][p] + n * n * r.ar[l][p];
        F += 9 * n * n * n;
        st.max_case1_terms = std::max(st.max_case1_terms, t1);
        st.max_case2_terms = std::max(st.max_case2_terms, t2);
      }
      for (int p = 0; p < L.n; ++p) {
        const int64_t n = nq(p);
        int t1 = 0, t3 = 0;
        for (int e = L.col_merged.ptr[p]; e < L.col_merged.ptr[p + 1]; ++e) {
          F += n * n * nr(L.merged_row[L.col_merged.li[e]]);
          ++t1;
        }
        for (int e = L.col_near.ptr[p]; e < L.col_near.ptr[p + 1]; ++e) {
          const int j = L.brow[L.nearb[L.col_near.li[e]]];
          const int64_t na = r.ac[l + 1][2 * j] + r.ac[l + 1][2 * j + 1];
          F += r.ac[l][j] * na * n + n * n * r.ac[l][j];
          ++t3;
        }
        F += n * (r.bc[l + 1][2 * p] + r.bc[l + 1][2 * p + 1]) * r.bc[l][p] + n * n * r.bc[l][p];
        F += 9 * n * n * n;
        st.max_case1_terms = std::max(st.max_case1_terms, t1);
        st.max_case3_terms = std::max(st.max_case3_terms, t3);
      }
      // projections (mmp.cpp:523-537)
      for (int p = 0; p < L.n; ++p)
        for (int s = 0; s < 2; ++s) {
          const int c = 2 * p + s;
          F += r.cr[l][p] * r.cr[l + 1][c] * r.ar[l + 1][c] + r.cr[l][p] * r.ar[l + 1][c] * r.ar[l][p];
          F += r.bc[l][p] * r.bc[l + 1][c] * r.cc[l + 1][c] + r.bc[l][p] * r.cc[l + 1][c] * r.cc[l][p];
        }
    }
    for (int p = 0; p < L.n; ++p) {
      st.max_row_rank = std::max<int64_t>(st.max_row_rank, r.cr[l][p]);
      st.max_col_rank = std::max<int64_t>(st.max_col_rank, r.cc[l][p]);
    }
    // collects (mmp.cpp:544-552)
    for (int b : L.nearb) {
      const int t = L.brow[b], s = L.bcol[b];
      const int64_t nb = r.br[l + 1][2 * s] + r.br[l + 1][2 * s + 1];
      const int64_t na = r.ac[l + 1][2 * t] + r.ac[l + 1][2 * t + 1];
      F += r.cr[l][t] * nr(t) * nb + r.cr[l][t] * nb * r.br[l][s];
      F += r.ac[l][t] * na * nq(s) + r.ac[l][t] * nq(s) * r.cc[l][s];
    }
    // case 1 over merged (mmp.cpp:573-585)
    for (size_t m = 0; m < L.merged_row.size(); ++m) {
      const int i = L.merged_row[m], k = L.merged_col[m];
      cf(0, r.cr[l][i] * nr(i) * nq(k) + r.cr[l][i] * nq(k) * r.cc[l][k]);
    }
    // cases 2-4 (mmp.cpp:587-612)
    for (int t = 0; t < L.n_targets(); ++t) {
      const int i = L.target_row[t], k = L.target_col[t];
      const int64_t kc = r.cr[l][i], kq = r.cc[l][k];
      for (int e = L.ly.ptr[t]; e < L.ly.ptr[t + 1]; ++e) {
        const int ab = L.ly.li[e];
        const int j = L.bcol[ab];
        if (L.bkind[ab] != kAdm) {
          cf(1, kc * r.br[l][j] * r.bc[l][k] + kc * r.bc[l][k] * kq);
        } else {
          cf(3, kc * r.ar[l][i] * r.ac[l][j] + kc * r.ac[l][j] * r.br[l][j] +
                    kc * r.br[l][j] * r.bc[l][k] + kc * r.bc[l][k] * kq);
        }
      }
      for (int e = L.xr.ptr[t]; e < L.xr.ptr[t + 1]; ++e) {
        const int j = L.bcol[L.adm[L.xr.li[e]]];
        cf(2, kc * r.ar[l][i] * r.ac[l][j] + kc * r.ac[l][j] * kq);
      }
    }
  }

  // ---- top-down split (mmp.cpp:617-659)
  for (int l = 1; l < D; ++l) {
    const LevelPlan& L = P.lv[l];
    const LevelPlan& C = P.lv[l + 1];
    for (int32_t b : L.nl_block) {
      const int i = L.brow[b], k = L.bcol[b];
      for (int q = 0; q < 4; ++q) {
        const int ic = 2 * i + (q >> 1), kc = 2 * k + (q & 1);
        F += r.cr[l + 1][ic] * r.cr[l][i] * r.cc[l][k] + r.cr[l + 1][ic] * r.cc[l][k] * r.cc[l + 1][kc];
        if (l + 1 == D) {
          const int cb = L.sub_child[4 * L.kidx[b] + q];
          if (C.bkind[cb] == kFull)
            F += C.size[ic] * r.cr[l + 1][ic] * r.cc[l + 1][kc] + C.size[ic] * r.cc[l + 1][kc] * C.size[kc];
        }
      }
    }
  }
}

}  // namespace h2b
