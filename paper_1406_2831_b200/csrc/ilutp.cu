// ILUTP split preconditioning (reference ilutp.py): the factorization on the
// host, the triangular solves on the device.
//
// Host: krb_ilutp_factor restates ilutp_factor (ilutp.py:131-281) operation
// for operation -- the same row-by-row elimination over a min-heap of frozen
// positions, the same dual-threshold drop rule (|v| <= drop_tol ||a_i||),
// the same column-pivot test and swap, the same per-row fill limit, the same
// IEEE double arithmetic (one rounding per multiply / subtract / divide, no
// contraction: -ffp-contract=off) -- so L, U and perm equal the reference's
// bit for bit (tests/test_ilutp.py against krecycle.ilutp_factor).  Only
// ||a_i|| may differ in the last bit (the reference takes it from BLAS ddot);
// it enters nothing but the drop comparisons.
//
// Device: level-scheduled triangular solves for L^{-1}, U^{-1} and their
// adjoints (ilutp.py:76-97), see the kernels below.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <functional>
#include <queue>
#include <unordered_map>
#include <vector>

#include "krb_internal.cuh"

struct krb_ilutp {
  int64_t n = 0;
  std::vector<int64_t> Lrp, Urp, perm;
  std::vector<int32_t> Lci, Uci;
  std::vector<double> Lval, Uval;
};

namespace krb {

// ordered working row: insertion order kept (the reference's dict), O(1)
// lookup / removal by column
struct WorkRow {
  std::vector<int64_t> cols;
  std::vector<double> vals;
  std::vector<char> live;
  std::unordered_map<int64_t, int64_t> at;
  void clear() {
    cols.clear();
    vals.clear();
    live.clear();
    at.clear();
  }
  void set(int64_t c, double v) {   // insert (c must be absent)
    at[c] = (int64_t)cols.size();
    cols.push_back(c);
    vals.push_back(v);
    live.push_back(1);
  }
  double *find(int64_t c) {
    auto it = at.find(c);
    return it == at.end() ? nullptr : &vals[it->second];
  }
  bool pop(int64_t c, double *v) {
    auto it = at.find(c);
    if (it == at.end()) return false;
    *v = vals[it->second];
    live[it->second] = 0;
    at.erase(it);
    return true;
  }
};

static int ilutp_factor_host(int64_t n, const int64_t *rp, const int32_t *ci,
                             const double *val, double drop_tol, double pivot_tol,
                             int64_t fill_limit, krb_ilutp *F) {
  std::vector<int64_t> perm(n), ipos(n);
  for (int64_t i = 0; i < n; ++i) perm[i] = ipos[i] = i;
  std::vector<double> diag(n, 0.0);
  std::vector<std::vector<int64_t>> u_cols(n), l_pos(n);
  std::vector<std::vector<double>> u_vals(n), l_val(n);
  std::vector<char> done(n, 0);
  std::vector<int64_t> touched;
  WorkRow w;
  for (int64_t i = 0; i < n; ++i) {
    const int64_t lo = rp[i], hi = rp[i + 1];
    // ||a_i||_2 (ilutp.py:189): sum of squares in order, then sqrt
    double ss = 0.0;
    for (int64_t e = lo; e < hi; ++e) ss = ss + val[e] * val[e];
    const double row_norm = std::sqrt(ss);
    if (row_norm == 0.0) {
      set_error("zero pivot: row %lld is empty", (long long)i);
      return KRB_EFACTOR;
    }
    const double tau = drop_tol * row_norm;
    w.clear();
    std::priority_queue<int64_t, std::vector<int64_t>, std::greater<int64_t>> heap;
    for (int64_t e = lo; e < hi; ++e) {
      const int64_t c = ci[e];
      double *slot = w.find(c);
      if (slot)
        *slot = val[e];                 // w[c] = v (a repeated column overwrites)
      else
        w.set(c, val[e]);
      const int64_t p = ipos[c];
      if (p < i) heap.push(p);
    }
    std::vector<int64_t> lp;
    std::vector<double> lv;
    for (int64_t t : touched) done[t] = 0;
    touched.clear();
    while (!heap.empty()) {
      const int64_t p = heap.top();
      heap.pop();
      if (done[p]) continue;
      done[p] = 1;
      touched.push_back(p);
      const int64_t c = perm[p];
      double v;
      if (!w.pop(c, &v)) continue;
      if (std::fabs(v) <= tau) continue;            // drop (pre-division magnitude)
      const double factor = v / diag[p];
      lp.push_back(p);
      lv.push_back(factor);
      const std::vector<int64_t> &uc = u_cols[p];
      const std::vector<double> &uv = u_vals[p];
      for (size_t q = 0; q < uc.size(); ++q) {
        const int64_t c2 = uc[q];
        const double upd = factor * uv[q];
        double *slot = w.find(c2);
        if (slot) {
          *slot = *slot - upd;
        } else {
          w.set(c2, -upd);
          const int64_t p2 = ipos[c2];
          if (p2 < i) heap.push(p2);
        }
      }
    }
    // candidates: the remaining (upper) entries above the threshold plus the
    // natural diagonal candidate, in the working row's insertion order
    std::vector<int64_t> cand_cols;
    std::vector<double> cand_vals;
    for (size_t q = 0; q < w.cols.size(); ++q) {
      if (!w.live[q]) continue;
      const int64_t c = w.cols[q];
      const double v = w.vals[q];
      if (std::fabs(v) > tau || ipos[c] == i) {
        cand_cols.push_back(c);
        cand_vals.push_back(v);
      }
    }
    if (cand_cols.empty()) {
      set_error("zero pivot: row %lld lost all entries", (long long)i);
      return KRB_EFACTOR;
    }
    size_t m = 0;                                    // first maximum (np.argmax)
    for (size_t q = 1; q < cand_vals.size(); ++q)
      if (std::fabs(cand_vals[q]) > std::fabs(cand_vals[m])) m = q;
    const double *dslot = w.find(perm[i]);
    double diag_val = dslot ? *dslot : 0.0;
    if (std::fabs(diag_val) < pivot_tol * std::fabs(cand_vals[m])) {
      const int64_t c_new = cand_cols[m];
      const int64_t p_new = ipos[c_new];
      if (p_new != i) {
        const int64_t c_old = perm[i];
        std::swap(perm[i], perm[p_new]);
        ipos[c_old] = p_new;
        ipos[c_new] = i;
      }
      diag_val = cand_vals[m];
    }
    if (diag_val == 0.0) {
      set_error("zero pivot in row %lld", (long long)i);
      return KRB_EFACTOR;
    }
    // per-row fill limit: the fill_limit largest |v| (stable on ties), kept
    // in their original order
    auto limit = [&](std::vector<int64_t> &idx, std::vector<double> &v) {
      if (fill_limit < 0 || (int64_t)idx.size() <= fill_limit) return;
      std::vector<size_t> order(idx.size());
      for (size_t q = 0; q < order.size(); ++q) order[q] = q;
      std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) {
        return std::fabs(v[a]) > std::fabs(v[b]);
      });
      order.resize((size_t)fill_limit);
      std::sort(order.begin(), order.end());
      std::vector<int64_t> i2;
      std::vector<double> v2;
      for (size_t q : order) {
        i2.push_back(idx[q]);
        v2.push_back(v[q]);
      }
      idx.swap(i2);
      v.swap(v2);
    };
    limit(lp, lv);
    const int64_t pivot_col = perm[i];
    std::vector<int64_t> up_c;
    std::vector<double> up_v;
    for (size_t q = 0; q < cand_cols.size(); ++q)
      if (cand_cols[q] != pivot_col) {
        up_c.push_back(cand_cols[q]);
        up_v.push_back(cand_vals[q]);
      }
    limit(up_c, up_v);
    diag[i] = diag_val;
    u_cols[i].swap(up_c);
    u_vals[i].swap(up_v);
    l_pos[i].swap(lp);
    l_val[i].swap(lv);
  }
  // assemble canonical CSR (ilutp.py:265-279): L with its unit diagonal,
  // U with the pivot on the diagonal and the other columns mapped through
  // the final permutation; columns sorted within each row
  F->n = n;
  F->perm = perm;
  F->Lrp.assign(n + 1, 0);
  F->Urp.assign(n + 1, 0);
  std::vector<std::pair<int64_t, double>> row;
  for (int64_t i = 0; i < n; ++i) {
    row.clear();
    for (size_t q = 0; q < l_pos[i].size(); ++q) row.emplace_back(l_pos[i][q], l_val[i][q]);
    row.emplace_back(i, 1.0);
    std::sort(row.begin(), row.end(),
              [](const std::pair<int64_t, double> &a, const std::pair<int64_t, double> &b) {
                return a.first < b.first;
              });
    for (auto &e : row) {
      F->Lci.push_back((int32_t)e.first);
      F->Lval.push_back(e.second);
    }
    F->Lrp[i + 1] = (int64_t)F->Lci.size();
    row.clear();
    row.emplace_back(i, diag[i]);
    for (size_t q = 0; q < u_cols[i].size(); ++q)
      row.emplace_back(ipos[u_cols[i][q]], u_vals[i][q]);
    std::sort(row.begin(), row.end(),
              [](const std::pair<int64_t, double> &a, const std::pair<int64_t, double> &b) {
                return a.first < b.first;
              });
    for (auto &e : row) {
      F->Uci.push_back((int32_t)e.first);
      F->Uval.push_back(e.second);
    }
    F->Urp[i + 1] = (int64_t)F->Uci.size();
  }
  return KRB_OK;
}

}  // namespace krb

using namespace krb;

extern "C" {

int krb_ilutp_factor(int64_t n, const int64_t *h_row_ptr, const int32_t *h_col_idx,
                     const double *h_values, double drop_tol, double pivot_tol,
                     int64_t fill_limit, krb_ilutp **out) {
  KRB_REQUIRE(out && (n == 0 || (h_row_ptr && h_col_idx && h_values)),
              "krb_ilutp_factor: NULL argument");
  KRB_REQUIRE(n >= 0 && n < ((int64_t)1 << 31), "krb_ilutp_factor: bad n");
  krb_ilutp *F = new krb_ilutp();
  int rc = ilutp_factor_host(n, h_row_ptr, h_col_idx, h_values, drop_tol, pivot_tol,
                             fill_limit, F);
  if (rc != KRB_OK) {
    delete F;
    return rc;
  }
  *out = F;
  return KRB_OK;
}

int krb_ilutp_sizes(const krb_ilutp *F, int64_t *nnz_L, int64_t *nnz_U) {
  KRB_REQUIRE(F != nullptr, "krb_ilutp_sizes: NULL handle");
  if (nnz_L) *nnz_L = (int64_t)F->Lci.size();
  if (nnz_U) *nnz_U = (int64_t)F->Uci.size();
  return KRB_OK;
}

int krb_ilutp_export(const krb_ilutp *F, int64_t *L_rp, int32_t *L_ci, double *L_val,
                     int64_t *U_rp, int32_t *U_ci, double *U_val, int64_t *perm) {
  KRB_REQUIRE(F != nullptr, "krb_ilutp_export: NULL handle");
  auto cp = [](void *dst, const void *src, size_t bytes) {
    if (dst && bytes) std::memcpy(dst, src, bytes);
  };
  cp(L_rp, F->Lrp.data(), sizeof(int64_t) * F->Lrp.size());
  cp(L_ci, F->Lci.data(), sizeof(int32_t) * F->Lci.size());
  cp(L_val, F->Lval.data(), sizeof(double) * F->Lval.size());
  cp(U_rp, F->Urp.data(), sizeof(int64_t) * F->Urp.size());
  cp(U_ci, F->Uci.data(), sizeof(int32_t) * F->Uci.size());
  cp(U_val, F->Uval.data(), sizeof(double) * F->Uval.size());
  cp(perm, F->perm.data(), sizeof(int64_t) * F->perm.size());
  return KRB_OK;
}

int krb_ilutp_free(krb_ilutp *F) {
  delete F;
  return KRB_OK;
}

}  // extern "C"
