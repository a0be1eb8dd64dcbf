// fold.cpp — zdc_fold_weights: the offline, host-side, fp64 fold of ONE layer (not timed).
//
// P:977, P:989-990 (§4.3): per head — here per KV group g (reading c4) — find a common rotation
// R for the QK pair from the stacked [Q^h (h in group); K^g] (2 Sigma_S x d_h in MHA) and for the
// VW_L pair from [V^g; (W_O^h)^T (h in group)] ((Sigma_S + d) x d_h), where Q^h = X_c W_Q^h
// (Eq. 1).  R = right singular vectors of the stack (A = U Sigma R^T, §2.2), columns
// sorted by non-increasing sigma, canonical signs (reading c5).  Then fold (P:1204,
// P:1218-1219): W_Q^{R,h} = W_Q^h R_qk, W_K^{R,g} = W_K^g R_qk, W_V^{R,g} = W_V^g R_vl,
// W_O^{R,h} = R_vl^T W_O^h (reading c1).
//
// Numerics: the stack is never formed as a Gram matrix.  Each block is reduced by Householder
// QR, the triangular factors are stacked and reduced again (TSQR), and the d_h x d_h factor goes
// through one-sided Jacobi (Hestenes), which keeps small singular values to high relative accuracy.
#include <omp.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "api_util.h"

namespace {

// C[m][n] (+)= A[m][k] * B[k][n]; row-major with leading dimensions.  Cache-blocked, 4x8
// register micro-tiles, OpenMP over C tiles.
void dgemm(int m, int n, int k, const double* A, int64_t lda, const double* B, int64_t ldb, double* C, int64_t ldc) {
  constexpr int MC = 64, NC = 256, KC = 256;
  const int mt = (m + MC - 1) / MC, nt = (n + NC - 1) / NC;
#pragma omp parallel for collapse(2) schedule(dynamic)
  for (int ti = 0; ti < mt; ++ti)
    for (int tj = 0; tj < nt; ++tj) {
      const int i0 = ti * MC, i1 = std::min(m, i0 + MC);
      const int j0 = tj * NC, j1 = std::min(n, j0 + NC);
      for (int i = i0; i < i1; ++i)
        for (int j = j0; j < j1; ++j) C[i * ldc + j] = 0.0;
      for (int k0 = 0; k0 < k; k0 += KC) {
        const int k1 = std::min(k, k0 + KC);
        for (int jj = j0; jj < j1; jj += 8) {
          const int jw = std::min(8, j1 - jj);
          for (int ii = i0; ii < i1; ii += 4) {
            const int iw = std::min(4, i1 - ii);
            if (iw == 4 && jw == 8) {
              double c[4][8] = {};
              for (int kk = k0; kk < k1; ++kk) {
                const double* b = B + kk * ldb + jj;
                const double a0 = A[(ii + 0) * lda + kk], a1 = A[(ii + 1) * lda + kk];
                const double a2 = A[(ii + 2) * lda + kk], a3 = A[(ii + 3) * lda + kk];
#pragma GCC unroll 8
                for (int j = 0; j < 8; ++j) {
                  c[0][j] += a0 * b[j];
                  c[1][j] += a1 * b[j];
                  c[2][j] += a2 * b[j];
                  c[3][j] += a3 * b[j];
                }
              }
              for (int r = 0; r < 4; ++r)
                for (int j = 0; j < 8; ++j) C[(ii + r) * ldc + jj + j] += c[r][j];
            } else {
              for (int r = 0; r < iw; ++r)
                for (int kk = k0; kk < k1; ++kk) {
                  const double a = A[(ii + r) * lda + kk];
                  for (int j = 0; j < jw; ++j) C[(ii + r) * ldc + jj + j] += a * B[kk * ldb + jj + j];
                }
            }
          }
        }
      }
    }
}

// Householder QR of the m x n (m >= n) row-major matrix A (in place); the upper triangle of the
// first n rows becomes R (sign convention irrelevant: R^T R = A^T A).
void householder_r(double* A, int m, int n) {
  std::vector<double> v(m);
  for (int j = 0; j < n; ++j) {
    double norm2 = 0.0;
    for (int i = j; i < m; ++i) norm2 += A[i * n + j] * A[i * n + j];
    const double norm = std::sqrt(norm2);
    if (norm == 0.0) continue;
    const double alpha = A[j * n + j] > 0 ? -norm : norm;
    for (int i = j; i < m; ++i) v[i] = A[i * n + j];
    v[j] -= alpha;
    double vnorm2 = norm2 - A[j * n + j] * A[j * n + j] + v[j] * v[j];
    if (vnorm2 == 0.0) continue;
    for (int c = j; c < n; ++c) {
      double dot = 0.0;
      for (int i = j; i < m; ++i) dot += v[i] * A[i * n + c];
      const double f = 2.0 * dot / vnorm2;
      for (int i = j; i < m; ++i) A[i * n + c] -= f * v[i];
    }
  }
}

// Reduce a stack of row blocks to its n x n triangular factor, one block at a time (TSQR).
struct StackR {
  int n;
  std::vector<double> R;  // n x n
  bool empty = true;
  explicit StackR(int n_) : n(n_), R(static_cast<size_t>(n_) * n_, 0.0) {}
  void add(const double* block, int rows, int64_t ld) {
    std::vector<double> buf(static_cast<size_t>(rows + n) * n, 0.0);
    int off = 0;
    if (!empty) {
      std::memcpy(buf.data(), R.data(), sizeof(double) * n * n);
      off = n;
    }
    for (int i = 0; i < rows; ++i) std::memcpy(&buf[static_cast<size_t>(off + i) * n], block + i * ld, sizeof(double) * n);
    const int m = off + rows;
    if (m < n) {  // not enough rows yet for a square factor: keep the raw rows in R's slots
      std::fill(R.begin(), R.end(), 0.0);
      std::memcpy(R.data(), buf.data(), sizeof(double) * m * n);
      empty = false;
      return;
    }
    householder_r(buf.data(), m, n);
    for (int i = 0; i < n; ++i)
      for (int c = 0; c < n; ++c) R[i * n + c] = c >= i ? buf[static_cast<size_t>(i) * n + c] : 0.0;
    empty = false;
  }
};

// One-sided Jacobi SVD of the n x n matrix A (row-major): returns sigma (unsorted) and V with
// A V = U diag(sigma).  Returns false if 60 sweeps do not converge.
bool jacobi_svd(std::vector<double>& A, int n, std::vector<double>& sigma, std::vector<double>& V) {
  V.assign(static_cast<size_t>(n) * n, 0.0);
  for (int i = 0; i < n; ++i) V[i * n + i] = 1.0;
  // work on columns: transpose to column-major for contiguous column access
  std::vector<double> Ac(static_cast<size_t>(n) * n), Vc(static_cast<size_t>(n) * n, 0.0);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) Ac[j * n + i] = A[i * n + j];
  for (int i = 0; i < n; ++i) Vc[i * n + i] = 1.0;
  const double eps = 1e-15;
  bool converged = false;
  for (int sweep = 0; sweep < 60 && !converged; ++sweep) {
    converged = true;
    for (int p = 0; p < n - 1; ++p)
      for (int q = p + 1; q < n; ++q) {
        double* ap = &Ac[p * n];
        double* aq = &Ac[q * n];
        double alpha = 0, beta = 0, gamma = 0;
        for (int i = 0; i < n; ++i) {
          alpha += ap[i] * ap[i];
          beta += aq[i] * aq[i];
          gamma += ap[i] * aq[i];
        }
        if (gamma == 0.0 || std::fabs(gamma) <= eps * std::sqrt(alpha * beta)) continue;
        converged = false;
        const double zeta = (beta - alpha) / (2.0 * gamma);
        const double t = (zeta >= 0 ? 1.0 : -1.0) / (std::fabs(zeta) + std::sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / std::sqrt(1.0 + t * t), s = c * t;
        double* vp = &Vc[p * n];
        double* vq = &Vc[q * n];
        for (int i = 0; i < n; ++i) {
          const double x = ap[i], y = aq[i];
          ap[i] = c * x - s * y;
          aq[i] = s * x + c * y;
          const double u = vp[i], w = vq[i];
          vp[i] = c * u - s * w;
          vq[i] = s * u + c * w;
        }
      }
  }
  sigma.assign(n, 0.0);
  for (int j = 0; j < n; ++j) {
    double s2 = 0;
    for (int i = 0; i < n; ++i) s2 += Ac[j * n + i] * Ac[j * n + i];
    sigma[j] = std::sqrt(s2);
  }
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) V[i * n + j] = Vc[j * n + i];  // column j = right singular vector j
  return converged;
}

// Sort by non-increasing sigma and fix canonical signs (reading c5).  R out: [n][n], column j.
void finish_rotation(const std::vector<double>& sigma, const std::vector<double>& V, int n, double* R_out,
                     double* sig_out) {
  std::vector<int> order(n);
  for (int i = 0; i < n; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return sigma[a] > sigma[b]; });
  for (int j = 0; j < n; ++j) {
    const int src = order[j];
    sig_out[j] = sigma[src];
    int imax = 0;
    double vmax = -1.0;
    for (int i = 0; i < n; ++i) {
      const double av = std::fabs(V[i * n + src]);
      if (av > vmax) vmax = av, imax = i;
    }
    const double sgn = V[imax * n + src] < 0 ? -1.0 : 1.0;
    for (int i = 0; i < n; ++i) R_out[i * n + j] = sgn * V[i * n + src];
  }
}

bool all_finite(const double* p, int64_t n) {
  for (int64_t i = 0; i < n; ++i)
    if (!std::isfinite(p[i])) return false;
  return true;
}

}  // namespace

extern "C" zdc_status zdc_fold_weights(const zdc_dims* dims, const double* wq, const double* wk, const double* wv,
                                       const double* wo, const double* xc, int64_t n_calib, double* r_qk,
                                       double* r_vl, double* sigma_qk, double* sigma_vl, double* wq_f, double* wk_f,
                                       double* wv_f, double* wo_f) {
  using zdc::fail;
  if (!dims || !wq || !wk || !wv || !wo || !xc || !r_qk || !r_vl || !sigma_qk || !sigma_vl || !wq_f || !wk_f ||
      !wv_f || !wo_f)
    return fail(ZDC_ERR_INVALID_ARG, "zdc_fold_weights: null argument");
  const int d = dims->d_model, Nh = dims->n_heads, Nkv = dims->n_kv_heads, dh = dims->d_head;
  if (d <= 0 || Nh <= 0 || Nkv <= 0 || dh <= 0 || Nh % Nkv != 0)
    return fail(ZDC_ERR_SHAPE, "zdc_fold_weights: dims d=%d Nh=%d Nkv=%d dh=%d", d, Nh, Nkv, dh);
  const int G = Nh / Nkv;
  if (n_calib <= 0 || n_calib * (G + 1) < dh)
    return fail(ZDC_ERR_SHAPE, "zdc_fold_weights: insufficient samples: n_calib %lld * (G+1) < d_head %d",
                static_cast<long long>(n_calib), dh);
  const int64_t nq = static_cast<int64_t>(Nh) * dh, nk = static_cast<int64_t>(Nkv) * dh;
  if (!all_finite(wq, d * nq) || !all_finite(wk, d * nk) || !all_finite(wv, d * nk) || !all_finite(wo, nq * d) ||
      !all_finite(xc, n_calib * d))
    return fail(ZDC_ERR_INVALID_ARG, "zdc_fold_weights: non-finite input");
  const int n = static_cast<int>(n_calib);

  // Eq. 1 on the calibration rows: Q = X_c W_Q, K = X_c W_K, V = X_c W_V
  std::vector<double> XQ(static_cast<size_t>(n) * nq), XK(static_cast<size_t>(n) * nk),
      XV(static_cast<size_t>(n) * nk);
  dgemm(n, static_cast<int>(nq), d, xc, d, wq, nq, XQ.data(), nq);
  dgemm(n, static_cast<int>(nk), d, xc, d, wk, nk, XK.data(), nk);
  dgemm(n, static_cast<int>(nk), d, xc, d, wv, nk, XV.data(), nk);

  int bad = 0;
  double worst_orth = 0.0;
#pragma omp parallel for schedule(dynamic) reduction(| : bad) reduction(max : worst_orth)
  for (int g = 0; g < Nkv; ++g) {
    for (int pair = 0; pair < 2; ++pair) {
      StackR st(dh);
      if (pair == 0) {
        for (int h = g * G; h < (g + 1) * G; ++h) st.add(XQ.data() + static_cast<int64_t>(h) * dh, n, nq);
        st.add(XK.data() + static_cast<int64_t>(g) * dh, n, nk);
      } else {
        st.add(XV.data() + static_cast<int64_t>(g) * dh, n, nk);
        std::vector<double> wot(static_cast<size_t>(d) * dh);
        for (int h = g * G; h < (g + 1) * G; ++h) {
          for (int c = 0; c < dh; ++c)
            for (int j = 0; j < d; ++j) wot[static_cast<size_t>(j) * dh + c] = wo[(static_cast<int64_t>(h) * dh + c) * d + j];
          st.add(wot.data(), d, dh);
        }
      }
      std::vector<double> sig, V;
      if (!jacobi_svd(st.R, dh, sig, V)) bad |= 1;
      double* R = (pair == 0 ? r_qk : r_vl) + static_cast<int64_t>(g) * dh * dh;
      double* S = (pair == 0 ? sigma_qk : sigma_vl) + static_cast<int64_t>(g) * dh;
      finish_rotation(sig, V, dh, R, S);
      for (int a = 0; a < dh; ++a)
        for (int b = 0; b < dh; ++b) {
          double s = 0;
          for (int i = 0; i < dh; ++i) s += R[i * dh + a] * R[i * dh + b];
          worst_orth = std::max(worst_orth, std::fabs(s - (a == b ? 1.0 : 0.0)));
        }
    }
  }
  if (bad) return fail(ZDC_ERR_NO_CONVERGENCE, "zdc_fold_weights: one-sided Jacobi did not converge in 60 sweeps");
  if (worst_orth > 1e-10)
    return fail(ZDC_ERR_NOT_ORTHONORMAL, "zdc_fold_weights: |R^T R - I| = %g > 1e-10", worst_orth);

  // fold: W_Q^h R_qk, W_K^g R_qk, W_V^g R_vl (d x dh times dh x dh), R_vl^T W_O^h (dh x dh times dh x d)
#pragma omp parallel for schedule(static)
  for (int j = 0; j < d; ++j) {
    for (int h = 0; h < Nh; ++h) {
      const double* R = r_qk + static_cast<int64_t>(h / G) * dh * dh;
      const double* src = wq + static_cast<int64_t>(j) * nq + h * dh;
      double* dst = wq_f + static_cast<int64_t>(j) * nq + h * dh;
      for (int c = 0; c < dh; ++c) dst[c] = 0.0;
      for (int i = 0; i < dh; ++i) {
        const double a = src[i];
        for (int c = 0; c < dh; ++c) dst[c] += a * R[i * dh + c];
      }
    }
    for (int g = 0; g < Nkv; ++g)
      for (int pair = 0; pair < 2; ++pair) {
        const double* R = (pair == 0 ? r_qk : r_vl) + static_cast<int64_t>(g) * dh * dh;
        const double* src = (pair == 0 ? wk : wv) + static_cast<int64_t>(j) * nk + g * dh;
        double* dst = (pair == 0 ? wk_f : wv_f) + static_cast<int64_t>(j) * nk + g * dh;
        for (int c = 0; c < dh; ++c) dst[c] = 0.0;
        for (int i = 0; i < dh; ++i) {
          const double a = src[i];
          for (int c = 0; c < dh; ++c) dst[c] += a * R[i * dh + c];
        }
      }
  }
#pragma omp parallel for schedule(static)
  for (int h = 0; h < Nh; ++h) {
    const double* R = r_vl + static_cast<int64_t>(h / G) * dh * dh;
    for (int c = 0; c < dh; ++c) {
      double* dst = wo_f + (static_cast<int64_t>(h) * dh + c) * d;
      for (int j = 0; j < d; ++j) dst[j] = 0.0;
      for (int i = 0; i < dh; ++i) {
        const double a = R[i * dh + c];  // (R^T)[c][i]
        const double* src = wo + (static_cast<int64_t>(h) * dh + i) * d;
        for (int j = 0; j < d; ++j) dst[j] += a * src[j];
      }
    }
  }
  return ZDC_OK;
}
