// fold_gpu.cu — NEXT-3: the offline fold of ONE layer on the GPU, at the
// calibration sizes the paper uses (§5.1 "Offline rotation matrix computation": the
// Q, K, V vectors of the calibration tokens are consolidated by K-means, then the rotations of
// §4.3 are found; P:1897-1901 reports 7.8-282 min for this step on the paper's hardware).
//
//   1  calibration capture: Q^h = X_c W_Q^h, K^g = X_c W_K^g, V^g = X_c W_V^g      (fp64 GEMM)
//   2  K-means (Lloyd's, reading c21) on each of them -> k centroids            (fp64, deterministic)
//   3  Gram matrices of the stacks of P:989-990 (reading c4 for GQA):
//        G_qk^g = sum_{h in g} C_Q^hT C_Q^h + C_K^gT C_K^g
//        G_vl^g = C_V^gT C_V^g + sum_{h in g} W_O^h W_O^hT      (no K-means for W_L^h)
//   4  cyclic (round-robin parallel) Jacobi eigen-decomposition of every d_h x d_h Gram: the
//      eigenvectors are the right singular vectors R of the stack, sigma = sqrt(eigenvalue); columns
//      sorted by non-increasing sigma, canonical signs (reading c5)
//   5  fold: W_Q^h R_qk, W_K^g R_qk, W_V^g R_vl, R_vl^T W_O^h
// Everything is fp64 (the fold is untimed offline work; B200 keeps full-rate FP64).  Numerics:
// the Gram squares the stack's condition number, so R agrees with the host SVD fold to ~1e-10
// relative on the synthetic spectra (two decades) instead of ~1e-13 (tests/test_gpu_fold.py).
#include "common.cuh"
#include "kernels.h"

#include <algorithm>
#include <cmath>
#include <cstring>

#include "api_util.h"

namespace zdc {

// ---------------------------------------------------------------- fp64 GEMM
// C[m][n] = op(A)[m][k] op(B)[k][n] + beta C[m][n];  op(A)[m][k] = TA ? A[k lda + m] : A[m lda + k],
// op(B)[k][n] = TB ? B[n ldb + k] : B[k ldb + n].  64 x 64 tiles, 16-deep k slices, 4 x 4 per thread.
template <bool TA, bool TB>
__global__ void __launch_bounds__(256) dgemm_kernel(int M, int N, int K, const double* __restrict__ A, int64_t lda,
                                                    const double* __restrict__ B, int64_t ldb, double* __restrict__ C,
                                                    int64_t ldc, double beta) {
  __shared__ double As[16][65], Bs[16][65];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int m0 = blockIdx.y * 64, n0 = blockIdx.x * 64;
  double acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += 16) {
    for (int i = threadIdx.x; i < 16 * 64; i += 256) {
      const int kk = TA ? i / 64 : i % 16, mm = TA ? i % 64 : i / 16;
      const int m = m0 + mm, k = k0 + kk;
      As[kk][mm] = (m < M && k < K) ? (TA ? A[static_cast<int64_t>(k) * lda + m] : A[static_cast<int64_t>(m) * lda + k]) : 0.0;
      const int kb = TB ? i % 16 : i / 64, nn = TB ? i / 16 : i % 64;
      const int n = n0 + nn, k2 = k0 + kb;
      Bs[kb][nn] = (n < N && k2 < K) ? (TB ? B[static_cast<int64_t>(n) * ldb + k2] : B[static_cast<int64_t>(k2) * ldb + n]) : 0.0;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int r = 0; r < 4; ++r) a[r] = As[kk][ty * 4 + r];
#pragma unroll
      for (int c = 0; c < 4; ++c) b[c] = Bs[kk][tx * 4 + c];
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int c = 0; c < 4; ++c) acc[r][c] = fma(a[r], b[c], acc[r][c]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int r = 0; r < 4; ++r)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int m = m0 + ty * 4 + r, n = n0 + tx * 4 + c;
      if (m < M && n < N) {
        double* dst = C + static_cast<int64_t>(m) * ldc + n;
        *dst = beta == 0.0 ? acc[r][c] : acc[r][c] + beta * *dst;
      }
    }
}

template <bool TA, bool TB>
static cudaError_t dgemm(int M, int N, int K, const double* A, int64_t lda, const double* B, int64_t ldb, double* C,
                         int64_t ldc, double beta, cudaStream_t s) {
  dim3 grid((N + 63) / 64, (M + 63) / 64);
  dgemm_kernel<TA, TB><<<grid, 256, 0, s>>>(M, N, K, A, lda, B, ldb, C, ldc, beta);
  ++g_launches;
  return cudaGetLastError();
}

// ---------------------------------------------------------------- K-means (reading c21)
__global__ void km_init_kernel(const double* __restrict__ X, int n, int dim, int k, double* __restrict__ Cm) {
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < static_cast<int64_t>(k) * dim;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int j = static_cast<int>(i / dim), c = static_cast<int>(i - static_cast<int64_t>(j) * dim);
    Cm[i] = X[((static_cast<int64_t>(j) * n) / k) * dim + c];
  }
}

// nearest centroid of each row (squared Euclidean distance, ties -> lowest index): 128 rows per
// CTA in shared memory (padded rows), centroids streamed through shared memory 16 at a time
template <int DMAX>
__global__ void __launch_bounds__(128) km_assign_kernel(const double* __restrict__ X, int n, int dim, int k,
                                                        const double* __restrict__ Cm, int* __restrict__ assign) {
  extern __shared__ double kms[];
  double* xs = kms;                       // [128][dim + 1]
  double* cs = kms + 128 * (dim + 1);     // [16][dim]
  const int r0 = blockIdx.x * 128, t = threadIdx.x;
  for (int i = t; i < 128 * dim; i += 128) {
    const int rr = i / dim, c = i - rr * dim;
    xs[rr * (dim + 1) + c] = r0 + rr < n ? X[static_cast<int64_t>(r0 + rr) * dim + c] : 0.0;
  }
  double best = INFINITY;
  int besti = 0;
  for (int j0 = 0; j0 < k; j0 += 16) {
    const int nj = min(16, k - j0);
    __syncthreads();
    for (int i = t; i < nj * dim; i += 128) cs[i] = Cm[static_cast<int64_t>(j0) * dim + i];
    __syncthreads();
    for (int jj = 0; jj < nj; ++jj) {
      double dsum = 0.0;
      const double* xr = xs + t * (dim + 1);
      const double* cr = cs + jj * dim;
      for (int c = 0; c < dim; ++c) {
        const double df = xr[c] - cr[c];
        dsum = fma(df, df, dsum);
      }
      if (dsum < best) {  // strict: the first (lowest-index) minimum is kept
        best = dsum;
        besti = j0 + jj;
      }
    }
  }
  if (r0 + t < n) assign[r0 + t] = besti;
}

// centroid j = mean of its rows (fixed summation order: deterministic); empty -> unchanged
__global__ void __launch_bounds__(256) km_update_kernel(const double* __restrict__ X, int n, int dim,
                                                        const int* __restrict__ assign, double* __restrict__ Cm) {
  __shared__ double red[256];
  __shared__ int cnt_s[256];
  const int j = blockIdx.x, t = threadIdx.x;
  for (int c = 0; c < dim; ++c) {
    double sum = 0.0;
    int cnt = 0;
    for (int i = t; i < n; i += 256)
      if (assign[i] == j) {
        sum += X[static_cast<int64_t>(i) * dim + c];
        ++cnt;
      }
    red[t] = sum;
    cnt_s[t] = cnt;
    __syncthreads();
    for (int off = 128; off > 0; off >>= 1) {
      if (t < off) {
        red[t] += red[t + off];
        cnt_s[t] += cnt_s[t + off];
      }
      __syncthreads();
    }
    if (t == 0 && cnt_s[0] > 0) Cm[static_cast<int64_t>(j) * dim + c] = red[0] / cnt_s[0];
    __syncthreads();
  }
}

// ---------------------------------------------------------------- Jacobi eigen-decomposition
// One CTA per symmetric n x n matrix (n even, <= 128), A in shared memory.  Round r pairs index
// n-1 with r and (r+i) mod (n-1) with (r-i) mod (n-1): n/2 disjoint rotations per round, applied
// as J^T A J (Golub & Van Loan, symmetric Schur) to rows, then columns, and to V.
__global__ void __launch_bounds__(512) jacobi_eig_kernel(const double* __restrict__ G, int n, double* __restrict__ Vout,
                                                         double* __restrict__ sigma) {
  extern __shared__ double jsm[];
  const int ld = n + 1;
  double* A = jsm;                     // [n][n+1]
  double* cs = A + n * ld;             // [n/2] c
  double* sn = cs + n / 2;             // [n/2] s
  int* pp = reinterpret_cast<int*>(sn + n / 2);
  int* qq = pp + n / 2;
  __shared__ double red[512];
  const double* Gm = G + static_cast<int64_t>(blockIdx.x) * n * n;
  double* V = Vout + static_cast<int64_t>(blockIdx.x) * n * n;
  const int t = threadIdx.x, nt = blockDim.x, half = n / 2;
  for (int i = t; i < n * n; i += nt) {
    const int r = i / n, c = i - r * n;
    A[r * ld + c] = Gm[i];
    V[i] = r == c ? 1.0 : 0.0;
  }
  __syncthreads();
  for (int sweep = 0; sweep < 40; ++sweep) {
    double off = 0.0, dia = 0.0;
    for (int i = t; i < n * n; i += nt) {
      const int r = i / n, c = i - r * n;
      const double v = A[r * ld + c];
      if (r != c) off += v * v; else dia += v * v;
    }
    red[t] = off;
    __syncthreads();
    for (int o = nt / 2; o > 0; o >>= 1) {
      if (t < o) red[t] += red[t + o];
      __syncthreads();
    }
    const double off_tot = red[0];
    __syncthreads();
    red[t] = dia;
    __syncthreads();
    for (int o = nt / 2; o > 0; o >>= 1) {
      if (t < o) red[t] += red[t + o];
      __syncthreads();
    }
    const double dia_tot = red[0];
    __syncthreads();
    if (off_tot <= 1e-32 * dia_tot || off_tot == 0.0) break;
    for (int r = 0; r < n - 1; ++r) {
      for (int i = t; i < half; i += nt) {
        int p, q;
        if (i == 0) {
          p = r;
          q = n - 1;
        } else {
          p = (r + i) % (n - 1);
          q = (r - i + (n - 1)) % (n - 1);
        }
        if (p > q) { const int tmp = p; p = q; q = tmp; }
        const double apq = A[p * ld + q];
        double c = 1.0, s = 0.0;
        if (apq != 0.0) {
          const double tau = (A[q * ld + q] - A[p * ld + p]) / (2.0 * apq);
          const double tt = (tau >= 0.0 ? 1.0 : -1.0) / (fabs(tau) + sqrt(1.0 + tau * tau));
          c = 1.0 / sqrt(1.0 + tt * tt);
          s = tt * c;
        }
        pp[i] = p;
        qq[i] = q;
        cs[i] = c;
        sn[i] = s;
      }
      __syncthreads();
      for (int i = t; i < half * n; i += nt) {  // rows: A <- J^T A
        const int pr = i / n, j = i - pr * n;
        const int p = pp[pr], q = qq[pr];
        const double c = cs[pr], s = sn[pr];
        const double ap = A[p * ld + j], aq = A[q * ld + j];
        A[p * ld + j] = c * ap - s * aq;
        A[q * ld + j] = s * ap + c * aq;
      }
      __syncthreads();
      for (int i = t; i < half * n; i += nt) {  // columns: A <- A J, V <- V J
        const int pr = i / n, j = i - pr * n;
        const int p = pp[pr], q = qq[pr];
        const double c = cs[pr], s = sn[pr];
        const double ap = A[j * ld + p], aq = A[j * ld + q];
        A[j * ld + p] = c * ap - s * aq;
        A[j * ld + q] = s * ap + c * aq;
        const double vp = V[j * n + p], vq = V[j * n + q];
        V[j * n + p] = c * vp - s * vq;
        V[j * n + q] = s * vp + c * vq;
      }
      __syncthreads();
    }
  }
  // order by non-increasing eigenvalue (stable), sigma = sqrt(max(lambda, 0)), canonical signs
  int* order = pp;  // reuse (n/2 + n/2 ints = n)
  if (t == 0) {
    for (int i = 0; i < n; ++i) order[i] = i;
    for (int i = 1; i < n; ++i) {  // insertion sort, descending, stable
      const int o = order[i];
      const double lv = A[o * ld + o];
      int j = i - 1;
      while (j >= 0 && A[order[j] * ld + order[j]] < lv) {
        order[j + 1] = order[j];
        --j;
      }
      order[j + 1] = o;
    }
  }
  __syncthreads();
  double* Vs = A;  // A's diagonal is read below before being overwritten: stage eigenvalues first
  double* lam = cs;  // n doubles (cs + sn region)
  for (int i = t; i < n; i += nt) lam[i] = A[order[i] * ld + order[i]];
  __syncthreads();
  for (int i = t; i < n * n; i += nt) {
    const int r = i / n, c = i - r * n;
    Vs[r * ld + c] = V[r * n + order[c]];
  }
  __syncthreads();
  for (int c = t; c < n; c += nt) {
    int im = 0;
    double vm = fabs(Vs[c]);
    for (int r = 1; r < n; ++r)
      if (fabs(Vs[r * ld + c]) > vm) {  // strict: the lowest row on ties
        vm = fabs(Vs[r * ld + c]);
        im = r;
      }
    const double sg = Vs[im * ld + c] < 0.0 ? -1.0 : 1.0;
    for (int r = 0; r < n; ++r) V[r * n + c] = sg * Vs[r * ld + c];
    sigma[static_cast<int64_t>(blockIdx.x) * n + c] = sqrt(fmax(lam[c], 0.0));
  }
}

}  // namespace zdc

using namespace zdc;

namespace {

int64_t fold_ws_bytes(const zdc_dims* d, int64_t n_calib, int32_t k) {
  const int64_t dh = d->d_head;
  const int64_t kk = k > 0 && k < n_calib ? k : 0;
  auto al = [](int64_t x) { return (x + 255) / 256 * 256; };
  return al(n_calib * dh * 8) + al(n_calib * 4) + al(kk * dh * 8) + al(2LL * d->n_kv_heads * dh * dh * 8);
}

}  // namespace

extern "C" {

int64_t zdc_fold_gpu_workspace(const zdc_dims* dims, int64_t n_calib, int32_t k_clusters) {
  if (!dims || n_calib <= 0) return -1;
  return fold_ws_bytes(dims, n_calib, k_clusters);
}

zdc_status zdc_fold_weights_gpu(const zdc_dims* dims, const double* wq, const double* wk, const double* wv,
                                const double* wo, const double* calib_x, int64_t n_calib, int32_t k_clusters,
                                int32_t kmeans_iters, double* r_qk, double* r_vl, double* sigma_qk, double* sigma_vl,
                                double* wq_f, double* wk_f, double* wv_f, double* wo_f, void* workspace,
                                int64_t workspace_bytes, void* stream) {
  if (!dims || !wq || !wk || !wv || !wo || !calib_x || !r_qk || !r_vl || !sigma_qk || !sigma_vl || !wq_f || !wk_f ||
      !wv_f || !wo_f || !workspace)
    return fail(ZDC_ERR_INVALID_ARG, "zdc_fold_weights_gpu: null argument");
  const int d = dims->d_model, nh = dims->n_heads, nkv = dims->n_kv_heads, dh = dims->d_head;
  if (d <= 0 || nh <= 0 || nkv <= 0 || dh <= 0 || nh % nkv != 0)
    return fail(ZDC_ERR_SHAPE, "zdc_fold_weights_gpu: dims d=%d n_heads=%d n_kv_heads=%d d_head=%d", d, nh, nkv, dh);
  if (dh % 2 != 0 || dh > 128)
    return fail(ZDC_ERR_UNSUPPORTED, "zdc_fold_weights_gpu: d_head %d (even, <= 128)", dh);
  const int G = nh / nkv;
  const int64_t rows = k_clusters > 0 && k_clusters < n_calib ? k_clusters : n_calib;
  if (n_calib <= 0 || rows * (G + 1) < dh)
    return fail(ZDC_ERR_SHAPE, "zdc_fold_weights_gpu: insufficient samples: %lld rows x (G+1) < d_head %d",
                static_cast<long long>(rows), dh);
  if (n_calib > (1LL << 31) - 1) return fail(ZDC_ERR_SHAPE, "zdc_fold_weights_gpu: n_calib too large");
  if (workspace_bytes < fold_ws_bytes(dims, n_calib, k_clusters))
    return fail(ZDC_ERR_CAPACITY, "zdc_fold_weights_gpu: workspace %lld < %lld bytes",
                static_cast<long long>(workspace_bytes), static_cast<long long>(fold_ws_bytes(dims, n_calib, k_clusters)));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int n = static_cast<int>(n_calib);
  const bool km = k_clusters > 0 && k_clusters < n;
  auto al = [](int64_t x) { return (x + 255) / 256 * 256; };
  uint8_t* ws = static_cast<uint8_t*>(workspace);
  double* P = reinterpret_cast<double*>(ws);
  int* assign = reinterpret_cast<int*>(ws + al(static_cast<int64_t>(n) * dh * 8));
  double* Cm = reinterpret_cast<double*>(reinterpret_cast<uint8_t*>(assign) + al(static_cast<int64_t>(n) * 4));
  double* gram = reinterpret_cast<double*>(reinterpret_cast<uint8_t*>(Cm) + al((km ? k_clusters : 0) * static_cast<int64_t>(dh) * 8));
  double* gqk = gram;                                            // [nkv][dh][dh]
  double* gvl = gram + static_cast<int64_t>(nkv) * dh * dh;      // [nkv][dh][dh]
  g_launches = 0;
  ZDC_CUDA_TRY(cudaMemsetAsync(gram, 0, 2ULL * nkv * dh * dh * 8, s));
  const size_t asm_bytes = (128 * (dh + 1) + 16 * dh) * sizeof(double);
  static bool attr = false;
  if (!attr) {
    // the largest dynamic shared memory either kernel takes (d_head = 128)
    ZDC_CUDA_TRY(cudaFuncSetAttribute(km_assign_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>((128 * 129 + 16 * 128) * sizeof(double))));
    ZDC_CUDA_TRY(cudaFuncSetAttribute(jacobi_eig_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      static_cast<int>((128 * 129 + 128) * sizeof(double) + 128 * sizeof(int))));
    attr = true;
  }
  // one projected block (n x dh, ld_w = the weight's row length) -> optional K-means -> Gram += B^T B
  auto block = [&](const double* w, int64_t ld_w, double* g) -> zdc_status {
    if (cudaError_t e = dgemm<false, false>(n, dh, d, calib_x, d, w, ld_w, P, dh, 0.0, s))
      return fail(ZDC_ERR_CUDA, "fold gpu projection: %s", cudaGetErrorString(e));
    const double* Bm = P;
    int rows_b = n;
    if (km) {
      km_init_kernel<<<64, 256, 0, s>>>(P, n, dh, k_clusters, Cm);
      for (int it = 0; it < kmeans_iters; ++it) {
        km_assign_kernel<128><<<(n + 127) / 128, 128, asm_bytes, s>>>(P, n, dh, k_clusters, Cm, assign);
        km_update_kernel<<<k_clusters, 256, 0, s>>>(P, n, dh, assign, Cm);
      }
      g_launches += 1 + 2 * kmeans_iters;
      Bm = Cm;
      rows_b = k_clusters;
    }
    if (cudaError_t e = dgemm<true, false>(dh, dh, rows_b, Bm, dh, Bm, dh, g, dh, 1.0, s))
      return fail(ZDC_ERR_CUDA, "fold gpu gram: %s", cudaGetErrorString(e));
    return ZDC_OK;
  };
  for (int h = 0; h < nh; ++h)
    if (zdc_status st = block(wq + static_cast<int64_t>(h) * dh, static_cast<int64_t>(nh) * dh,
                              gqk + static_cast<int64_t>(h / G) * dh * dh))
      return st;
  for (int g = 0; g < nkv; ++g) {
    if (zdc_status st = block(wk + static_cast<int64_t>(g) * dh, static_cast<int64_t>(nkv) * dh,
                              gqk + static_cast<int64_t>(g) * dh * dh))
      return st;
    if (zdc_status st = block(wv + static_cast<int64_t>(g) * dh, static_cast<int64_t>(nkv) * dh,
                              gvl + static_cast<int64_t>(g) * dh * dh))
      return st;
  }
  for (int h = 0; h < nh; ++h) {  // + W_O^h W_O^hT (the d rows of W_L^h: no K-means)
    const double* woh = wo + static_cast<int64_t>(h) * dh * d;
    ZDC_CUDA_TRY((dgemm<false, true>(dh, dh, d, woh, d, woh, d, gvl + static_cast<int64_t>(h / G) * dh * dh, dh, 1.0, s)));
  }
  // eigen-decompositions: [R_qk of every group][R_vl of every group] -> the output arrays
  const size_t jsm = (static_cast<size_t>(dh) * (dh + 1) + dh) * sizeof(double) + dh * sizeof(int);
  jacobi_eig_kernel<<<nkv, 512, jsm, s>>>(gqk, dh, r_qk, sigma_qk);
  jacobi_eig_kernel<<<nkv, 512, jsm, s>>>(gvl, dh, r_vl, sigma_vl);
  g_launches += 2;
  ZDC_CUDA_TRY(cudaGetLastError());
  // fold
  for (int h = 0; h < nh; ++h) {
    const int g = h / G;
    const double* Rq = r_qk + static_cast<int64_t>(g) * dh * dh;
    const double* Rv = r_vl + static_cast<int64_t>(g) * dh * dh;
    ZDC_CUDA_TRY((dgemm<false, false>(d, dh, dh, wq + static_cast<int64_t>(h) * dh, static_cast<int64_t>(nh) * dh, Rq,
                                     dh, wq_f + static_cast<int64_t>(h) * dh, static_cast<int64_t>(nh) * dh, 0.0, s)));
    ZDC_CUDA_TRY((dgemm<true, false>(dh, d, dh, Rv, dh, wo + static_cast<int64_t>(h) * dh * d, d,
                                    wo_f + static_cast<int64_t>(h) * dh * d, d, 0.0, s)));
  }
  for (int g = 0; g < nkv; ++g) {
    const double* Rq = r_qk + static_cast<int64_t>(g) * dh * dh;
    const double* Rv = r_vl + static_cast<int64_t>(g) * dh * dh;
    ZDC_CUDA_TRY((dgemm<false, false>(d, dh, dh, wk + static_cast<int64_t>(g) * dh, static_cast<int64_t>(nkv) * dh, Rq,
                                     dh, wk_f + static_cast<int64_t>(g) * dh, static_cast<int64_t>(nkv) * dh, 0.0, s)));
    ZDC_CUDA_TRY((dgemm<false, false>(d, dh, dh, wv + static_cast<int64_t>(g) * dh, static_cast<int64_t>(nkv) * dh, Rv,
                                     dh, wv_f + static_cast<int64_t>(g) * dh, static_cast<int64_t>(nkv) * dh, 0.0, s)));
  }
  return ZDC_OK;
}

}  // extern "C"
