"""ZDC fp64 CPU ORACLE — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
legs may import this module.  The product path (paper_2408_04107_b200/, libzdc.so)
never imports, links or executes it, and shares no code with it.

A plain, slow, obviously-correct fp64 implementation of ZDC's hot path
(arxiv 2408.04107, /root/reference/PAPER.md), written in the paper's order and
notation.  Citations are "P:<line>" = PAPER.md line, with section/equation.

Contents
  softmax_rows      Eq. 3 row softmax with its denominator
  svd_right         A = U Sigma R^T, right vectors + singular values   P:300 (§2.2)
  fold_layer        common R per head from history; fold R into W     P:977, P:989-990 (§4.3), P:1204, P:1218-1219 (§5.1)
  truncate_layer    drop the right p fraction of columns / rows       P:862-864 (Lemma 1)
  unfolded_forward  plain Eqs. 1-4 of the uncompressed model
  importance        sum_h sum_{k<=t} exp(s_k^h), in the log domain    P:1442 (§5.2)
  select_important  sort descending, top g^l fraction important
  OracleModel       prefill / decode over a compressed KV cache, with
                    zero-filled unimportant rows and layer groups     P:774-776 (DEL)
  kmeans            K-means consolidation of calibration vectors      P:1157-1167 (§5.1 offline computation)
  e4m3 / quantize_rows  FP8 (E4M3) compressed KV cache, GEAR-ZDC      P:1642 (DEL), P:1606 (§6 compared methods)
  layer_groups      layers sharing the representative's classes       P:1455-1456 (repetition ratio > 95%)

Readings of silent / ambiguous points are DESIGN.md §3 (c1..c19), cited inline.
Every function here is pinned by tests/test_oracle_pins.py (P1-P13) except where a
docstring says "parity unpinned".

BF16-faithful mode (`faithful=True`): rounds to BF16 (RNE) at exactly the points
the GPU kernels round (DESIGN.md §3 "rounding points"): folded truncated weights,
Q'/K'/V' after projection, unnormalised P = exp(s - m) before PV (row sum from the
unrounded P), O' after division by l, and y.  fp64 everywhere else.
"""
from __future__ import annotations

import math
from typing import Dict, List, Optional

import numpy as np

NEG_INF = -math.inf


# --------------------------------------------------------------------------------------
# BF16 rounding (the oracle's own; shares nothing with the library or zdc_synth)
# --------------------------------------------------------------------------------------
def bf16(a: np.ndarray) -> np.ndarray:
    """Round fp64 -> fp32 -> bf16 (round-to-nearest-even), returned as fp64."""
    f = np.ascontiguousarray(np.asarray(a, dtype=np.float64), dtype=np.float32)
    bits = f.view(np.uint32).astype(np.uint64)
    lsb = (bits >> 16) & 1
    bits = (bits + 0x7FFF + lsb) & 0xFFFF0000
    return bits.astype(np.uint32).view(np.float32).astype(np.float64)


# --------------------------------------------------------------------------------------
# FP8 E4M3 (the oracle's own; OCP 8-bit "e4m3fn": bias 7, 3 mantissa bits, no infinities,
# largest finite 448, smallest subnormal 2^-9) for the quantized compressed cache of NEXT-4
# --------------------------------------------------------------------------------------
def _e4m3_table():
    vals, codes = [], []
    for code in range(0x7F):          # 0x7F is NaN; non-negative codes only
        e, m = code >> 3, code & 7
        v = (m / 8.0) * 2.0 ** -6 if e == 0 else (1.0 + m / 8.0) * 2.0 ** (e - 7)
        vals.append(v)
        codes.append(code)
    return np.array(vals), np.array(codes)


_E4M3_VALS, _E4M3_CODES = _e4m3_table()


def e4m3(a) -> np.ndarray:
    """Round to the nearest E4M3 value, ties to the even code (round-to-nearest-even), magnitudes
    above 448 saturate to 448 (reading c23: the GPU converts with RNE + satfinite).  Returns the
    E4M3 value as fp64 (the sign is kept, so -0 stays -0)."""
    a = np.asarray(a, dtype=np.float64)
    mag = np.minimum(np.abs(a), 448.0)
    idx = np.searchsorted(_E4M3_VALS, mag)              # first table value >= mag
    hi = np.minimum(idx, len(_E4M3_VALS) - 1)
    lo = np.maximum(idx - 1, 0)
    dlo = mag - _E4M3_VALS[lo]
    dhi = _E4M3_VALS[hi] - mag
    pick_hi = (dhi < dlo) | ((dhi == dlo) & (_E4M3_CODES[hi] % 2 == 0))
    out = np.where(pick_hi, _E4M3_VALS[hi], _E4M3_VALS[lo])
    return np.copysign(out, a)


def quantize_rows(x) -> np.ndarray:
    """GEAR-ZDC's quantized compressed cache (P:1642 DEL: "quantizes each matrix element of the
    compressed data after ZDC compression and dequantizes them before ZDC decompression"), with the
    reading c23 scheme: per cached row (token, KV head) of r values, in FP32 as the GPU computes it,
    scale = max|x| / 448 (1 for an all-zero row), code = E4M3(x / scale), stored value = code * scale.
    x [..., r] -> the dequantized values (fp64 holding FP32 results)."""
    x32 = np.asarray(x, dtype=np.float64).astype(np.float32)
    amax = np.max(np.abs(x32), axis=-1, keepdims=True)
    scale = np.where(amax > 0, amax / np.float32(448.0), np.float32(1.0)).astype(np.float32)
    codes = e4m3((x32 / scale).astype(np.float64))
    return (codes.astype(np.float32) * scale).astype(np.float64)


# --------------------------------------------------------------------------------------
# Eq. 3: row softmax; the denominator is what §5.2 reuses as token importance
# --------------------------------------------------------------------------------------
def softmax_rows(a: np.ndarray, causal: bool = False):
    """P:254-260 (Eq. 3): b_ij = exp(a_ij) / sum_{k<=t_i} exp(a_ik).

    Returns (probs, denominators, log_denominators).  Rows are max-shifted; the
    returned denominator is sum_k exp(a_ik) (un-shifted), its log is m + log sum exp(a-m).
    With causal=True, row i sees columns k <= i (t_i = i).
    A fully masked row is an error.
    """
    a = np.asarray(a, dtype=np.float64)
    n_rows, n_cols = a.shape
    probs = np.zeros_like(a)
    denom = np.zeros(n_rows)
    logd = np.zeros(n_rows)
    for i in range(n_rows):
        t = min(i + 1, n_cols) if causal else n_cols
        if t == 0:
            raise ValueError("softmax_rows: fully masked row %d" % i)
        row = a[i, :t]
        m = np.max(row)
        e = np.exp(row - m)
        ssum = np.sum(e)
        probs[i, :t] = e / ssum
        logd[i] = m + math.log(ssum)
        denom[i] = math.exp(logd[i]) if logd[i] < 700 else math.inf
    return probs, denom, logd


# --------------------------------------------------------------------------------------
# §2.2 SVD and §4.3 / §5.1 offline fold
# --------------------------------------------------------------------------------------
def canonical_signs(R: np.ndarray) -> np.ndarray:
    """Reading c5: for each column, the entry of largest |.| is made positive (ties -> lowest row)."""
    R = R.copy()
    for j in range(R.shape[1]):
        i = int(np.argmax(np.abs(R[:, j])))  # argmax returns the first (lowest row) on ties
        if R[i, j] < 0:
            R[:, j] = -R[:, j]
    return R


def svd_right(A: np.ndarray):
    """P:300 (§2.2): A = U Sigma R^T.  Returns (sigma [n], R [n][n]) with columns of R the
    right singular vectors sorted by non-increasing sigma, canonical signs (reading c5).
    A has at least n rows (checked by the caller, 'insufficient samples')."""
    _, s, vt = np.linalg.svd(A, full_matrices=False)
    order = np.argsort(-s, kind="stable")
    s = s[order]
    R = vt.T[:, order]
    return s, canonical_signs(R)


def kmeans(X: np.ndarray, k: int, iters: int, row_block: int = 4096):
    """P:1157-1167 (§5.1 "Offline rotation matrix computation"): "K-means is a common quantization
    technique that consolidates vectors within each cluster by averaging them into a single vector."
    Lloyd's algorithm as written (reading c21): centroid j starts at row floor(j n / k); each round
    assigns every row to the nearest centroid by squared Euclidean distance (ties -> the lowest
    centroid index) and replaces each centroid by the mean of its rows (an empty cluster keeps its
    centroid); `iters` rounds.  k <= 0 or k >= n: no consolidation (the rows themselves).
    Returns (centroids [k][dim], assignment of the last round [n])."""
    X = np.asarray(X, dtype=np.float64)
    n = X.shape[0]
    if k <= 0 or k >= n:
        return X.copy(), np.arange(n)
    C = X[(np.arange(k) * n) // k].copy()
    assign = np.zeros(n, dtype=np.int64)
    for _ in range(iters):
        for r0 in range(0, n, row_block):   # complete rows per block: identical to the unblocked argmin
            xb = X[r0:r0 + row_block]
            d2 = np.sum((xb[:, None, :] - C[None, :, :]) ** 2, axis=2)
            assign[r0:r0 + row_block] = np.argmin(d2, axis=1)   # first minimum = lowest index
        for j in range(k):
            rows = X[assign == j]
            if rows.shape[0]:
                C[j] = rows.mean(axis=0)
    return C, assign


def fold_layer(dims, wq, wk, wv, wo, xc, k_clusters: int = 0, kmeans_iters: int = 0) -> Dict[str, np.ndarray]:
    """Offline fold of one layer (host, untimed).

    P:989-990 (§4.3): "since Q and K need the same R, we concatenate them into a
    2 Sigma_S x d_h matrix ... For the VW_L pair, we also concatenate them vertically to
    generate a (Sigma_S + d) x d_h matrix."  GQA (reading c4): one R per (layer, KV group);
    the QK stack holds the Q of all G heads of the group and the group's K; the VL stack
    holds the group's V and (W_O^h)^T of all G heads.  W_L^h orientation: reading c1.
    P:1204: W_Q^{R,h} = W_Q^h R^h, W_K^{R,h} = W_K^h R^h.
    P:1218-1219: W_V^h <- W_V^h R_h; [W_L^1, ...] <- [W_L^1 R^1, ...]; in Eq. 4's
    orientation (W_O^h is d_h x d) this is R_vl^T W_O^h (reading c1).
    Returns full-rank folded weights in the input shapes plus R and sigma per group.
    k_clusters > 0: the Q, K and V vectors of the calibration rows are each
    consolidated by kmeans() before stacking ("we conduct the K-means clustering on Q, K, and V,
    respectively"); the W_L^h rows are not ("there is no need to use pruning and K-mean for W_L^h").
    """
    def red(A):
        return kmeans(A, k_clusters, kmeans_iters)[0] if k_clusters > 0 else A

    d, nh, nkv, dh = dims.d_model, dims.n_heads, dims.n_kv_heads, dims.d_head
    G = nh // nkv
    n_rows = min(xc.shape[0], k_clusters) if k_clusters > 0 else xc.shape[0]
    if n_rows * (G + 1) < dh:
        raise ValueError("insufficient samples: n_calib*(G+1) < d_head")
    out = dict(r_qk=np.zeros((nkv, dh, dh)), r_vl=np.zeros((nkv, dh, dh)),
               sigma_qk=np.zeros((nkv, dh)), sigma_vl=np.zeros((nkv, dh)),
               wq_f=np.zeros_like(wq), wk_f=np.zeros_like(wk), wv_f=np.zeros_like(wv),
               wo_f=np.zeros_like(wo))
    for g in range(nkv):
        heads = range(g * G, (g + 1) * G)
        cols_g = slice(g * dh, (g + 1) * dh)
        # QK pair: [Q^h for h in group; K^g] with Q^h = X_c W_Q^h (Eq. 1)
        blocks = [red(xc @ wq[:, h * dh:(h + 1) * dh]) for h in heads] + [red(xc @ wk[:, cols_g])]
        s_qk, R_qk = svd_right(np.vstack(blocks))
        # VW_L pair: [V^g; (W_O^h)^T for h in group]
        blocks = [red(xc @ wv[:, cols_g])] + [wo[h * dh:(h + 1) * dh, :].T for h in heads]
        s_vl, R_vl = svd_right(np.vstack(blocks))
        out["r_qk"][g], out["r_vl"][g] = R_qk, R_vl
        out["sigma_qk"][g], out["sigma_vl"][g] = s_qk, s_vl
        for h in heads:
            out["wq_f"][:, h * dh:(h + 1) * dh] = wq[:, h * dh:(h + 1) * dh] @ R_qk
            out["wo_f"][h * dh:(h + 1) * dh, :] = R_vl.T @ wo[h * dh:(h + 1) * dh, :]
        out["wk_f"][:, cols_g] = wk[:, cols_g] @ R_qk
        out["wv_f"][:, cols_g] = wv[:, cols_g] @ R_vl
    return out


def kept_width(p: float, n: int) -> int:
    """SPEC.md:67-72 (reading c6): keep ceil((1-p) n) columns, never 0.  Integer-exact:
    p is converted through a rational approximation of its decimal value."""
    from fractions import Fraction
    fp = Fraction(str(p))
    k = math.ceil((1 - fp) * n)
    return max(1, int(k))


def truncate_layer(dims, folded: Dict[str, np.ndarray], r_k: int, r_v: int, faithful: bool = False):
    """P:862-864 (Lemma 1, "drop the right p fraction of columns of W_Q^R")
    (same for W_K^R), P:1219-1221 ("discard p x d_h dimensions from each W_L^{R,h} and
    concatenate").  Keeps columns [:r_k] of W_Q^{R,h}, W_K^{R,g}; [:r_v] of W_V^{R,g};
    rows [:r_v] of W_O^{R,h}.  Returns per-head lists.  Faithful mode rounds to BF16."""
    d, nh, nkv, dh = dims.d_model, dims.n_heads, dims.n_kv_heads, dims.d_head
    rnd = bf16 if faithful else (lambda a: a)
    wq = [rnd(folded["wq_f"][:, h * dh:h * dh + r_k]) for h in range(nh)]
    wk = [rnd(folded["wk_f"][:, g * dh:g * dh + r_k]) for g in range(nkv)]
    wv = [rnd(folded["wv_f"][:, g * dh:g * dh + r_v]) for g in range(nkv)]
    wo = [rnd(folded["wo_f"][h * dh:h * dh + r_v, :]) for h in range(nh)]
    return dict(wq=wq, wk=wk, wv=wv, wo=wo)


# --------------------------------------------------------------------------------------
# Eqs. 1-4 of the uncompressed model (used by pin P1; no fold involved)
# --------------------------------------------------------------------------------------
def unfolded_forward(dims, x, wq, wk, wv, wo):
    """P:243-265, Eqs. 1-4 with the causal denominator of Eq. 3: x [B][S][d] -> O_L [B][S][d]."""
    nh, nkv, dh = dims.n_heads, dims.n_kv_heads, dims.d_head
    G = nh // nkv
    B, S, _ = x.shape
    y = np.zeros((B, S, dims.d_model))
    for b in range(B):
        heads_out = []
        for h in range(nh):
            g = h // G
            Q = x[b] @ wq[:, h * dh:(h + 1) * dh]
            K = x[b] @ wk[:, g * dh:(g + 1) * dh]
            V = x[b] @ wv[:, g * dh:(g + 1) * dh]
            P, _, _ = softmax_rows(Q @ K.T / math.sqrt(dh), causal=True)
            heads_out.append(P @ V)
        y[b] = np.hstack(heads_out) @ wo
    return y


# --------------------------------------------------------------------------------------
# §5.2 lightweight token importance and selection
# --------------------------------------------------------------------------------------
def importance(lse: np.ndarray, positions: np.ndarray, mode: int = 0) -> np.ndarray:
    """importance(t_i) = sum_h sum_{k<=t_i} exp(s_k^h), the reused softmax
    denominators.  Computed in the log domain (reading c9): score = log sum_h exp(LSE_h).
    lse: [N_h][T] log-denominators of the token's own row per head.  mode 1 (reading c10)
    subtracts log(t+1) from each LSE first (per-key mean)."""
    lse = np.asarray(lse, dtype=np.float64)
    if mode == 1:
        lse = lse - np.log(np.asarray(positions, dtype=np.float64) + 1.0)[None, :]
    m = np.max(lse, axis=0)
    return m + np.log(np.sum(np.exp(lse - m[None, :]), axis=0))


def important_count(g_bp: int, S: int) -> int:
    """Reading c11: k = ceil(g S) in integer basis points, k = (g_bp S + 9999) div 10000."""
    return (int(g_bp) * int(S) + 9999) // 10000


def select_important(scores: np.ndarray, g_bp: int):
    """"The tokens in layer l are then sorted in descending order, and g^l
    proportion of tokens from the top are classified as important".
    Order key (score desc, index asc) (reading c11); -0.0 == +0.0; NaN is an error.
    Returns (is_important bool[S], tau, k); tau = score of the k-th token, -inf if k=S,
    +inf if k=0 (reading c12)."""
    scores = np.asarray(scores)
    if np.any(np.isnan(scores)):
        raise ValueError("select_important: NaN score")
    S = scores.shape[0]
    k = important_count(g_bp, S)
    order = sorted(range(S), key=lambda t: (-float(scores[t]) + 0.0, t))
    imp = np.zeros(S, dtype=bool)
    imp[order[:k]] = True
    if k == S:
        tau = NEG_INF
    elif k == 0:
        tau = math.inf
    else:
        tau = float(scores[order[k - 1]])
    return imp, tau, k


# --------------------------------------------------------------------------------------
# The hot path: prefill / decode over a compressed KV cache
# --------------------------------------------------------------------------------------
class OracleModel:
    """Layer stack of ZDC attention blocks (attention only: no MLP/norm/residual/RoPE,
    reading c3).  Per layer l: Eq. 1 with folded, truncated weights,
    KV cache of compressed K'/V' (P:78-79, P:813 DEL), Eqs. 2-3 at head dim r with
    scale 1/sqrt(d_h) (reading c2), Eq. 4 with the folded W_O.

    Token split (P:1409-1411, P:1442, P:1455-1456, P:774-776 DEL): at a representative
    layer (group_rep[l] == l, g_bp < 10000) the classes are computed from the softmax
    denominators; unimportant tokens' K'/V' dims >= r^u are zero-filled in the cache
    (reading c13/c14: queries stay at r^i).  Other layers of the group reuse the classes
    and truncate unimportant key rows *before* attention, including the current token's
    own key.  Decode: new token important iff score > tau (reading c12).
    """

    def __init__(self, dims, plan, folded: List[Dict[str, np.ndarray]], faithful: bool = False):
        self.dims, self.plan, self.faithful = dims, plan, faithful
        L = dims.n_layers
        assert len(folded) == L
        self.w = [truncate_layer(dims, folded[l], plan.r_qk_imp[l], plan.r_vl_imp[l], faithful)
                  for l in range(L)]
        self.reset()

    # cache state ---------------------------------------------------------------------
    def reset(self):
        L = self.dims.n_layers
        self.K: List[Optional[np.ndarray]] = [None] * L   # [B][Nkv][len][r_k]
        self.V: List[Optional[np.ndarray]] = [None] * L
        self.length = [0] * L
        self.classes: Dict[int, np.ndarray] = {}          # rep layer -> bool [B][len]
        self.tau: Dict[int, np.ndarray] = {}              # rep layer -> [B]
        self.scores: Dict[int, np.ndarray] = {}           # rep layer -> [B][len] importance
        self.lse: List[Optional[np.ndarray]] = [None] * L  # last call's [B][Nh][T]
        self.alive: List[Optional[np.ndarray]] = [None] * L  # eviction (H2O-ZDC): kept cache rows [B][len]

    def _rnd(self, a):
        return bf16(a) if self.faithful else a

    def _store(self, a):
        """What the cache keeps of K'/V' rows: FP8 codes x per-row scale when plan.kv_fp8 (NEXT-4)."""
        return quantize_rows(a) if getattr(self.plan, "kv_fp8", 0) else a

    def _split(self, l):
        return self.plan.g_bp[l] < 10000

    def _evict(self, l):
        """H2O-ZDC (P:1642 DEL: "first compresses Q, K, and V using SVD and then evicts unimportant
        tokens"), reading c26: a split group with r^u = 0 evicts its unimportant tokens from the
        cache instead of truncating them: every query still attends (at r^i) to the prompt it is
        computed with and to itself, but no later query sees an evicted row."""
        return self._split(l) and self.plan.r_qk_unimp[l] == 0 and self.plan.r_vl_unimp[l] == 0

    def _truncate_rows(self, l, K, V, unimp):
        """Zero-fill (P:774-776 DEL): dims >= r^u of unimportant rows read back as 0.
        K, V [B][Nkv][T][r]; unimp bool [B][T]."""
        ru_k, ru_v = self.plan.r_qk_unimp[l], self.plan.r_vl_unimp[l]
        K = K.copy()
        V = V.copy()
        for b in range(K.shape[0]):
            rows = np.nonzero(unimp[b])[0]
            K[b][:, rows, ru_k:] = 0.0
            V[b][:, rows, ru_v:] = 0.0
        return K, V

    def _project(self, l, x):
        """Eq. 1 with W^R truncated: x [B][T][d] -> Q [B][Nh][T][r_k], K, V [B][Nkv][T][r]."""
        w = self.w[l]
        Q = np.stack([np.stack([x[b] @ w["wq"][h] for h in range(self.dims.n_heads)]) for b in range(x.shape[0])])
        K = np.stack([np.stack([x[b] @ w["wk"][g] for g in range(self.dims.n_kv_heads)]) for b in range(x.shape[0])])
        V = np.stack([np.stack([x[b] @ w["wv"][g] for g in range(self.dims.n_kv_heads)]) for b in range(x.shape[0])])
        return self._rnd(Q), self._rnd(K), self._rnd(V)

    def _attend(self, q, Kc, Vc, q_pos, row_block=512, alive=None):
        """Eqs. 2-3 for the rows of one (b, h): s_tj = q_t.k_j / sqrt(d_h), j <= q_pos[t]
        (and alive[j] when rows were evicted, reading c26).
        Complete rows per query-row block (no online-softmax tiling).  Returns O [T][r_v], LSE [T]."""
        dh = self.dims.d_head
        T = q.shape[0]
        O = np.zeros((T, Vc.shape[1]))
        lse = np.zeros(T)
        q_pos = np.asarray(q_pos)
        for r0 in range(0, T, row_block):
            r1 = min(T, r0 + row_block)
            n_keys = int(np.max(q_pos[r0:r1])) + 1
            s = q[r0:r1] @ Kc[:n_keys].T / math.sqrt(dh)
            visible = np.arange(n_keys)[None, :] <= q_pos[r0:r1, None]   # j <= t_i (Eq. 3)
            if alive is not None:
                visible = visible & np.asarray(alive[:n_keys], dtype=bool)[None, :]
            s = np.where(visible, s, -np.inf)
            m = np.max(s, axis=1, keepdims=True)
            e = np.exp(s - m)                           # masked keys -> exactly 0
            l_sum = np.sum(e, axis=1, keepdims=True)    # row sum from the unrounded P
            p = self._rnd(e)                            # faithful: P rounded before PV
            O[r0:r1] = (p @ Vc[:n_keys]) / l_sum
            lse[r0:r1] = m[:, 0] + np.log(l_sum[:, 0])
        return self._rnd(O), lse

    def _output(self, l, O):
        """Eq. 4 with the folded W_O: y = sum_h O'^h W_O^{R,h}[:r_v]."""
        w = self.w[l]
        y = np.zeros((O.shape[0], O.shape[2], self.dims.d_model))
        for b in range(O.shape[0]):
            for h in range(self.dims.n_heads):
                y[b] += O[b, h] @ w["wo"][h]
        return self._rnd(y)

    # prefill -------------------------------------------------------------------------
    def prefill_layer(self, l, x):
        """One layer of prompt processing on an empty cache: x [B][S][d] -> y [B][S][d]."""
        if self.length[l] != 0:
            raise ValueError("prefill requires an empty cache")
        dims, plan = self.dims, self.plan
        G = dims.group
        B, S, _ = x.shape
        Q, K, V = self._project(l, x)
        rep = plan.group_rep[l]
        split = self._split(l)
        if split and rep != l:
            if rep not in self.classes or self.classes[rep].shape[1] < S:
                raise ValueError("layer %d: representative layer %d has not classified these tokens" % (l, rep))
            if not self._evict(l):   # eviction: the prompt attends in full; the cache drops rows below
                K, V = self._truncate_rows(l, K, V, ~self.classes[rep][:, :S])
        pos = np.arange(S)
        O = np.zeros((B, dims.n_heads, S, V.shape[3]))
        lse = np.zeros((B, dims.n_heads, S))
        for b in range(B):
            for h in range(dims.n_heads):
                O[b, h], lse[b, h] = self._attend(Q[b, h], K[b, h // G], V[b, h // G], pos)
        self.lse[l] = lse
        if split and rep == l:
            cls = np.zeros((B, S), dtype=bool)
            tau = np.zeros(B)
            sc = np.zeros((B, S))
            for b in range(B):
                sc[b] = importance(lse[b], pos, plan.importance_mode)
                cls[b], tau[b], _ = select_important(sc[b], plan.g_bp[l])
            self.classes[l], self.tau[l], self.scores[l] = cls, tau, sc
            if not self._evict(l):
                K, V = self._truncate_rows(l, K, V, ~cls)
        if self._evict(l):   # the cache keeps the important rows only (evicted rows read back as 0)
            keep = self.classes[rep][:, :S].copy()
            K = K * keep[:, None, :, None]
            V = V * keep[:, None, :, None]
            self.alive[l] = keep
        self.K[l], self.V[l] = self._store(K), self._store(V)   # the prompt attended at full precision
        self.length[l] = S
        return self._output(l, O)

    def prefill(self, x, l0=0, l1=None):
        """Layers [l0, l1) chained: y of layer l feeds x of layer l+1."""
        l1 = self.dims.n_layers if l1 is None else l1
        for l in range(l0, l1):
            x = self.prefill_layer(l, x)
        return x

    def prefill_rows(self, l, x, rows):
        """Sampled-output check at full size: y rows `rows` of a prefill of layer l on an
        empty cache, no split (the whole K'/V' is projected; only the listed query rows attend).
        Does not modify the cache."""
        dims = self.dims
        G = dims.group
        w = self.w[l]
        B, S, _ = x.shape
        rows = np.asarray(rows)
        y = np.zeros((B, len(rows), dims.d_model))
        for b in range(B):
            K = [self._rnd(x[b] @ w["wk"][g]) for g in range(dims.n_kv_heads)]
            V = [self._rnd(x[b] @ w["wv"][g]) for g in range(dims.n_kv_heads)]
            for h in range(dims.n_heads):
                q = self._rnd(x[b, rows] @ w["wq"][h])
                O, _ = self._attend(q, K[h // G], V[h // G], rows)
                y[b] += O @ w["wo"][h]
        return self._rnd(y)

    # decode --------------------------------------------------------------------------
    def decode_layer(self, l, x):
        """One token per sequence at position len[l]: x [B][d] -> y [B][d].
        The new token's K'/V' are appended before it attends (it attends to itself)."""
        dims, plan = self.dims, self.plan
        G = dims.group
        B = x.shape[0]
        t = self.length[l]
        if self.K[l] is None:
            raise ValueError("decode requires a prefilled cache")
        Q, K, V = self._project(l, x[:, None, :])
        rep = plan.group_rep[l]
        split = self._split(l)
        evict = self._evict(l)
        if split and rep != l:
            if self.classes[rep].shape[1] <= t:
                raise ValueError("layer %d: representative %d has not classified position %d" % (l, rep, t))
            if not evict:
                K, V = self._truncate_rows(l, K, V, ~self.classes[rep][:, t:t + 1])
        self.K[l] = np.concatenate([self.K[l], self._store(K)], axis=2)   # quantized on append (NEXT-4)
        self.V[l] = np.concatenate([self.V[l], self._store(V)], axis=2)
        self.length[l] = t + 1
        if evict:   # the new token attends to the kept rows and to itself, then may be evicted
            self.alive[l] = np.concatenate([self.alive[l], np.ones((B, 1), dtype=bool)], axis=1)
        O = np.zeros((B, dims.n_heads, 1, V.shape[3]))
        lse = np.zeros((B, dims.n_heads, 1))
        for b in range(B):
            for h in range(dims.n_heads):
                O[b, h], lse[b, h] = self._attend(Q[b, h], self.K[l][b, h // G], self.V[l][b, h // G],
                                                  np.array([t]), alive=self.alive[l][b] if evict else None)
        self.lse[l] = lse
        if split and rep == l:
            new_cls = np.zeros((B, 1), dtype=bool)
            new_sc = np.zeros((B, 1))
            for b in range(B):
                new_sc[b, 0] = importance(lse[b], np.array([t]), plan.importance_mode)[0]
                new_cls[b, 0] = new_sc[b, 0] > self.tau[l][b]
            self.classes[l] = np.concatenate([self.classes[l], new_cls], axis=1)
            self.scores[l] = np.concatenate([self.scores[l], new_sc], axis=1)
            if not evict:
                Kt, Vt = self._truncate_rows(l, self.K[l][:, :, t:t + 1], self.V[l][:, :, t:t + 1], ~new_cls)
                self.K[l][:, :, t:t + 1] = Kt
                self.V[l][:, :, t:t + 1] = Vt
        if evict:   # representative: its own decision above; other layers: the representative's class
            keep = self.classes[rep][:, t]
            self.alive[l][:, t] = keep
            self.K[l][:, :, t] *= keep[:, None, None]
            self.V[l][:, :, t] *= keep[:, None, None]
        return self._output(l, O)[:, 0, :]

    def decode(self, x, l0=0, l1=None):
        l1 = self.dims.n_layers if l1 is None else l1
        for l in range(l0, l1):
            x = self.decode_layer(l, x)
        return x


# --------------------------------------------------------------------------------------
# Byte counts (pin P12)
# --------------------------------------------------------------------------------------
def cache_floats(dims, plan, classes_per_layer: List[np.ndarray]) -> int:
    """SPEC.md:287 / :583: cache floats = sum over tokens, layers, KV heads of (w_k + w_v),
    with w = r^i for important tokens and r^u for unimportant tokens."""
    total = 0
    for l in range(dims.n_layers):
        imp = classes_per_layer[l]
        n_imp = int(np.sum(imp))
        n_un = int(imp.size - n_imp)
        total += dims.n_kv_heads * (n_imp * (plan.r_qk_imp[l] + plan.r_vl_imp[l])
                                    + n_un * (plan.r_qk_unimp[l] + plan.r_vl_unimp[l]))
    return total


def sp_bytes_received(P: int, B: int, S: int, n_kv: int, r_k: int, r_v: int, elem_bytes: int = 2) -> int:
    """Bytes one of P ranks receives in an all-gather of compressed K'/V' for one layer:
    (P-1)/P * B * S * N_kv * (r_k + r_v) * elem_bytes."""
    assert S % P == 0
    return (P - 1) * (S // P) * B * n_kv * (r_k + r_v) * elem_bytes


def sp_bytes_received_ulysses(P: int, B: int, S: int, n_h: int, n_kv: int, r_k: int, r_v: int,
                              elem_bytes: int = 2) -> int:
    """Bytes one of P ranks receives per layer in the paper's Ulysses SP (Fig.
    bkg:fig:all2all): all-to-all #1 delivers, from each of the P-1 peers, its S/P tokens' compressed
    Q'/K'/V' columns of this rank's N_h/P heads and N_kv/P KV groups; all-to-all #2 delivers, from
    each peer, that peer's heads' O' (r_v columns per head) for this rank's S/P tokens:
    (P-1) * (B S / P) * [(N_h r_k + N_kv (r_k + r_v)) / P + N_h r_v / P] * elem_bytes."""
    assert S % P == 0 and n_kv % P == 0 and n_h % P == 0
    rows = B * (S // P)
    cols1 = (n_h * r_k + n_kv * (r_k + r_v)) // P
    cols2 = n_h * r_v // P
    return (P - 1) * rows * (cols1 + cols2) * elem_bytes


def layer_groups(classes: np.ndarray, threshold_bp: int = 9500) -> List[int]:
    """"we offline identify layers that have the same important and unimportant token
    sets (i.e., repetition ratio > 95%)"; the classification of a group's first layer is then
    reused by the others.  Reading c22: consecutive layers; layer l joins the current
    group when the fraction of (sequence, token) positions whose class equals the group
    representative's exceeds threshold_bp / 10000 (strict, integer arithmetic), else it starts a
    new group.  classes: bool [L][B][S] (every layer classified as its own representative).
    Returns group_rep [L]."""
    classes = np.asarray(classes, dtype=bool)
    L = classes.shape[0]
    total = int(classes[0].size)
    rep = [0] * L
    cur = 0
    for l in range(1, L):
        same = int(np.sum(classes[l] == classes[cur]))
        if same * 10000 > threshold_bp * total:
            rep[l] = cur
        else:
            cur = l
            rep[l] = l
    return rep

