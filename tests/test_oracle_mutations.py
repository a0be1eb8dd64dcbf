"""Mutation check of the oracle's pins: each plausible mistake below, applied to a
copy of oracle/zdc_oracle.py, must make at least one pin in tests/test_oracle_pins.py fail.
A surviving mutant means part of the oracle is unpinned.  CPU only (~1 min)."""
import inspect
import os
import types

import pytest

import test_oracle_pins as pins

SRC_PATH = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "zdc_oracle.py")

# (name, exact source text, replacement); each text occurs exactly once in zdc_oracle.py
MUTANTS = [
    ("bf16 round half up", "bits = (bits + 0x7FFF + lsb) & 0xFFFF0000", "bits = (bits + 0x8000) & 0xFFFF0000"),
    ("bf16 truncation", "bits = (bits + 0x7FFF + lsb) & 0xFFFF0000", "bits = bits & 0xFFFF0000"),
    ("P not rounded before PV", "p = self._rnd(e)                            # faithful",
     "p = e                            # faithful"),
    ("l from the rounded P", "l_sum = np.sum(e, axis=1, keepdims=True)", "l_sum = np.sum(self._rnd(e), axis=1, keepdims=True)"),
    ("O' not rounded", "return self._rnd(O), lse", "return O, lse"),
    ("y not rounded", "return self._rnd(y)\n\n    # prefill", "return y\n\n    # prefill"),
    ("Q' not rounded", "return self._rnd(Q), self._rnd(K), self._rnd(V)", "return Q, self._rnd(K), self._rnd(V)"),
    ("K' not rounded", "return self._rnd(Q), self._rnd(K), self._rnd(V)", "return self._rnd(Q), K, self._rnd(V)"),
    ("V' not rounded", "return self._rnd(Q), self._rnd(K), self._rnd(V)", "return self._rnd(Q), self._rnd(K), V"),
    ("weights not rounded", "rnd = bf16 if faithful else (lambda a: a)", "rnd = (lambda a: a)"),
    ("decode class >= tau", "new_cls[b, 0] = new_sc[b, 0] > self.tau[l][b]", "new_cls[b, 0] = new_sc[b, 0] >= self.tau[l][b]"),
    ("scale 1/sqrt(r)", "s = q[r0:r1] @ Kc[:n_keys].T / math.sqrt(dh)", "s = q[r0:r1] @ Kc[:n_keys].T / math.sqrt(Kc.shape[1])"),
    ("causal mask off by one", "visible = np.arange(n_keys)[None, :] <= q_pos[r0:r1, None]",
     "visible = np.arange(n_keys)[None, :] <= q_pos[r0:r1, None] + 1"),
    ("W_O fold without transpose", "R_vl.T @ wo[h * dh:(h + 1) * dh, :]", "R_vl @ wo[h * dh:(h + 1) * dh, :]"),
    ("W_K folded with R_vl", "out[\"wk_f\"][:, cols_g] = wk[:, cols_g] @ R_qk", "out[\"wk_f\"][:, cols_g] = wk[:, cols_g] @ R_vl"),
    ("truncation keeps the wrong columns", "wq = [rnd(folded[\"wq_f\"][:, h * dh:h * dh + r_k])",
     "wq = [rnd(folded[\"wq_f\"][:, h * dh + 1:h * dh + r_k + 1])"),
    ("W_O keeps the bottom rows", "wo = [rnd(folded[\"wo_f\"][h * dh:h * dh + r_v, :])",
     "wo = [rnd(folded[\"wo_f\"][(h + 1) * dh - r_v:(h + 1) * dh, :])"),
    ("canonical sign flipped", "if R[i, j] < 0:", "if R[i, j] > 0:"),
    ("mean-mode offset log(t+2)", "np.log(np.asarray(positions, dtype=np.float64) + 1.0)",
     "np.log(np.asarray(positions, dtype=np.float64) + 2.0)"),
    ("importance drops the max shift", "return m + np.log(np.sum(np.exp(lse - m[None, :]), axis=0))",
     "return np.log(np.sum(np.exp(lse - m[None, :]), axis=0))"),
    ("count rounds down", "(int(g_bp) * int(S) + 9999) // 10000", "(int(g_bp) * int(S)) // 10000"),
    ("ties to the newer token", "key=lambda t: (-float(scores[t]) + 0.0, t)", "key=lambda t: (-float(scores[t]) + 0.0, -t)"),
    ("tau is the (k+1)-th score", "tau = float(scores[order[k - 1]])", "tau = float(scores[order[min(k, S - 1)]])"),
    ("unimportant keeps one dim too many", "K[b][:, rows, ru_k:] = 0.0", "K[b][:, rows, ru_k + 1:] = 0.0"),
    ("non-representative layer truncates important rows",
     "K, V = self._truncate_rows(l, K, V, ~self.classes[rep][:, :S])",
     "K, V = self._truncate_rows(l, K, V, self.classes[rep][:, :S])"),
    ("decode attends before appending", "self.length[l] = t + 1\n        if evict:",
     "self.length[l] = t + 1\n        self.K[l], self.V[l] = self.K[l][:, :, :-1], self.V[l][:, :, :-1]\n        if evict:"),
    ("Ulysses bytes without all-to-all #2", "return (P - 1) * rows * (cols1 + cols2) * elem_bytes",
     "return (P - 1) * rows * cols1 * elem_bytes"),
    ("k-means ties to the highest index", "assign[r0:r0 + row_block] = np.argmin(d2, axis=1)",
     "assign[r0:r0 + row_block] = d2.shape[1] - 1 - np.argmin(d2[:, ::-1], axis=1)"),
    ("k-means init from the first k rows", "C = X[(np.arange(k) * n) // k].copy()", "C = X[:k].copy()"),
    ("k-means empty cluster reset to 0", "            if rows.shape[0]:\n                C[j] = rows.mean(axis=0)",
     "            C[j] = rows.mean(axis=0) if rows.shape[0] else 0.0"),
    ("layer groups compare to the previous layer", "same = int(np.sum(classes[l] == classes[cur]))",
     "same = int(np.sum(classes[l] == classes[l - 1]))"),
    ("layer groups >= threshold", "if same * 10000 > threshold_bp * total:", "if same * 10000 >= threshold_bp * total:"),
    ("e4m3 ties away from zero", "pick_hi = (dhi < dlo) | ((dhi == dlo) & (_E4M3_CODES[hi] % 2 == 0))",
     "pick_hi = (dhi <= dlo)"),
    ("e4m3 subnormals at 2^-7", "v = (m / 8.0) * 2.0 ** -6 if e == 0", "v = (m / 8.0) * 2.0 ** -7 if e == 0"),
    ("fp8 scale over 240", "scale = np.where(amax > 0, amax / np.float32(448.0), np.float32(1.0)).astype(np.float32)",
     "scale = np.where(amax > 0, amax / np.float32(240.0), np.float32(1.0)).astype(np.float32)"),
    ("fp8 cache not quantized on append", "self.K[l] = np.concatenate([self.K[l], self._store(K)], axis=2)",
     "self.K[l] = np.concatenate([self.K[l], K], axis=2)"),
    ("eviction keeps evicted rows visible", "                visible = visible & np.asarray(alive[:n_keys], dtype=bool)[None, :]",
     "                visible = visible"),
    ("eviction truncates before the prompt attention", "            if not self._evict(l):   # eviction: the prompt attends in full; the cache drops rows below",
     "            if True:"),
    ("decode token does not attend itself under eviction", "            self.alive[l] = np.concatenate([self.alive[l], np.ones((B, 1), dtype=bool)], axis=1)",
     "            self.alive[l] = np.concatenate([self.alive[l], np.zeros((B, 1), dtype=bool)], axis=1)"),
    ("SP bytes without (P-1)", "return (P - 1) * (S // P) * B * n_kv * (r_k + r_v) * elem_bytes",
     "return P * (S // P) * B * n_kv * (r_k + r_v) * elem_bytes"),
]


def _pin_calls():
    calls = []
    for name, fn in inspect.getmembers(pins, inspect.isfunction):
        if not name.startswith("test_"):
            continue
        params = [m for m in getattr(fn, "pytestmark", []) if m.name == "parametrize"]
        if not params:
            calls.append((name, fn, {}))
            continue
        argnames = [a.strip() for a in params[0].args[0].split(",")]
        for vals in params[0].args[1]:
            vals = vals if len(argnames) > 1 else (vals,)
            calls.append((name, fn, dict(zip(argnames, vals))))
    return calls


def _mutant(old, new):
    src = open(SRC_PATH).read()
    assert src.count(old) == 1, "mutation anchor not unique / missing: %r" % old
    mod = types.ModuleType("zdc_oracle_mutant")
    exec(compile(src.replace(old, new), SRC_PATH + "<mutant>", "exec"), mod.__dict__)
    return mod


def test_unmutated_oracle_passes_every_pin(monkeypatch):
    monkeypatch.setattr(pins, "O", _mutant("NEG_INF = -math.inf", "NEG_INF = -math.inf"))
    for name, fn, kw in _pin_calls():
        fn(**kw)


@pytest.mark.parametrize("name,old,new", MUTANTS, ids=[m[0] for m in MUTANTS])
def test_mutant_is_killed(monkeypatch, name, old, new):
    monkeypatch.setattr(pins, "O", _mutant(old, new))
    for pin, fn, kw in _pin_calls():
        try:
            fn(**kw)
        except Exception:            # AssertionError or a crash both kill the mutant
            return
    pytest.fail("mutant survived every pin: %s" % name)
