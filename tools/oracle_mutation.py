"""Mutation check of the oracle's pins (tests/test_oracle_pins.py): each
mutation below is a plausible mistake in oracle/grass_oracle.py (a dropped
term, a wrong sign or index, a swapped operand, an off-by-one); the pin suite
must FAIL for every one of them.  Runs on CPU in a scratch copy of the repo.

    python tools/oracle_mutation.py            # prints one line per mutation, exits 1 if one survives
"""
import os
import shutil
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

# (name, original text, mutated text) — each original must occur exactly once
MUTATIONS = [
    ("norm: fp32 accumulation", "g64 = g.astype(np.float64, copy=False).ravel()",
     "g64 = g.astype(np.float32, copy=False).ravel()"),
    ("norm: chunk parts summed twice", "parts.append(float(np.dot(c, c)))", "parts.append(2 * float(np.dot(c, c)))"),
    ("rms: missing sqrt", "return math.sqrt(ss / n_p)", "return ss / n_p"),
    ("rms: divides by N_p + 1", "return math.sqrt(ss / n_p)", "return math.sqrt(ss / (n_p + 1))"),
    ("dp average: sum not mean", "return acc / len(grads_per_rank)", "return acc"),
    ("window: divides by count + 1",
     "return [self.S[l] / self.c[l] if self.c[l] > 0 else None for l in range(self.n)]",
     "return [self.S[l] / (self.c[l] + 1) if self.c[l] > 0 else None for l in range(self.n)]"),
    ("EMA: alpha on the old value", "self.m[l] = alpha * w[l] + (1.0 - alpha) * self.m[l]",
     "self.m[l] = (1.0 - alpha) * w[l] + alpha * self.m[l]"),
    ("EMA: frozen layers reset", "                if w[l] is not None:\n                    self.m[l] = alpha",
     "                if True:\n                    self.m[l] = 0.0 if w[l] is None else alpha"),
    ("first commit with EMA", "            self.m = [w[l] if w[l] is not None else 0.0 for l in range(self.n)]",
     "            self.m = [alpha * w[l] if w[l] is not None else 0.0 for l in range(self.n)]"),
    ("window not reset", "        self.S = [0.0] * self.n\n        self.c = [0] * self.n\n", ""),
    ("T_p = 0: empty commits allowed after the first (R22)",
     "if sum(self.c) == 0 and not (empty_first_ok and not self.committed):",
     "if sum(self.c) == 0 and not empty_first_ok:"),
    ("T_p = 0: first empty commit rejected (R22)", "m = self.mgn.commit(self.alpha, empty_first_ok=self.T_p == 0)",
     "m = self.mgn.commit(self.alpha)"),
    ("softmax: tau multiplies", "e = [math.exp((x - mx) / tau) for x in mt]", "e = [math.exp((x - mx) * tau) for x in mt]"),
    ("softmax: sign flipped", "e = [math.exp((x - mx) / tau) for x in mt]", "e = [math.exp((mx - x) / tau) for x in mt]"),
    ("softmax: no max-normalisation", "mt = [x / M for x in m] if M > 0.0 else [0.0] * len(m)", "mt = m"),
    ("splitmix64: wrong shift", "z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64",
     "z = ((z ^ (z >> 31)) * 0xBF58476D1CE4E5B9) & MASK64"),
    ("uniform: 52-bit mantissa", "return (splitmix64(key ^ ctr) >> 11) * (2.0 ** -53)",
     "return (splitmix64(key ^ ctr) >> 12) * (2.0 ** -52)"),
    ("uniform: period/draw swapped", "ctr = ((period << 16) + k) & MASK64", "ctr = ((k << 16) + period) & MASK64"),
    ("sampler: <= instead of <", "            if x < c:", "            if x <= c:"),
    ("sampler: R not renormalised", "        for l in avail:\n            R += p[l]", "        for l in range(n):\n            R += p[l]"),
    ("sampler: fallback first", "        pick = avail[-1]", "        pick = avail[0]"),
    ("adamw: no weight decay", "th1 = th * (1.0 - lr * weight_decay)", "th1 = th"),
    ("adamw: decay applied after the step", "th2 = th1 - (lr / bc1) * m1 / denom",
     "th2 = (th - (lr / bc1) * m1 / denom) * (1.0 - lr * weight_decay)"),
    ("adamw: bias correction t-1", "bc1 = 1.0 - beta1 ** t", "bc1 = 1.0 - beta1 ** max(t - 1, 1)"),
    ("adamw: no bc2", "denom = np.sqrt(v1) / math.sqrt(bc2) + eps", "denom = np.sqrt(v1) + eps"),
    ("adamw: eps inside sqrt", "denom = np.sqrt(v1) / math.sqrt(bc2) + eps", "denom = np.sqrt(v1 / bc2 + eps)"),
    ("adamw: betas swapped in m", "m1 = beta1 * m0 + (1.0 - beta1) * gg", "m1 = beta2 * m0 + (1.0 - beta2) * gg"),
    ("adamw: v uses |g|", "v1 = beta2 * v0 + (1.0 - beta2) * gg * gg", "v1 = beta2 * v0 + (1.0 - beta2) * np.abs(gg)"),
    ("bf16: truncation not RNE", "r = (u + np.uint64(0x7FFF) + ((u >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)",
     "r = u >> np.uint64(16)"),
    ("clip: no epsilon and no cap", "return min(1.0, max_norm / (total + 1e-6))", "return max_norm / total"),
    ("schedule: resample at T_u", "    if d % T_s == 0:\n        return \"resample\"", "    if d % T_u == 0:\n        return \"resample\""),
    ("schedule: probe includes T_p", "    if step < T_p:", "    if step <= T_p:"),
    ("clip: MGN records the clipped norm", "        self.accumulate(layer_ids, grads)\n        return params",
     "        self.accumulate(layer_ids, eff)\n        return params"),
    ("clip: coefficient from the first layer only",
     "coef = clip_coefficient([sq_norm(g) for g in grads], max_grad_norm)",
     "coef = clip_coefficient([sq_norm(grads[0])], max_grad_norm)"),
    ("bf16: master not initialised from the bf16 parameter",
     "    if theta_bits is not None:\n        master = bf16_to_f32(theta_bits)", "    if False:\n        pass"),
    ("bf16: widening drops the low mantissa bits",
     "    b = np.asarray(bits, dtype=np.uint16).astype(np.uint32) << np.uint32(16)",
     "    b = (np.asarray(bits, dtype=np.uint16).astype(np.uint32) & np.uint32(0xFFF0)) << np.uint32(16)"),
    ("always groups recorded in the MGN window", "            if l < self.n_s:                  # always-active groups are not sampled (R19)\n                self.mgn.record(",
     "            if l < self.n:\n                self.mgn.record("),
    ("always groups sampled", "        return sample_layers(list(p)[:self.n_s], self.gamma, self.seed, period)",
     "        return sample_layers(list(p), self.gamma, self.seed, period)"),
]


def main() -> int:
    src = open(os.path.join(ROOT, "oracle", "grass_oracle.py")).read()
    survivors = []
    with tempfile.TemporaryDirectory() as tmp:
        for d in ("oracle", "tests", "synth"):
            shutil.copytree(os.path.join(ROOT, d), os.path.join(tmp, d),
                            ignore=shutil.ignore_patterns("__pycache__"))
        target = os.path.join(tmp, "oracle", "grass_oracle.py")
        for name, a, b in MUTATIONS:
            if src.count(a) != 1:
                print(f"SKIP  {name}: original text not found exactly once")
                survivors.append(name)
                continue
            open(target, "w").write(src.replace(a, b))
            r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider",
                                os.path.join(tmp, "tests", "test_oracle_pins.py")],
                               cwd=tmp, capture_output=True, text=True, timeout=900)
            killed = r.returncode != 0
            print(f"{'killed ' if killed else 'SURVIVED'} {name}", flush=True)
            if not killed:
                survivors.append(name)
        open(target, "w").write(src)
    print(f"{len(MUTATIONS) - len(survivors)}/{len(MUTATIONS)} mutations killed by the pins")
    return 1 if survivors else 0


if __name__ == "__main__":
    sys.exit(main())
