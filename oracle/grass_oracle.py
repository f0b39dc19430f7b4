"""GRASS hot-path ORACLE — plain, slow, obviously-correct CPU reference (fp64).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
module.  The product path (``paper_2604_07808_b200``) never imports it, and this
module never imports the product: the two share no code.

It follows the paper (arxiv 2604.07808, ``PAPER.md`` = /root/reference/PAPER.md)
step by step, in the paper's order and notation:

  * Eq. 2 (§3.1) — per-step RMS gradient norm
        r_{l,t} = sqrt(||g_t^(l)||_2^2 / N_p^(l))
    and its window mean  m_l(T) = (1/T) sum_t r_{l,t}.
  * Probing phase (§3.2) — T_p steps, no parameter update,
    yields the initial estimate m_l(T_p).
  * Eq. 3 — p^(l) = exp(m_l/tau) / sum_i exp(m_i/tau).
  * Sampling — "samples gamma layers out of N_L".
  * Eq. 4 — m_l(T) = alpha m_l(T_u) + (1-alpha) m_l(T-T_u);
    "Frozen layers retain their previous MGN values".
  * Optimizer update of trainable layers (the paper never
    names the optimizer) — AdamW with torch.optim.AdamW semantics (DESIGN.md
    reading R1).
  * Layer-wise offload — numerically a no-op; the oracle has
    none.

Every place where the paper is silent takes the reading listed in DESIGN.md
("Readings of the paper"); each function names the reading(s) it uses.

Parity pins for every function live in ``tests/test_oracle_pins.py`` and the
fixtures in ``tests/golden/``.  Parity status per function:
  sq_norm / rms_norm ............ pinned (exact rational sums, closed forms)
  MgnState (window, commit, EMA)  pinned (SPEC examples, brute force, invariants)
  softmax_probs ................. pinned (closed forms, limits, invariants)
  splitmix64 / uniform .......... pinned (published SplitMix64 output vectors)
  sample_layers ................. pinned (exact law enumeration, torch.multinomial)
  adamw_step .................... pinned (closed forms, torch.optim.AdamW fp64)
  schedule_decision ............. pinned (paper values T_p=150, T_s=25)
  clip_coefficient (R17) ........ pinned (torch.nn.utils.clip_grad_norm_)
  bf16_to_f32 / f32_to_bf16 ..... pinned (torch bfloat16 conversions, RNE)
  adamw_step_bf16 (R18) ......... pinned (torch.optim.AdamW on an fp32 master)
  GrassOracle n_always (R19) .... pinned (torch.optim.AdamW over every tensor at
                                  gamma = N_L; MGN / p / sampler equal a run without
                                  the groups)
  Paper-level choices of tau, alpha, the RNG and the draw scheme: **parity
  unpinned** against the paper itself (the paper gives no values); they are
  pinned only against our stated readings (R3, R5, R6, R7).
"""
from __future__ import annotations

import math
from fractions import Fraction

import numpy as np

MASK64 = (1 << 64) - 1
GOLDEN_GAMMA = 0x9E3779B97F4A7C15

# ---------------------------------------------------------------------------
# Eq. 2 — per-layer squared norm and RMS
# ---------------------------------------------------------------------------

_FSUM_LIMIT = 1 << 16     # below this many elements: math.fsum (correctly rounded)
_CHUNK = 1 << 22          # above: fsum over fp64 chunk sums


def sq_norm(g) -> float:
    """||g||_2^2 in fp64 (Eq. 2 numerator).

    Each fp32 element is widened to fp64 and squared; the square of a 24-bit
    mantissa fits in fp64's 53 bits, so every square is exact and only the sum
    rounds.  Small inputs: ``math.fsum`` (correctly rounded).  Large inputs:
    fp64 ``np.sum`` per chunk, then ``math.fsum`` over chunk sums.
    """
    g = np.asarray(g)
    if g.size == 0:
        return 0.0
    g64 = g.astype(np.float64, copy=False).ravel()
    if g64.size <= _FSUM_LIMIT:
        return math.fsum((g64 * g64).tolist())
    parts = []
    for s in range(0, g64.size, _CHUNK):
        c = g64[s:s + _CHUNK]
        parts.append(float(np.dot(c, c)))
    return math.fsum(parts)


def rms_norm(ss: float, n_p: int) -> float:
    """r_l = sqrt(||g||^2 / N_p)  (Eq. 2 inner term).

    N_p is the TRUE parameter count of the layer (no padding) — reading R10.
    """
    if n_p <= 0:
        raise ValueError("N_p must be positive")
    return math.sqrt(ss / n_p)


def dp_average(grads_per_rank):
    """Data-parallel averaged gradient (sum over ranks)/W in fp64 (reading R9)."""
    acc = np.zeros(np.asarray(grads_per_rank[0]).shape, dtype=np.float64)
    for g in grads_per_rank:
        acc += np.asarray(g, dtype=np.float64)
    return acc / len(grads_per_rank)


# ---------------------------------------------------------------------------
# Eq. 2 window mean + Eq. 4 EMA
# ---------------------------------------------------------------------------

class MgnState:
    """Window accumulators S_l, c_l and committed MGN m_l.

    record(l, r):  S_l += r; c_l += 1            (Eq. 2 sum over t)
    commit(alpha): w_l = S_l / c_l for c_l > 0   (Eq. 2 mean, reading R4)
        first commit  -> m_l = w_l               (reading R8)
        later commits -> m_l = alpha w_l + (1-alpha) m_l   if c_l > 0   (Eq. 4)
                         m_l unchanged                      if c_l = 0
                         ("Frozen layers retain their previous MGN values",
                          PAPER.md:127; "previous" = prior EMA, reading R5)
        then S, c reset.
    """

    def __init__(self, n_layers: int):
        self.n = n_layers
        self.S = [0.0] * n_layers
        self.c = [0] * n_layers
        self.m = [0.0] * n_layers
        self.committed = False

    def record(self, layer: int, r: float) -> None:
        if not math.isfinite(r):
            raise FloatingPointError(f"non-finite gradient norm in layer {layer}")
        self.S[layer] += r
        self.c[layer] += 1

    def window(self):
        return [self.S[l] / self.c[l] if self.c[l] > 0 else None for l in range(self.n)]

    def commit(self, alpha: float, empty_first_ok: bool = False) -> list:
        """empty_first_ok: a schedule without probing (T_p = 0, SPEC.md:451's
        degenerate configuration) commits its first window before any
        observation: m = 0 (uniform probabilities under Eq. 3); every other
        commit needs observations."""
        if not (0.0 <= alpha <= 1.0):
            raise ValueError("alpha must lie in [0, 1]")
        if sum(self.c) == 0 and not (empty_first_ok and not self.committed):
            raise ValueError("commit with zero observations")
        w = self.window()
        if not self.committed:
            # Probing-phase estimate m_l(T_p): every layer observed.
            self.m = [w[l] if w[l] is not None else 0.0 for l in range(self.n)]
            self.committed = True
        else:
            for l in range(self.n):
                if w[l] is not None:
                    self.m[l] = alpha * w[l] + (1.0 - alpha) * self.m[l]
        self.S = [0.0] * self.n
        self.c = [0] * self.n
        return list(self.m)


# ---------------------------------------------------------------------------
# Eq. 3 — softmax sampling distribution
# ---------------------------------------------------------------------------

def softmax_probs(m, tau: float, normalize: bool = True) -> list:
    """p^(l) = exp(m~_l / tau) / sum_i exp(m~_i / tau)   (Eq. 3).

    Reading R3: with ``normalize`` the MGN is max-normalised first,
    m~ = m / max(m) (Fig. 1 plots "normalized" MGN); m == 0
    everywhere gives m~ = 0 (uniform).  The max-subtraction
    z_l = (m~_l - max m~)/tau is the standard overflow-safe form of the same
    ratio.  exp is ``math.exp``; the denominator is the ascending sequential sum.
    """
    if not tau > 0.0:
        raise ValueError("tau must be positive")
    m = [float(x) for x in m]
    if normalize:
        M = max(m)
        mt = [x / M for x in m] if M > 0.0 else [0.0] * len(m)
    else:
        mt = m
    mx = max(mt)
    e = [math.exp((x - mx) / tau) for x in mt]
    tot = 0.0
    for x in e:
        tot += x
    return [x / tot for x in e]


# ---------------------------------------------------------------------------
# gamma-of-N_L layer sampling   (readings R6, R7)
# ---------------------------------------------------------------------------

def splitmix64(x: int) -> int:
    """Standard SplitMix64 output function applied to state x (mod 2^64):
    z = x + 0x9E3779B97F4A7C15; z = (z ^ z>>30)*0xBF58476D1CE4E5B9;
    z = (z ^ z>>27)*0x94D049BB133111EB; return z ^ z>>31."""
    z = (x + GOLDEN_GAMMA) & MASK64
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK64
    return z ^ (z >> 31)


def uniform(seed: int, period: int, k: int) -> float:
    """Counter-based u in [0,1) for draw k of sampling period `period` (R7):
    u = (splitmix64(splitmix64(seed) ^ (period*2^16 + k)) >> 11) * 2^-53."""
    key = splitmix64(seed & MASK64)
    ctr = ((period << 16) + k) & MASK64
    return (splitmix64(key ^ ctr) >> 11) * (2.0 ** -53)


def sample_layers(p, gamma: int, seed: int = 0, period: int = 0, u_fn=None) -> list:
    """Draw gamma DISTINCT layers by sequential draws proportional to p with
    renormalisation (reading R6), in draw order.

    For draw k: R = sum of p over the still-available layers (ascending,
    recomputed), x = u_k * R, walk available layers ascending accumulating
    c += p_l and take the first l with x < c; if none (R == 0), take the last
    available layer.  ``u_fn(k)`` overrides the RNG (used by law tests).
    """
    n = len(p)
    if not (1 <= gamma <= n):
        raise ValueError("gamma must lie in [1, N_L]")
    avail = list(range(n))
    out = []
    for k in range(gamma):
        u = u_fn(k) if u_fn is not None else uniform(seed, period, k)
        R = 0.0
        for l in avail:
            R += p[l]
        x = u * R
        c = 0.0
        pick = avail[-1]
        for l in avail:
            c += p[l]
            if x < c:
                pick = l
                break
        out.append(pick)
        avail.remove(pick)
    return out


def sampling_law_exact(p, gamma: int) -> dict:
    """Exact law of the sequential-draw procedure by enumeration of ordered
    tuples with rational arithmetic (brute force; independent of the RNG)."""
    p = [Fraction(x) for x in p]
    law = {}

    def rec(prefix, prob, remaining_mass):
        if len(prefix) == gamma:
            key = tuple(prefix)
            law[key] = law.get(key, Fraction(0)) + prob
            return
        for l in range(len(p)):
            if l in prefix:
                continue
            rec(prefix + [l], prob * p[l] / remaining_mass, remaining_mass - p[l])

    rec([], Fraction(1), sum(p))
    return law


# ---------------------------------------------------------------------------
# Optimizer update of trainable layers   (reading R1, R2)
# ---------------------------------------------------------------------------

def adamw_step(theta, m, v, g, t: int, lr: float, beta1: float = 0.9,
               beta2: float = 0.999, eps: float = 1e-8, weight_decay: float = 0.0):
    """One AdamW step (torch.optim.AdamW semantics), elementwise, t = t_l + 1:

        theta1 = theta * (1 - lr*wd)
        m'     = beta1*m + (1-beta1)*g
        v'     = beta2*v + (1-beta2)*g^2
        theta' = theta1 - (lr/(1-beta1^t)) * m' / (sqrt(v')/sqrt(1-beta2^t) + eps)

    Computed in fp64 from the (fp32) inputs; theta', m', v' are rounded to fp32
    ONCE (fp32 storage between steps, reading R2).  Returns fp32 arrays.
    """
    if t < 1:
        raise ValueError("t counts updates and starts at 1")
    th = np.asarray(theta, dtype=np.float64)
    m0 = np.asarray(m, dtype=np.float64)
    v0 = np.asarray(v, dtype=np.float64)
    gg = np.asarray(g, dtype=np.float64)
    bc1 = 1.0 - beta1 ** t
    bc2 = 1.0 - beta2 ** t
    th1 = th * (1.0 - lr * weight_decay)
    m1 = beta1 * m0 + (1.0 - beta1) * gg
    v1 = beta2 * v0 + (1.0 - beta2) * gg * gg
    denom = np.sqrt(v1) / math.sqrt(bc2) + eps
    th2 = th1 - (lr / bc1) * m1 / denom
    return th2.astype(np.float32), m1.astype(np.float32), v1.astype(np.float32)


def bf16_to_f32(bits):
    """bf16 bit patterns (uint16) -> exact fp32 values (upper half of the fp32 word)."""
    b = np.asarray(bits, dtype=np.uint16).astype(np.uint32) << np.uint32(16)
    return b.view(np.float32)


def f32_to_bf16(x):
    """fp32 -> bf16 bit patterns, round to nearest even (NaN kept quiet)."""
    u = np.asarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    nan = np.isnan(np.asarray(x, dtype=np.float32))
    r = (u + np.uint64(0x7FFF) + ((u >> np.uint64(16)) & np.uint64(1))) >> np.uint64(16)
    r = np.where(nan, (u >> np.uint64(16)) | np.uint64(0x40), r)
    return r.astype(np.uint16)


def adamw_step_bf16(master, m, v, g_bits, t: int, lr: float, beta1: float = 0.9,
                    beta2: float = 0.999, eps: float = 1e-8, weight_decay: float = 0.0,
                    theta_bits=None):
    """Mixed-precision AdamW (reading R18): bf16 gradient and
    parameters, fp32 master copy and moments.  On a layer's first update
    (theta_bits given) the master is the exact fp32 value of the bf16 parameter.
    Returns (master', m', v' as fp32, theta' as bf16 bits = RNE(master'))."""
    if theta_bits is not None:
        master = bf16_to_f32(theta_bits)
    g = bf16_to_f32(g_bits)
    th, m1, v1 = adamw_step(master, m, v, g, t, lr, beta1, beta2, eps, weight_decay)
    return th, m1, v1, f32_to_bf16(th)


def clip_coefficient(sq_norms, max_norm: float) -> float:
    """Optional global-norm clipping (paper silent; "optional
    global-norm clip flag", reading R17): total = sqrt(sum of the trainable
    layers' squared norms), coef = min(1, max_norm / (total + 1e-6)) —
    torch.nn.utils.clip_grad_norm_ semantics.  The clipped gradient g*coef
    feeds AdamW; the MGN still sees the raw norm (R9)."""
    total = math.sqrt(math.fsum(sq_norms))
    return min(1.0, max_norm / (total + 1e-6))


# ---------------------------------------------------------------------------
# Schedule   (reading R11: T_u = T_s)
# ---------------------------------------------------------------------------

def schedule_decision(step: int, T_p: int, T_s: int, T_u: int | None = None) -> str:
    """'probe' for steps [0, T_p); at T_p 'commit+resample'; thereafter every
    T_s steps 'resample', and at multiples of T_u also 'commit' first."""
    T_u = T_s if T_u is None else T_u
    if step < T_p:
        return "probe"
    d = step - T_p
    if d == 0:
        return "commit+resample"
    if d % T_u == 0:
        return "commit+resample"
    if d % T_s == 0:
        return "resample"
    return "continue"


# ---------------------------------------------------------------------------
# End-to-end driver of the hot path (all rows) on the CPU
# ---------------------------------------------------------------------------

class GrassOracle:
    """The whole hot path: probing accumulation, commit/EMA, softmax, sampling,
    AdamW on the active layers with per-layer step counters t_l (reading R2),
    and MGN accumulation of the active layers' norms.  Optimizer state is kept
    for every layer and never reset.

    n_always (reading R19): the last n_always entries of
    layer_numel are always-trainable groups (embedding, head) -- excluded from
    the MGN window, the probabilities and the sampler; updated like any layer
    when listed."""

    def __init__(self, layer_numel, gamma, tau=1.0, alpha=0.5, normalize=True,
                 beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.0, seed=0, n_always=0, T_p=None):
        self.numel = list(layer_numel)
        self.n = len(self.numel)
        self.n_s = self.n - n_always          # sampled layers [0, n_s)
        assert 1 <= self.n_s and 1 <= gamma <= self.n_s
        self.gamma = gamma
        self.tau, self.alpha, self.normalize = tau, alpha, normalize
        self.beta1, self.beta2, self.eps, self.wd = beta1, beta2, eps, weight_decay
        self.seed = seed
        self.T_p = T_p
        self.mgn = MgnState(self.n_s)
        self.probs = [1.0 / self.n_s] * self.n_s + [0.0] * (self.n - self.n_s)
        self.m = [np.zeros(k, np.float32) for k in self.numel]
        self.v = [np.zeros(k, np.float32) for k in self.numel]
        self.t = [0] * self.n
        self.last_ss = [None] * self.n

    def accumulate(self, layer_ids, grads):
        """Eq. 2 inner term for the listed layers (probing or active)."""
        for l, g in zip(layer_ids, grads):
            ss = sq_norm(g)
            self.last_ss[l] = ss
            if l < self.n_s:                  # always-active groups are not sampled (R19)
                self.mgn.record(l, rms_norm(ss, self.numel[l]))

    def update_probs(self):
        m = self.mgn.commit(self.alpha, empty_first_ok=self.T_p == 0)
        self.probs = list(softmax_probs(m, self.tau, self.normalize)) + [0.0] * (self.n - self.n_s)
        return list(self.probs)

    def sample(self, period, probs=None):
        p = self.probs if probs is None else probs
        return sample_layers(list(p)[:self.n_s], self.gamma, self.seed, period)

    def step_layers(self, layer_ids, params, grads, lr, max_grad_norm=None):
        """AdamW on each listed layer (ascending id, reading R12) and MGN
        accumulation of its (raw) gradient norm; params updated in place
        (fp32).  With max_grad_norm the gradients of this call are clipped by
        their global norm first (R17), rounded to fp32 like a stored grad."""
        order = sorted(range(len(layer_ids)), key=lambda i: layer_ids[i])
        if max_grad_norm:
            coef = clip_coefficient([sq_norm(g) for g in grads], max_grad_norm)
            eff = [(np.asarray(g, np.float64) * coef).astype(np.float32) for g in grads]
        else:
            eff = grads
        for i in order:
            l = layer_ids[i]
            self.t[l] += 1
            th, m1, v1 = adamw_step(params[i], self.m[l], self.v[l], eff[i],
                                    self.t[l], lr, self.beta1, self.beta2,
                                    self.eps, self.wd)
            params[i][...] = th
            self.m[l], self.v[l] = m1, v1
        self.accumulate(layer_ids, grads)
        return params
