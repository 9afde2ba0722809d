"""Seeded synthetic inputs for the five BASELINE configs.

This module is shared by the product tests, the oracle tests and bench.py.
It holds NO arithmetic of the method (no log-factors, weights, moments,
M-step or EMA): only model *shapes*, ancestral data generation from the prior
(numpy PCG64, data seed = config id) and standard-normal
draws for the parity mode of the sampler.

Configs (BASELINE.json ``configs``; readings in DESIGN.md):
  1  tiny conjugate Gaussian:  mu~N(0,1); z_i~N(mu,1), M=4; x_ij~N(z_i,1), J=5; K=8, T=20
  2  hierarchical logistic:    mu in R^18, psi~N(0,1); z_i~N(mu, e^psi I), M=300;
                               x_ij in {0,1}^18 ~ Bern(0.2); y~Bern(sigmoid(z.x)), J=5; K=30, T=100
  3  three-level Poisson:      g, beta in R^6 ~ N(0,1); u_a~N(g,1), A=6; v_ab~N(u_a,0.5^2), B=30;
                               x~N(0,I_6); y~Pois(exp(v+beta.x)), J=10; K=30, T=100
  4  large Gaussian:           mu, logsigma ~N(0,1); z_i~N(mu, e^{2 logsigma}), M=1e5; x~N(z,1), J=32;
                               K=256, T=50
  5  large-K logistic:         as 2 with d=16, M=1e4, J=20, K=1024, T=10
The paper's datasets are not in the container; these
prior-drawn synthetic sets stand in for them (Radon-shaped: 1 and 4,
PAPER.md:1245-1262; MovieLens-shaped: 2 and 5, PAPER.md:1002-1029;
Bus-like nesting: 3).
"""
from __future__ import annotations

import dataclasses
from typing import Optional

import numpy as np

# Family / kind codes (plain ints; the C-ABI and the oracle each define their own).
FAMILY_TWO_LEVEL = 2
FAMILY_THREE_LEVEL = 3
SCALE_FIXED = 0
SCALE_LOGSIGMA = 1  # group variance exp(2 s)
SCALE_LOGVAR = 2    # group variance exp(s)  (psi)
OBS_GAUSS = 1
OBS_BERNOULLI_LOGIT = 2
OBS_POISSON_LOG = 3


@dataclasses.dataclass
class Model:
    family: int
    K: int
    T: int
    # two-level
    d: int = 1
    scale_kind: int = SCALE_FIXED
    fixed_var: float = 1.0
    obs_kind: int = OBS_GAUSS
    obs_var: float = 1.0
    n: int = 0          # groups (two-level) / top-level groups A (three-level)
    J: int = 0
    # three-level
    B: int = 0
    P: int = 0
    top_var: float = 1.0
    sub_var: float = 0.25
    prior_mean: float = 0.0
    prior_var: float = 1.0
    config_id: int = 0
    name: str = ""

    @property
    def R(self) -> int:
        """Root latent dims (one shared copy index, R2)."""
        if self.family == FAMILY_TWO_LEVEL:
            return self.d + (1 if self.scale_kind != SCALE_FIXED else 0)
        return 1 + self.P

    @property
    def pairs(self) -> int:
        """Factor pairs N*K^2 of one E-step."""
        if self.family == FAMILY_TWO_LEVEL:
            return self.n * self.K * self.K
        return (self.n * self.B) * self.K * self.K


def config(cid: int, *, n: Optional[int] = None, K: Optional[int] = None, J: Optional[int] = None,
           d: Optional[int] = None, B: Optional[int] = None) -> Model:
    """The BASELINE config ``cid`` (1..5), optionally resized (mini shapes for tests)."""
    if cid == 1:
        m = Model(FAMILY_TWO_LEVEL, K=8, T=20, d=1, scale_kind=SCALE_FIXED, fixed_var=1.0,
                  obs_kind=OBS_GAUSS, obs_var=1.0, n=4, J=5, config_id=1, name="tiny-conjugate-gaussian")
    elif cid == 2:
        m = Model(FAMILY_TWO_LEVEL, K=30, T=100, d=18, scale_kind=SCALE_LOGVAR, obs_kind=OBS_BERNOULLI_LOGIT,
                  n=300, J=5, config_id=2, name="hier-logistic-d18")
    elif cid == 3:
        m = Model(FAMILY_THREE_LEVEL, K=30, T=100, n=6, B=30, J=10, P=6, top_var=1.0, sub_var=0.25,
                  obs_kind=OBS_POISSON_LOG, config_id=3, name="three-level-poisson")
    elif cid == 4:
        m = Model(FAMILY_TWO_LEVEL, K=256, T=50, d=1, scale_kind=SCALE_LOGSIGMA, obs_kind=OBS_GAUSS,
                  obs_var=1.0, n=100_000, J=32, config_id=4, name="large-gaussian-M1e5-K256")
    elif cid == 5:
        m = Model(FAMILY_TWO_LEVEL, K=1024, T=10, d=16, scale_kind=SCALE_LOGVAR, obs_kind=OBS_BERNOULLI_LOGIT,
                  n=10_000, J=20, config_id=5, name="large-K-logistic-d16-K1024")
    else:
        raise ValueError(f"unknown config {cid}")
    if n is not None:
        m.n = n
    if K is not None:
        m.K = K
    if J is not None:
        m.J = J
    if d is not None:
        m.d = d
    if B is not None:
        m.B = B
    return m


@dataclasses.dataclass
class Data:
    """Observations (host numpy) plus the true latents they were drawn from."""
    xg: Optional[np.ndarray] = None   # [n][J] f32 (OBS_GAUSS)
    xb: Optional[np.ndarray] = None   # [n][J][d] u8 (OBS_BERNOULLI_LOGIT)
    yb: Optional[np.ndarray] = None   # [n][J] u8
    xp: Optional[np.ndarray] = None   # [A*B][J][P] f32 (OBS_POISSON_LOG)
    yp: Optional[np.ndarray] = None   # [A*B][J] i32
    truth: dict = dataclasses.field(default_factory=dict)


def make_data(m: Model, seed: Optional[int] = None) -> Data:
    """Ancestral draw from the prior (data seed = config id unless given)."""
    rng = np.random.Generator(np.random.PCG64(m.config_id if seed is None else seed))
    if m.family == FAMILY_TWO_LEVEL:
        mu = rng.standard_normal(m.d)
        s = rng.standard_normal() if m.scale_kind != SCALE_FIXED else 0.0
        if m.scale_kind == SCALE_FIXED:
            var = m.fixed_var
        elif m.scale_kind == SCALE_LOGSIGMA:
            var = np.exp(2.0 * s)
        else:
            var = np.exp(s)
        z = mu[None, :] + np.sqrt(var) * rng.standard_normal((m.n, m.d))
        out = Data(truth={"mu": mu, "s": s, "z": z})
        if m.obs_kind == OBS_GAUSS:
            assert m.d == 1
            x = z[:, 0:1] + np.sqrt(m.obs_var) * rng.standard_normal((m.n, m.J))
            out.xg = x.astype(np.float32)
        else:
            xb = (rng.random((m.n, m.J, m.d)) < 0.2).astype(np.uint8)
            eta = np.einsum("njd,nd->nj", xb.astype(np.float64), z)
            p = 1.0 / (1.0 + np.exp(-eta))
            out.xb = xb
            out.yb = (rng.random((m.n, m.J)) < p).astype(np.uint8)
        return out
    # three-level
    g = rng.standard_normal()
    beta = rng.standard_normal(m.P)
    u = g + np.sqrt(m.top_var) * rng.standard_normal(m.n)
    v = np.repeat(u, m.B) + np.sqrt(m.sub_var) * rng.standard_normal(m.n * m.B)
    x = rng.standard_normal((m.n * m.B, m.J, m.P)).astype(np.float32)
    eta = v[:, None] + np.einsum("sjp,p->sj", x.astype(np.float64), beta)
    y = rng.poisson(np.exp(eta)).astype(np.int32)
    return Data(xp=x, yp=y, truth={"g": g, "beta": beta, "u": u, "v": v})


def make_test_data(m: Model, data: Data, J_test: Optional[int] = None, seed: Optional[int] = None) -> Data:
    """Held-out observations of the SAME groups (a separate 'test' set), drawn
    from the likelihood at the training draw's true group latents (two-level family); seed
    defaults to 1000 + config id, J_test to the training J."""
    assert m.family == FAMILY_TWO_LEVEL
    J = m.J if J_test is None else J_test
    rng = np.random.Generator(np.random.PCG64(1000 + m.config_id if seed is None else seed))
    z = data.truth["z"]
    out = Data(truth=data.truth)
    if m.obs_kind == OBS_GAUSS:
        out.xg = (z[:, 0:1] + np.sqrt(m.obs_var) * rng.standard_normal((m.n, J))).astype(np.float32)
    else:
        xb = (rng.random((m.n, J, m.d)) < 0.2).astype(np.uint8)
        eta = np.einsum("njd,nd->nj", xb.astype(np.float64), z)
        out.xb = xb
        out.yb = (rng.random((m.n, J)) < 1.0 / (1.0 + np.exp(-eta))).astype(np.uint8)
    return out


def eps_normal(shape, seed: int) -> np.ndarray:
    """Host standard-normal draws (fp32) for the sampler's parity mode."""
    rng = np.random.Generator(np.random.PCG64(seed))
    return rng.standard_normal(shape).astype(np.float32)


def latent_shapes(m: Model):
    """Per-level (instances, dims) of the sample bank, root first."""
    if m.family == FAMILY_TWO_LEVEL:
        return [(1, m.R), (m.n, m.d)]
    return [(1, m.R), (m.n, 1), (m.n * m.B, 1)]


def initial_q(m: Model):
    """Q initialised to N(0,1) per latent dim (App. F Q blocks, e.g. PAPER.md:883-893, 1023-1025)."""
    return [(np.zeros(n * dd, np.float32), np.ones(n * dd, np.float32)) for n, dd in latent_shapes(m)]


def random_q(m: Model, seed: int, spread: float = 1.0):
    """A non-trivial Q (seeded) for E-step parity cases: means near the data truth, various widths."""
    rng = np.random.Generator(np.random.PCG64(seed))
    out = []
    for n, dd in latent_shapes(m):
        mean = (0.5 * rng.standard_normal(n * dd)).astype(np.float32)
        var = (spread * np.exp(0.3 * rng.standard_normal(n * dd))).astype(np.float32)
        out.append((mean, var))
    return out



# ------------------------------------------------------------------ discrete latents (row f1)


@dataclasses.dataclass
class Occupancy:
    """Occupancy-shaped discrete-latent model (R30): root r in R^d
    ~ N(0, I); per site i a categorical z_i in {0..C-1} with prior logits x_ic . r; R repeated
    Bernoulli detections y_ir with per-state logits l_irc.  Default shape: J=12 species x M=6
    years x I=200 routes = 14400 sites, R=5 repeats, C=2 (absent / present),
    d=2 (occupancy intercept, weather weight)."""
    n: int
    C: int
    R: int
    d: int
    K: int
    x: np.ndarray       # [n][C][d] float64 state covariates (state 0: zeros)
    logit: np.ndarray   # [n][R][C] float64 detection logits
    y: np.ndarray       # [n][R] uint8
    r_true: np.ndarray  # [d] the root draw the data came from
    z_true: np.ndarray  # [n] int


def occupancy(n: int = 14400, R: int = 5, K: int = 64, C: int = 2, seed: int = 6) -> Occupancy:
    """Ancestral draw from the prior (numpy PCG64, `seed`).  Covariates: weather_i ~ N(0, 1);
    present-state covariates (1, weather_i) (further states: independent N(0, 1) covariates);
    detection logits: absent -10 (the paper's false-positive logit), present
    2 quality_ir - 0.5 with quality_ir ~ Bern(0.8) (the paper's quality covariate with its weight
    fixed), further states N(0, 1)."""
    rng = np.random.default_rng(seed)
    d = 2
    x = np.zeros((n, C, d))
    weather = rng.normal(0.0, 1.0, n)
    x[:, 1, 0] = 1.0
    x[:, 1, 1] = weather
    if C > 2:
        x[:, 2:, :] = rng.normal(0.0, 1.0, (n, C - 2, d))
    logit = np.zeros((n, R, C))
    logit[:, :, 0] = -10.0
    quality = rng.random((n, R)) < 0.8
    logit[:, :, 1] = 2.0 * quality - 0.5
    if C > 2:
        logit[:, :, 2:] = rng.normal(0.0, 1.0, (n, R, C - 2))
    r = rng.normal(0.0, 1.0, d)
    eta = x @ r                                              # [n][C]
    pz = np.exp(eta - eta.max(axis=1, keepdims=True))
    pz /= pz.sum(axis=1, keepdims=True)
    u = rng.random(n)
    z = np.minimum((u[:, None] >= np.cumsum(pz, axis=1)).sum(axis=1), C - 1)
    lz = logit[np.arange(n), :, z]                           # [n][R]
    y = (rng.random((n, R)) < 1.0 / (1.0 + np.exp(-lz))).astype(np.uint8)
    return Occupancy(n=n, C=C, R=R, d=d, K=K, x=x, logit=logit, y=y, r_true=r, z_true=z)


@dataclasses.dataclass
class GammaPoisson:
    """Gamma-Poisson hierarchy under a Gaussian root (row f1's Gamma Q; R32):
    mu ~ N(0, 1); lambda_i | mu ~ Gamma(shape alpha, rate alpha e^-mu); y_ij ~ Poisson(lambda_i)."""
    n: int
    J: int
    K: int
    alpha: float
    y: np.ndarray        # [n][J] int32
    mu_true: float
    lam_true: np.ndarray  # [n]


def gamma_poisson(n: int = 2000, J: int = 8, K: int = 128, alpha: float = 2.0, seed: int = 7) -> GammaPoisson:
    """Ancestral draw from the prior (numpy PCG64, `seed`)."""
    rng = np.random.default_rng(seed)
    mu = float(rng.normal())
    lam = rng.gamma(alpha, np.exp(mu) / alpha, n)          # numpy: (shape, scale = 1 / rate)
    y = rng.poisson(lam[:, None], (n, J)).astype(np.int32)
    return GammaPoisson(n=n, J=J, K=K, alpha=alpha, y=y, mu_true=mu, lam_true=lam)


@dataclasses.dataclass
class BetaBinomial:
    """Beta-Binomial hierarchy under a Gaussian root (row f1's Beta Q; R32):
    mu ~ N(0, 1); p_i | mu ~ Beta(kappa s, kappa (1 - s)), s = sigmoid(mu); y_i ~ Binomial(N_i, p_i)."""
    n: int
    K: int
    kappa: float
    y: np.ndarray   # [n] int32
    N: np.ndarray   # [n] int32 trials
    mu_true: float
    p_true: np.ndarray


def beta_binomial(n: int = 2000, K: int = 128, kappa: float = 8.0, n_max: int = 30, seed: int = 8) -> BetaBinomial:
    """Ancestral draw from the prior (numpy PCG64, `seed`); trials N_i uniform on 1..n_max."""
    rng = np.random.default_rng(seed)
    mu = float(rng.normal())
    s = 1.0 / (1.0 + np.exp(-mu))
    p = rng.beta(kappa * s, kappa * (1.0 - s), n)
    N = rng.integers(1, n_max + 1, n).astype(np.int32)
    y = rng.binomial(N, p).astype(np.int32)
    return BetaBinomial(n=n, K=K, kappa=kappa, y=y, N=N, mu_true=mu, p_true=p)


@dataclasses.dataclass
class Crossed:
    """Bus-Breakdown-shaped crossed effects (row f4; R33): root
    (mu, C company weights, T journey-type weights) ~ N(0, I); n year-borough groups
    w_i ~ N(mu, 1); J delays per group ~ Bernoulli(sigmoid(w_i + cw_comp + jw_type)) with
    per-observation company / journey-type index tables."""
    n: int
    J: int
    C: int
    T: int
    K: int
    comp: np.ndarray    # [n][J] int32
    jtype: np.ndarray   # [n][J] int32
    y: np.ndarray       # [n][J] uint8
    root_true: np.ndarray
    w_true: np.ndarray

    @property
    def R(self) -> int:
        return 1 + self.C + self.T


def bus_crossed(n: int = 120, J: int = 40, C: int = 57, T: int = 6, K: int = 64, seed: int = 9) -> Crossed:
    """Ancestral draw from the prior (numpy PCG64, `seed`).  Defaults: 57 companies and 6
    journey types as in the paper's Bus data, 12 years x 10 boroughs = 120
    year-borough groups, 40 recorded journeys each."""
    rng = np.random.default_rng(seed)
    root = rng.normal(0.0, 1.0, 1 + C + T)
    w = root[0] + rng.normal(0.0, 1.0, n)
    comp = rng.integers(0, C, (n, J)).astype(np.int32)
    jtype = rng.integers(0, T, (n, J)).astype(np.int32)
    eta = w[:, None] + root[1 + comp] + root[1 + C + jtype]
    y = (rng.random((n, J)) < 1.0 / (1.0 + np.exp(-eta))).astype(np.uint8)
    return Crossed(n=n, J=J, C=C, T=T, K=K, comp=comp, jtype=jtype, y=y, root_true=root, w_true=w)


def posterior_like_q(m: Model, data: Data, seed: int = 5, shrink: float = 1.0):
    """A Q centred near the data-generating truth with roughly posterior widths:
    the converged regime of QEM, where the root weights are spread (H1)."""
    rng = np.random.Generator(np.random.PCG64(seed))
    t = data.truth
    if m.family == FAMILY_TWO_LEVEL:
        rm = list(t["mu"]) + ([t["s"]] if m.scale_kind != SCALE_FIXED else [])
        rsd = shrink * 1.0 / np.sqrt(max(m.n, 1))
        root_m = np.asarray(rm) + rsd * rng.standard_normal(m.R)
        root_v = np.full(m.R, rsd ** 2)
        z = np.asarray(t["z"]).reshape(-1)
        gsd = shrink * 1.0 / np.sqrt(max(m.J, 1) * 0.25 + 1.0)
        gm = z + gsd * rng.standard_normal(z.size)
        gv = np.full(z.size, gsd ** 2)
        return [(root_m.astype(np.float32), root_v.astype(np.float32)),
                (gm.astype(np.float32), gv.astype(np.float32))]
    rm = [t["g"]] + list(t["beta"])
    rsd = shrink * 0.01
    root_m = np.asarray(rm) + rsd * rng.standard_normal(m.R)
    u, v = np.asarray(t["u"]), np.asarray(t["v"])
    return [(root_m.astype(np.float32), np.full(m.R, rsd ** 2, np.float32)),
            ((u + 0.3 * rng.standard_normal(u.size)).astype(np.float32), np.full(u.size, 0.09, np.float32)),
            ((v + 0.01 * rng.standard_normal(v.size)).astype(np.float32), np.full(v.size, 1e-4, np.float32))]
