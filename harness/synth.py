"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NONE of the method's arithmetic (no decode, no projection, no
compositing): it only draws scene attributes, cameras and frame packets from
seeded numpy PCG64 streams, with the shapes and distributions SURVEY.md §8(d)
gives for BASELINE.json's configs.  Both sides of every parity test receive the
same arrays from here; neither side's results ever flow back into it.

Conventions:
  * Gaussian SoA ``planes``: float32 ``[P][n_pad]``, P = 11 + 3B, B = (deg+1)^2.
    rows 0-2 position xyz, 3-6 raw quaternion (w,x,y,z), 7-9 log-scale,
    10 opacity logit, 11+3b+ch SH coefficient b, channel ch.
    (PAPER.md:213-215 attributes {p,q,s,o,h}; raw storage per DESIGN reading R1.)
  * Latents: int8 ``[sum L_c][n_pad]`` category-major, categories
    (rot, scale, opacity, sh_dc, sh_rest) = PAPER.md:447 {q, s, o, h} with h split
    into base/freq as in the quantisation table PAPER.md:1333-1372.
  * Decoders: float32 concatenation of row-major ``D_c`` (M_c x L_c).
  * Position residual: COO (strictly increasing u32 indices, float32 [3][k]),
    PAPER.md:1389-1390; or trainer-state gates (log alpha, pre-gated l_p),
    PAPER.md:319-338.
  * Camera: world->camera x_c = R p + t, pinhole fx, fy, cx, cy; pixel k is
    sampled at coordinate k (DESIGN reading R12).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

BASE_SEED = 241204469  # arXiv id, SURVEY.md §8(d)

# PAPER.md:1300-1301 (Table "Gating Hyperparameters"): (tau, gamma0, gamma1)
GATE_N3DV = (0.3, -0.5, 1.01)
GATE_IMMERSIVE = (0.5, -0.1, 1.1)

# residual dimension M_c per category for SH degree `deg`
def category_m(deg: int) -> tuple[int, int, int, int, int]:
    b = (deg + 1) ** 2
    return (4, 3, 1, 3, 3 * (b - 1))


def n_planes(deg: int) -> int:
    return 11 + 3 * (deg + 1) ** 2


@dataclass
class Config:
    name: str
    index: int
    n: int
    frames: int
    views: int
    width: int
    height: int
    focal: float
    deg: int
    lat: tuple  # latent dims (rot, scale, opacity, sh_dc, sh_rest)
    beta: float  # Laplace scale of the integer latents
    rho: float   # fraction of position gates open
    rig: str
    gate: tuple = GATE_N3DV
    logscale_mean: float = math.log(0.01)
    logscale_std: float = 0.6
    n_pad_align: int = 128
    extra: dict = field(default_factory=dict)

    @property
    def n_pad(self) -> int:
        a = self.n_pad_align
        return max(a, (self.n + a - 1) // a * a)

    @property
    def seed(self) -> int:
        return BASE_SEED + self.index


CONFIGS = {
    # BASELINE.json configs[0]: 1,000 Gaussians, 2 frames, 1 camera 64x64, SH 0, 8-dim latents
    "tiny": Config("tiny", 0, 1000, 2, 1, 64, 64, 60.0, 0, (8, 8, 8, 8, 0), 0.22, 0.10,
                   "single", logscale_mean=math.log(0.03), logscale_std=0.5),
    # configs[1]: 300k, 300 frames, 20 views 1352x1014, SH 3, ~10% gates
    "n3dv": Config("n3dv", 1, 300_000, 300, 20, 1352, 1014, 1100.0, 3, (6, 8, 3, 8, 4), 0.22, 0.10, "arc"),
    # configs[2]: 500k, 300 frames, 46 views 1280x960, ~30% gates, highly dynamic
    "immersive": Config("immersive", 2, 500_000, 300, 46, 1280, 960, 640.0, 3, (6, 8, 3, 8, 12), 0.5, 0.30,
                        "hemi", gate=GATE_IMMERSIVE),
    # configs[3]: 150k, 300 frames, 13 views 1280x720, sparse dynamics
    "meetroom": Config("meetroom", 3, 150_000, 300, 13, 1280, 720, 1000.0, 3, (6, 8, 3, 8, 4), 0.15, 0.05, "row"),
    # configs[4]: 3M, 64 views 3840x2160, SH 3, dense residuals
    "stress": Config("stress", 4, 3_000_000, 300, 64, 3840, 2160, 3000.0, 3, (6, 8, 3, 8, 12), 3.0, 1.0,
                     "grid", logscale_mean=math.log(0.006)),
}


def get_config(name: str, **over) -> Config:
    import dataclasses
    return dataclasses.replace(CONFIGS[name], **over)


# ----------------------------------------------------------------------------
# cameras
# ----------------------------------------------------------------------------
@dataclass
class Camera:
    fx: float
    fy: float
    cx: float
    cy: float
    R: np.ndarray  # (3,3) float32 world->camera rotation
    t: np.ndarray  # (3,) float32
    C: np.ndarray  # (3,) float32 camera centre (= -R^T t, computed in float64 then rounded)
    limx: float    # 1.3 * 0.5 W / fx (3D-GS frustum clamp, DESIGN reading R11)
    limy: float
    near: float
    width: int
    height: int

    def as_floats(self) -> np.ndarray:
        """24-word record: fx fy cx cy R[9] t[3] C[3] limx limy near | width height (int32)."""
        f = np.zeros(24, dtype=np.float32)
        f[0:4] = (self.fx, self.fy, self.cx, self.cy)
        f[4:13] = self.R.reshape(-1)
        f[13:16] = self.t
        f[16:19] = self.C
        f[19:22] = (self.limx, self.limy, self.near)
        iv = f.view(np.int32)
        iv[22] = self.width
        iv[23] = self.height
        return f


def _look_at(center, target):
    center = np.asarray(center, np.float64)
    z = np.asarray(target, np.float64) - center
    z /= np.linalg.norm(z)
    down = np.array([0.0, 1.0, 0.0])
    x = np.cross(down, z)
    x /= np.linalg.norm(x)
    y = np.cross(z, x)
    R = np.stack([x, y, z])
    t = -R @ center
    return R, t


def make_camera(R64, t64, fx, fy, width, height, near=0.2) -> Camera:
    R = np.asarray(R64, np.float64)
    t = np.asarray(t64, np.float64)
    C = -R.T @ t
    return Camera(
        fx=float(np.float32(fx)), fy=float(np.float32(fy)),
        cx=float(np.float32((width - 1) / 2.0)), cy=float(np.float32((height - 1) / 2.0)),
        R=R.astype(np.float32), t=t.astype(np.float32), C=C.astype(np.float32),
        limx=float(np.float32(1.3 * 0.5 * width / fx)), limy=float(np.float32(1.3 * 0.5 * height / fy)),
        near=float(np.float32(near)), width=int(width), height=int(height))


def make_cameras(cfg: Config, views: int | None = None) -> list[Camera]:
    V = cfg.views if views is None else views
    rng = np.random.Generator(np.random.PCG64([cfg.seed, 0xCA]))
    cams = []
    for v in range(V):
        if cfg.rig == "single":
            R, t = np.eye(3), np.zeros(3)
        elif cfg.rig == "arc":  # forward-facing, ~1 m arc at z = 0 looking at the scene centre
            a = (v / max(V - 1, 1) - 0.5) * 0.25  # +-0.125 rad on a 4 m radius arc ~ 1 m
            c = np.array([4.0 * math.sin(a), 0.05 * rng.standard_normal(), 4.0 - 4.0 * math.cos(a)])
            R, t = _look_at(c, [0.0, 0.0, 5.0])
        elif cfg.rig == "hemi":  # outward-facing hemispherical rig (Immersive), undistorted pinhole
            g = (1 + 5 ** 0.5) / 2
            k = v + 0.5
            el = math.acos(1 - 0.55 * k / V)  # polar angle up to ~63 deg
            az = 2 * math.pi * k / g
            d = np.array([math.sin(el) * math.cos(az), math.sin(el) * math.sin(az), math.cos(el)])
            c = 0.45 * d
            R, t = _look_at(c, c + d)
        elif cfg.rig == "row":  # MeetRoom: cameras in a horizontal row
            x = (v / max(V - 1, 1) - 0.5) * 1.2
            R, t = _look_at([x, 0.0, 0.0], [0.0, 0.0, 5.0])
        elif cfg.rig == "grid":  # stress: 8x8 grid of forward-facing cameras
            gx = int(math.ceil(math.sqrt(V)))
            i, j = v % gx, v // gx
            c = np.array([(i / max(gx - 1, 1) - 0.5) * 1.0, (j / max(gx - 1, 1) - 0.5) * 0.6, 0.0])
            R, t = _look_at(c, [0.0, 0.0, 5.0])
        else:
            raise ValueError(cfg.rig)
        cams.append(make_camera(R, t, cfg.focal, cfg.focal, cfg.width, cfg.height))
    return cams


# ----------------------------------------------------------------------------
# scene (frame 0 attributes A_0)
# ----------------------------------------------------------------------------
@dataclass
class Scene:
    cfg: Config
    n: int
    n_pad: int
    deg: int
    planes: np.ndarray      # float32 [P][n_pad]
    dynamic: np.ndarray     # int64 indices of "foreground / dynamic" Gaussians (gate pool)


def _rotations(rng, n):
    q = rng.standard_normal((4, n))
    q /= np.linalg.norm(q, axis=0, keepdims=True)
    q *= rng.uniform(0.5, 2.0, n)  # unnormalised storage exercises normalisation
    return q


def make_scene(cfg: Config, n: int | None = None) -> Scene:
    n = cfg.n if n is None else n
    import dataclasses
    if n != cfg.n:
        cfg = dataclasses.replace(cfg, n=n)
    n_pad = cfg.n_pad
    rng = np.random.Generator(np.random.PCG64([cfg.seed, 0x5C]))
    P = n_planes(cfg.deg)
    B = (cfg.deg + 1) ** 2
    pl = np.zeros((P, n_pad), np.float32)
    if cfg.rig == "single":
        pos = np.stack([rng.uniform(-0.5, 0.5, n), rng.uniform(-0.5, 0.5, n), rng.uniform(2.0, 4.0, n)])
        dynamic = np.arange(n)
    else:
        wide = {"arc": 1.0, "row": 1.0, "grid": 1.3, "hemi": 2.2}[cfg.rig]
        n_bg = int(round(0.6 * n))
        n_fg = n - n_bg
        bg = np.stack([rng.uniform(-5.5 * wide, 5.5 * wide, n_bg), rng.uniform(-4.0 * wide, 4.0 * wide, n_bg),
                       rng.uniform(6.0, 8.0, n_bg)])
        centres = np.stack([rng.uniform(-1.0 * wide, 1.0 * wide, 8), rng.uniform(-0.7 * wide, 0.7 * wide, 8),
                            rng.uniform(2.5, 4.5, 8)])
        blob = rng.integers(0, 8, n_fg)
        fg = centres[:, blob] + 0.3 * rng.standard_normal((3, n_fg))
        pos = np.concatenate([bg, fg], axis=1)
        perm = rng.permutation(n)  # interleave background and foreground in index order
        pos = pos[:, perm]
        is_fg = np.concatenate([np.zeros(n_bg, bool), np.ones(n_fg, bool)])[perm]
        dynamic = np.nonzero(is_fg)[0]
    pl[0:3, :n] = pos
    pl[3:7, :n] = _rotations(rng, n)
    ls = rng.normal(cfg.logscale_mean, cfg.logscale_std, (3, n))
    if cfg.rig != "single":
        ls = np.clip(ls, math.log(1e-3), math.log(0.2))
    pl[7:10, :n] = ls
    hi = rng.random(n) < 0.6
    pl[10, :n] = np.where(hi, rng.normal(2.5, 1.0, n), rng.normal(-2.0, 1.5, n))
    pl[11:14, :n] = rng.uniform(-1.5, 1.5, (3, n))
    if B > 1:
        pl[14:11 + 3 * B, :n] = rng.normal(0.0, 0.05, (3 * (B - 1), n))
    return Scene(cfg, n, n_pad, cfg.deg, pl, dynamic.astype(np.int64))


# ----------------------------------------------------------------------------
# frame packets R_t
# ----------------------------------------------------------------------------
@dataclass
class Packet:
    n: int
    n_pad: int
    deg: int
    lat: tuple
    latents: np.ndarray          # int8 [sum L][n_pad]  (wire form)
    latents_f32: np.ndarray | None  # float32 [sum L][n_pad] trainer-state l_hat (rounds to `latents`)
    decoders: np.ndarray         # float32 concat of D_c row-major (M_c x L_c)
    coo_idx: np.ndarray          # uint32 [k] strictly increasing
    coo_val: np.ndarray          # float32 [3][k]
    log_alpha: np.ndarray | None  # float32 [n_pad] (gates mode)
    pos_pregate: np.ndarray | None  # float32 [3][n_pad]
    gate: tuple                  # (tau, gamma0, gamma1)

    @property
    def k(self) -> int:
        return int(self.coo_idx.shape[0])


DEC_SCALE = (2e-3, 5e-3, 2e-2, 5e-3, 2e-3)  # rot, scale, opacity, DC, rest


def make_packet(scene: Scene, t: int, *, gates: bool = True, beta: float | None = None,
                rho: float | None = None, dyadic: bool = False) -> Packet:
    """Residual packet R_t for frame t >= 1."""
    cfg = scene.cfg
    n, n_pad, deg = scene.n, scene.n_pad, scene.deg
    beta = cfg.beta if beta is None else beta
    rho = cfg.rho if rho is None else rho
    rng = np.random.Generator(np.random.PCG64([cfg.seed, 0x9A, t]))
    lat = tuple(cfg.lat if deg > 0 else (cfg.lat[0], cfg.lat[1], cfg.lat[2], cfg.lat[3], 0))
    M = category_m(deg)
    SL = sum(lat)
    q = np.zeros((SL, n_pad), np.int8)
    if dyadic:
        q[:, :n] = rng.integers(-8, 9, (SL, n)).astype(np.int8)
    else:
        lap = np.clip(np.round(rng.laplace(0.0, beta, (SL, n))), -127, 127)
        q[:, :n] = lap.astype(np.int8)
    # trainer-state continuous latents that round (half away from zero) back to q
    lhat = np.zeros((SL, n_pad), np.float32)
    lhat[:, :n] = q[:, :n].astype(np.float32) + rng.uniform(-0.49, 0.49, (SL, n)).astype(np.float32)
    decs = []
    for c in range(5):
        if lat[c] == 0 or M[c] == 0:
            continue
        if dyadic:
            d = rng.integers(-128, 129, (M[c], lat[c])).astype(np.float32) / 1024.0
        else:
            d = (rng.uniform(-1, 1, (M[c], lat[c])) / math.sqrt(lat[c]) * DEC_SCALE[c]).astype(np.float32)
        decs.append(d.reshape(-1))
    decoders = np.concatenate(decs).astype(np.float32) if decs else np.zeros(0, np.float32)
    # position gates: clustered on the dynamic pool
    k = int(round(rho * n))
    pool = scene.dynamic
    if k >= len(pool):
        chosen = np.union1d(pool, rng.choice(np.setdiff1d(np.arange(n), pool), k - len(pool), replace=False)) \
            if k > len(pool) else pool
    else:
        chosen = np.sort(rng.choice(pool, k, replace=False))
    chosen = np.sort(chosen).astype(np.uint32)
    if dyadic:
        val = rng.integers(-64, 65, (3, len(chosen))).astype(np.float32) / 1024.0
    else:
        val = rng.normal(0.0, 2e-3, (3, len(chosen))).astype(np.float32)
    log_alpha = pregate = None
    tau, g0, g1 = cfg.gate
    if gates:
        th0 = np.float32(tau * math.log(-g0 / g1))
        th1 = np.float32(tau * math.log((1 - g0) / (g1 - 1)))
        log_alpha = np.zeros(n_pad, np.float32)
        la = rng.uniform(th0 - 4.0, th0 - 1e-3, n).astype(np.float32)
        la[chosen] = rng.uniform(th0 + 1e-3, th1 + 1.0, len(chosen)).astype(np.float32)
        log_alpha[:n] = la
        log_alpha[n:] = th0 - 1.0
        pregate = np.zeros((3, n_pad), np.float32)
        pregate[:, :n] = rng.normal(0.0, 2e-3, (3, n)).astype(np.float32)
    return Packet(n, n_pad, deg, lat, q, lhat, decoders, chosen, val.astype(np.float32),
                  log_alpha, pregate, (tau, g0, g1))


# ----------------------------------------------------------------------------- first frame
@dataclass
class FirstFrameSH:
    """Frame 0's high-frequency SH coefficients in quantised form: integer latents
    [L][n_pad] int8 (the colour-frequency latent dim of the config) and the decoder [3(B-1)][L]."""
    n: int
    n_pad: int
    deg: int
    latents: np.ndarray
    decoder: np.ndarray


def make_first_frame_sh(scene: Scene, *, beta: float = 1.5, dyadic: bool = False) -> FirstFrameSH:
    """Seeded frame-0 SH latents (Laplace, scale beta: absolute coefficients, not residuals) and
    decoder (U[-1,1]/sqrt(L) x 0.05 -- SH-rest magnitudes of N(0, 0.05^2)); dyadic:
    |l| <= 8 and D on the 2^-10 grid (|D| <= 1/8), so any accumulation order is exact."""
    cfg = scene.cfg
    n, n_pad, deg = scene.n, scene.n_pad, scene.deg
    L = cfg.lat[4] if cfg.lat[4] > 0 else 4
    M = 3 * ((deg + 1) ** 2 - 1)
    rng = np.random.Generator(np.random.PCG64([cfg.seed, 0xF0]))
    q = np.zeros((L, n_pad), np.int8)
    if dyadic:
        q[:, :n] = rng.integers(-8, 9, (L, n)).astype(np.int8)
        d = rng.integers(-128, 129, (M, L)).astype(np.float32) / 1024.0
    else:
        q[:, :n] = np.clip(np.round(rng.laplace(0.0, beta, (L, n))), -127, 127).astype(np.int8)
        d = (rng.uniform(-1, 1, (M, L)) / math.sqrt(L) * 0.05).astype(np.float32)
    return FirstFrameSH(n, n_pad, deg, q, np.ascontiguousarray(d, np.float32))


# ----------------------------------------------------------------------------- NEXT #2
@dataclass
class Delta:
    """Densification delta of frame t (DESIGN reading R21): removals (sorted indices into the
    current set) then additions (raw parameters as IEEE binary16, SoA [P][n_add])."""
    rem: np.ndarray   # uint32 [n_rem], strictly increasing
    add: np.ndarray   # float16 [P][n_add]


def make_delta(state: Scene, t: int, rem_frac: float = 0.005, add_frac: float = 0.01) -> Delta:
    """Synthetic densification of frame t: ~rem_frac of the current Gaussians pruned (uniform),
    ~add_frac cloned from random dynamic Gaussians (3D-GS clone: same attributes, position
    jittered by 5 mm, log-scales shrunk by ln 1.6), stored as binary16."""
    cfg = state.cfg
    rng = np.random.Generator(np.random.PCG64([cfg.seed, 0xD3, t]))
    n = state.n
    n_rem = int(round(rem_frac * n))
    rem = np.sort(rng.choice(n, n_rem, replace=False)).astype(np.uint32) if n_rem else np.zeros(0, np.uint32)
    n_add = int(round(add_frac * n))
    P = 11 + 3 * (state.deg + 1) ** 2
    pool = state.dynamic if len(state.dynamic) else np.arange(n)
    src = rng.choice(pool, n_add, replace=True) if n_add else np.zeros(0, np.int64)
    add = np.zeros((P, n_add), np.float32)
    if state.planes is not None and n_add:
        add[:] = state.planes[:, src]
    else:  # attribute-free state: fresh Gaussians drawn like the scene
        add[0:3] = rng.uniform(-1, 1, (3, n_add))
        add[0:3, :] += np.array([[0.0], [0.0], [3.5]])
        add[3:7] = _rotations(rng, n_add)
        add[7:10] = np.log(0.01)
        add[10] = 2.0
        add[11:14] = rng.uniform(-1.5, 1.5, (3, n_add))
    add[0:3] += rng.normal(0.0, 5e-3, (3, n_add))
    add[7:10] -= np.log(1.6)
    return Delta(rem, add.astype(np.float16))


def advance_state(state: Scene, delta: Delta, n_pad: int | None = None) -> Scene:
    """Bookkeeping of the synthetic stream after a delta (no method arithmetic): new count, the
    dynamic pool re-indexed after the removals, additions counted as dynamic.  The returned
    state carries no planes (the stream's attributes live on the renderer / oracle side)."""
    n = state.n
    keep = np.ones(n, bool)
    keep[delta.rem.astype(np.int64)] = False
    new_index = np.cumsum(keep) - 1
    pool = state.dynamic[keep[state.dynamic]] if len(state.dynamic) else state.dynamic
    pool = new_index[pool]
    n_kept = int(keep.sum())
    n_new = n_kept + delta.add.shape[1]
    pool = np.concatenate([pool, np.arange(n_kept, n_new)]).astype(np.int64)
    n_pad = state.n_pad if n_pad is None else n_pad
    if n_new > n_pad:
        raise ValueError("stream outgrew the capacity n_pad")
    return Scene(state.cfg, n_new, n_pad, state.deg, None, pool)


def make_dyadic_scene(cfg: Config, n: int | None = None) -> Scene:
    """A_0 on the 2^-10 grid with |A_0| <= 256, so dyadic decode/apply is exact in fp32."""
    s = make_scene(cfg, n)
    s.planes = (np.round(s.planes.astype(np.float64) * 1024.0) / 1024.0).astype(np.float32)
    return s


def zero_packet(scene: Scene, lat: tuple | None = None) -> Packet:
    cfg = scene.cfg
    deg = scene.deg
    lat = tuple(lat or (cfg.lat if deg > 0 else (cfg.lat[0], cfg.lat[1], cfg.lat[2], cfg.lat[3], 0)))
    M = category_m(deg)
    SL = sum(lat)
    ndec = sum(M[c] * lat[c] for c in range(5))
    return Packet(scene.n, scene.n_pad, deg, lat, np.zeros((SL, scene.n_pad), np.int8),
                  np.zeros((SL, scene.n_pad), np.float32), np.zeros(ndec, np.float32),
                  np.zeros(0, np.uint32), np.zeros((3, 0), np.float32), None, None, cfg.gate)
