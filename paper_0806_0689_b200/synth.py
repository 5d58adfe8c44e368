"""Seeded synthetic inputs (frame pairs) shared by the CUDA path's tests/bench and the oracle.

This module holds NONE of the method's arithmetic (no SAD, no search, no PSNR): it only
produces uint8 luma frames.  The paper measures on 18 standard sequences that are
not available; BASELINE.json's configs replace them with synthetic sequences that carry the
paper's statistical shape -- centre-biased, horizontally-directional motion (Table II:
58% zero MV; "22.69% horizontal ... 7.42% vertical").  DESIGN.md "Inputs" states the
recipe; SURVEY.md 8(d) is its source.

Layout: a sequence of ``npairs`` independent pairs is one uint8 tensor ``[npairs, 2, H, W]``;
``[:, 0]`` is the current frame and ``[:, 1]`` the reference frame of the pair, so pair t's
cur/ref sit at a fixed byte stride ``2*H*W`` (the C-ABI's ``pair_stride``).
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np
import torch

MASTER_SEED = 806689


@dataclasses.dataclass(frozen=True)
class SeqConfig:
    name: str
    W: int
    H: int
    B: int
    p: int
    frames: int
    octaves: tuple
    mix: tuple            # (p_zero, p_small, k): zero / directional-small(|mv|<=k, 2:1 h:v) / uniform
    region: int           # MV persistence region, pixels
    epoch_len: int        # MVs are redrawn every epoch_len pairs
    noise: float          # sigma of additive N(0, sigma^2) noise on cur
    pan: str = "none"     # global horizontal pan schedule
    note: str = ""

    @property
    def npairs(self) -> int:
        return self.frames - 1

    @property
    def nb(self) -> int:
        return (self.W // self.B) * (self.H // self.B)

    @property
    def seed(self) -> int:
        return MASTER_SEED + 1000 * int(self.name[1:])


# BASELINE.json "configs" c0..c4 ([proposed] details noted there).
CONFIGS = {
    "c0": SeqConfig("c0", 176, 144, 16, 7, 2, (2.0,), (0.55, 0.25, 1), 16, 1, 2.0,
                    note="one QCIF pair"),
    "c1": SeqConfig("c1", 352, 288, 16, 7, 30, (2.0,), (0.55, 0.25, 1), 48, 5, 2.0,
                    note="CIF, MVs per 3x3-block region, redrawn every 5 frames"),
    "c2": SeqConfig("c2", 352, 288, 16, 15, 300, (2.0,), (0.30, 0.40, 3), 48, 5, 3.0,
                    pan="plus4_half", note="CIF large motion, +4 px pan on half the frames"),
    "c3": SeqConfig("c3", 1920, 1088, 8, 16, 240, (1.0, 4.0, 16.0), (0.55, 0.25, 1), 64, 1, 2.0,
                    pan="pm8", note="1080p, 8x8 blocks, +-8 px/frame pan"),
    "c4": SeqConfig("c4", 3840, 2160, 16, 32, 960, (1.0, 4.0, 16.0), (0.40, 0.35, 4), 64, 8, 2.0,
                    note="2160p, +-32 window"),
}


def _rng(seed: int, stream: int) -> np.random.Generator:
    return np.random.Generator(np.random.Philox(key=[seed & 0xFFFFFFFFFFFFFFFF, stream]))


def _gauss_spectrum(n: int, sigma: float, device) -> torch.Tensor:
    """FFT of a normalised circular Gaussian of radius ceil(3 sigma) on a ring of n."""
    r = int(math.ceil(3 * sigma))
    k = torch.zeros(n, dtype=torch.float64)
    offs = torch.arange(-r, r + 1, dtype=torch.float64)
    w = torch.exp(-0.5 * (offs / sigma) ** 2)
    w = w / w.sum()
    for o, v in zip(range(-r, r + 1), w.tolist()):
        k[o % n] += v
    return torch.fft.fft(k.to(device))


def texture(W: int, H: int, octaves, seed: int, device="cpu") -> torch.Tensor:
    """Toroidal smooth texture: per octave, U[0,1) noise, circular Gaussian blur, standardise;
    sum the octaves, rescale min->16 max->235, round half to even, uint8.  Shape [H, W]."""
    acc = torch.zeros(H, W, dtype=torch.float64, device=device)
    for i, sigma in enumerate(octaves):
        u = torch.from_numpy(_rng(seed, i).random((H, W))).to(device)
        f = torch.fft.fft2(u)
        f = f * _gauss_spectrum(H, sigma, device)[:, None] * _gauss_spectrum(W, sigma, device)[None, :]
        b = torch.fft.ifft2(f).real
        acc += (b - b.mean()) / b.std()
    lo, hi = acc.min(), acc.max()
    t = 16.0 + (acc - lo) * (235.0 - 16.0) / (hi - lo)
    return torch.round(t).clamp(0, 255).to(torch.uint8)


def _pan_step(cfg: SeqConfig, t: int) -> int:
    if cfg.pan == "plus4_half":
        return 4 if ((t - 1) // 10) % 2 == 1 else 0
    if cfg.pan == "pm8":
        return 8 if ((t - 1) // 30) % 2 == 0 else -8
    return 0


def _draw_mix(rng: np.random.Generator, n: int, mix, p: int) -> np.ndarray:
    pz, ps, k = mix
    u = rng.random(n)
    out = np.zeros((n, 2), np.int64)
    small = (u >= pz) & (u < pz + ps)
    unif = u >= pz + ps
    ns = int(small.sum())
    a = rng.integers(1, k + 1, ns)
    sgn = np.where(rng.random(ns) < 0.5, -1, 1)
    minor = np.array([rng.integers(-(ai - 1), ai) for ai in a], np.int64) if ns else np.zeros(0, np.int64)
    horiz = rng.random(ns) < 2.0 / 3.0
    out[small, 0] = np.where(horiz, sgn * a, minor)
    out[small, 1] = np.where(horiz, minor, sgn * a)
    nu = int(unif.sum())
    out[unif] = rng.integers(-p, p + 1, (nu, 2))
    return out


def block_mvs(cfg: SeqConfig, t: int) -> np.ndarray:
    """True (generated) MV per block for pair t (1-based), shape [nby, nbx, 2] (dx, dy)."""
    nbx, nby = cfg.W // cfg.B, cfg.H // cfg.B
    rx, ry = -(-cfg.W // cfg.region), -(-cfg.H // cfg.region)
    epoch = (t - 1) // cfg.epoch_len
    M = _draw_mix(_rng(cfg.seed, 2000 + epoch), rx * ry, cfg.mix, cfg.p).reshape(ry, rx, 2)
    bx = (np.arange(nbx) * cfg.B) // cfg.region
    by = (np.arange(nby) * cfg.B) // cfg.region
    m = M[by[:, None], bx[None, :]].copy()
    m[..., 0] += _pan_step(cfg, t)
    return np.clip(m, -cfg.p, cfg.p)


def make_pair(cfg: SeqConfig, t: int, tex: torch.Tensor, out: torch.Tensor = None) -> torch.Tensor:
    """Pair t (1-based) as a [2, H, W] uint8 tensor on tex.device: (cur, ref).

    ref_t(x,y) = T((x+P_t) mod W, y) with P_t the accumulated pan; cur_t(x,y) =
    clamp(rne(T((x+P_t+m_x) mod W, (y+m_y) mod H) + n)), m the block's MV, n ~ N(0, sigma^2)."""
    dev = tex.device
    H, W, B = cfg.H, cfg.W, cfg.B
    P = sum(_pan_step(cfg, s) for s in range(1, t))
    m = torch.from_numpy(block_mvs(cfg, t)).to(dev)
    mx = m[..., 0].repeat_interleave(B, 0).repeat_interleave(B, 1)
    my = m[..., 1].repeat_interleave(B, 0).repeat_interleave(B, 1)
    ys = torch.arange(H, device=dev)[:, None]
    xs = torch.arange(W, device=dev)[None, :]
    if out is None:
        out = torch.empty(2, H, W, dtype=torch.uint8, device=dev)
    out[1] = tex[ys.expand(H, W), (xs + P) % W]
    disp = tex[(ys + my) % H, (xs + P + mx) % W].to(torch.float32)
    g = torch.Generator(device=dev)
    g.manual_seed(cfg.seed * 7919 + 1000 + t)
    noise = torch.randn(H, W, generator=g, device=dev, dtype=torch.float32) * cfg.noise
    out[0] = torch.round(disp + noise).clamp(0, 255).to(torch.uint8)
    return out


def make_sequence(cfg: SeqConfig, device="cpu", pairs=None) -> torch.Tensor:
    """All pairs (or the 1-based pair indices in ``pairs``) as [n, 2, H, W] uint8."""
    idx = list(range(1, cfg.frames)) if pairs is None else list(pairs)
    tex = texture(cfg.W, cfg.H, cfg.octaves, cfg.seed, device)
    out = torch.empty(len(idx), 2, cfg.H, cfg.W, dtype=torch.uint8, device=device)
    for k, t in enumerate(idx):
        make_pair(cfg, t, tex, out[k])
    return out


def shard(npairs: int, world: int, rank: int):
    """Contiguous pair range [lo, hi) of rank (ceil split); last ranks may be short."""
    per = -(-npairs // world)
    lo = min(npairs, rank * per)
    return lo, min(npairs, lo + per)


# ---------------------------------------------------------------------------------------
# Special-purpose fixtures (tests): flat, binary noise, translation, pixel-ideal mosaic.
# ---------------------------------------------------------------------------------------

def flat_pair(W, H, value=128):
    f = np.full((H, W), value, np.uint8)
    return f.copy(), f.copy()


def binary_pair(W, H, seed):
    r = _rng(seed, 77)
    return r.integers(0, 2, (H, W)).astype(np.uint8), r.integers(0, 2, (H, W)).astype(np.uint8)


def random_pair(W, H, seed):
    r = _rng(seed, 78)
    return r.integers(0, 256, (H, W)).astype(np.uint8), r.integers(0, 256, (H, W)).astype(np.uint8)


def translated_pair(tex: np.ndarray, dx: int, dy: int):
    """cur(x,y) = ref(x+dx, y+dy) on a toroidal texture (no noise): the true MV is (dx,dy)."""
    ref = np.ascontiguousarray(tex, dtype=np.uint8)
    cur = np.roll(np.roll(ref, -dy, axis=0), -dx, axis=1)
    return np.ascontiguousarray(cur), ref


def _ideal_profile(B: int, p: int, o: int, t: int, n: int) -> np.ndarray:
    """u on [0, n) with sum_{j<B} u(o+d+j) = (d-t)^2 + const for |d| <= p (block origin o).

    Built from u(c+B) = u(c) + 2(c-o-t)+1, each residue chain shifted to a minimum of 0."""
    u = np.zeros(n, np.int64)
    start = o - p
    for c0 in range(start, start + B):
        vals = [0]
        c = c0
        while c + B < o + p + B:
            vals.append(vals[-1] + 2 * (c - o - t) + 1)
            c += B
        vals = np.array(vals) - min(vals)
        for k, v in enumerate(vals):
            u[c0 + k * B] = v
    return u


def ideal_mosaic(B: int, p: int = 7):
    """Pixel-ideal mosaic (SURVEY finding 5): a (2p+1) x (2p+1) grid of tiles; tile (ty,tx)
    has its checked block at tile offset (B_off, B_off) with a true MV t = (tx-p, ty-p).

    cur is 0 everywhere; ref in each tile is u(x)+v(y), so every candidate's SAD of the
    checked block is exactly B*|q-t|^2 + K -- the ideal surface of P:301 up to a monotone
    map.  Returns (cur, ref, tile, off, checked_block_indices[ty, tx])."""
    tile = 3 * B if B == 16 else 4 * B     # 48 for B=16; 32 for B=8 (keeps W % 16 == 0)
    off = B
    assert off - p >= 0 and off + B + p <= tile
    side = 2 * p + 1
    W = H = tile * side
    cur = np.zeros((H, W), np.uint8)
    ref = np.zeros((H, W), np.uint8)
    nbx = W // B
    blocks = np.zeros((side, side), np.int64)
    for ty in range(side):
        for tx in range(side):
            u = _ideal_profile(B, p, off, tx - p, tile)
            v = _ideal_profile(B, p, off, ty - p, tile)
            t = u[None, :] + v[:, None]
            assert t.max() <= 255
            ref[ty * tile:(ty + 1) * tile, tx * tile:(tx + 1) * tile] = t
            blocks[ty, tx] = ((ty * tile + off) // B) * nbx + (tx * tile + off) // B
    return cur, ref, tile, off, blocks
