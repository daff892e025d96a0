"""Synthetic image batches of BASELINE.json configs 4 and 5, generated on the GPU.

Per image i and channel c: seeded standard-normal noise,
Gaussian blur sigma = 8 px (truncate 4 sigma, reflect padding), standardise,
add a random linear gradient a (x/(W-1) - 1/2) + b (y/(H-1) - 1/2) with
a, b ~ U(-2, 2), min-max rescale to [0, 255], round, clip, uint8.  Config 5
additionally saturates 10 % of pixel positions (each channel independently
to 0 or 255) and turns a disjoint 5 % into exact grays R = G = B = rint(mean).

The generator is seeded per image, so image i has the same bytes whatever the
sharding (rank r of N generates only its own images).  This is input
plumbing (torch ops), not part of the measured path.
"""

from __future__ import annotations


def _gauss_kernel(sigma: float, truncate: float, device):
    import torch

    r = int(truncate * sigma + 0.5)
    x = torch.arange(-r, r + 1, device=device, dtype=torch.float32)
    k = torch.exp(-0.5 * (x / sigma) ** 2)
    return (k / k.sum()).view(1, 1, -1), r


def correlated_image(index: int, height: int, width: int, *, seed: int = 2010, device="cuda",
                     sigma: float = 8.0, degenerate: bool = False):
    """One (H, W, 3) uint8 image on ``device``."""
    import torch
    import torch.nn.functional as F

    g = torch.Generator(device=device)
    g.manual_seed((seed * 1_000_003 + index) & 0x7FFFFFFFFFFF)
    k, r = _gauss_kernel(sigma, 4.0, device)
    yy = torch.linspace(-0.5, 0.5, height, device=device).view(height, 1)
    xx = torch.linspace(-0.5, 0.5, width, device=device).view(1, width)
    chans = []
    for _ in range(3):
        n = torch.randn((height, width), generator=g, device=device, dtype=torch.float32)
        # separable blur, reflect padding (scipy mode='reflect' ~ torch 'reflect' + edge)
        n = F.pad(n.view(1, 1, height, width), (r, r, 0, 0), mode="reflect")
        n = F.conv2d(n, k.view(1, 1, 1, -1))
        n = F.pad(n, (0, 0, r, r), mode="reflect")
        n = F.conv2d(n, k.view(1, 1, -1, 1)).view(height, width)
        n = (n - n.mean()) / n.std().clamp_min(1e-12)
        ab = torch.rand(2, generator=g, device=device) * 4.0 - 2.0
        n = n + ab[0] * xx + ab[1] * yy
        lo, hi = n.min(), n.max()
        n = (n - lo) * (255.0 / (hi - lo).clamp_min(1e-12))
        chans.append(torch.round(n).clamp_(0, 255).to(torch.uint8))
    img = torch.stack(chans, dim=-1)
    if degenerate:
        flat = img.view(-1, 3)
        u = torch.rand(flat.shape[0], generator=g, device=device)
        sat = u < 0.10
        gray = (u >= 0.10) & (u < 0.15)
        bits = torch.randint(0, 2, flat.shape, generator=g, device=device, dtype=torch.uint8) * 255
        flat[sat] = bits[sat]
        m = torch.round(flat.float().mean(dim=1)).clamp_(0, 255).to(torch.uint8)
        flat[gray] = m[gray].unsqueeze(1).expand(-1, 3)
    return img


def batch(indices, height: int, width: int, *, seed: int = 2010, device="cuda",
          degenerate: bool = False, out=None):
    """(len(indices), H, W, 3) uint8 batch, contiguous (one pixel stream)."""
    import torch

    idx = list(indices)
    if out is None:
        out = torch.empty((len(idx), height, width, 3), dtype=torch.uint8, device=device)
    for j, i in enumerate(idx):
        out[j] = correlated_image(i, height, width, seed=seed, device=device, degenerate=degenerate)
    return out


def shard(n_items: int, world: int, rank: int):
    """Contiguous block partition of n_items over world ranks (rank order = index order)."""
    base, extra = divmod(n_items, world)
    lo = rank * base + min(rank, extra)
    return range(lo, lo + base + (1 if rank < extra else 0))
