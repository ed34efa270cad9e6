"""Hardware presets (presets.py:1-56 of the reference) plus a B200 preset.

The reference presets derive per-direction link rates from a measured
sequential and pipelined swap bandwidth pair.  `b200()` instead takes the
host-link rates this box actually measured (tools/link_probe.cu; see
profiles/ and DESIGN.md) and the 180 GB HBM budget.
"""

from __future__ import annotations

from .model import ConfigError, HwConfig

GIB = 1 << 30

__all__ = ["GIB", "PRESETS", "get_preset", "calibrated", "b200"]


def calibrated(name: str, sequential_swap_bw: float, pipelined_swap_bw: float,
               hbm_bytes: int) -> HwConfig:
    """Sequential swap bw = 2/(E+P), pipelined = 2/max(E,P) solved for the two
    link rates (presets.py:21-37)."""
    d2h = pipelined_swap_bw / 2.0
    denom = 2.0 * d2h - sequential_swap_bw
    if denom <= 0:
        raise ConfigError(f"preset {name}: pipelined bw must exceed sequential")
    return HwConfig(hbm_capacity_bytes=hbm_bytes, dram_capacity_bytes=256 * GIB,
                    bw_d2h_bytes_per_s=d2h,
                    bw_h2d_bytes_per_s=sequential_swap_bw * d2h / denom)


PRESETS = {
    "rtx5080": calibrated("rtx5080", 41.7e9, 63.5e9, 16 * GIB),
    "rtx3080": calibrated("rtx3080", 22.22e9, 39.8e9, 10 * GIB),
}


def get_preset(name: str) -> HwConfig:
    try:
        return PRESETS[name]
    except KeyError:
        raise ConfigError(f"unknown hardware preset {name!r}; available: {sorted(PRESETS)}") from None


def b200(h2d_bytes_per_s: float = 55.5e9, d2h_bytes_per_s: float = 57.2e9,
         hbm_bytes: int = int(180e9), page_size: int = 4096) -> HwConfig:
    """Defaults are this pool's measured pinned-copy rates (link_probe, 1 GiB)."""
    return HwConfig(hbm_capacity_bytes=hbm_bytes, dram_capacity_bytes=1 << 41,
                    bw_d2h_bytes_per_s=d2h_bytes_per_s, bw_h2d_bytes_per_s=h2d_bytes_per_s,
                    page_size_bytes=page_size)
