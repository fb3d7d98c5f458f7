"""gen/configs.py — the BASELINE.json workloads as concrete, seeded generator settings.

BASELINE.json "configs":
  C1 one 2^17-packet window, uniform IPv4 pairs                (oracle-sized parity case)
  C2 2^23 packets (64 windows), Zipf s=1.1 over K=2^20 per side (the north_star metric's workload)
  C3 2^23 packets, heavy skew: Bernoulli(1/2) hot source 10.0.0.1, uniform destinations
  C4 2^30 packets (8192 windows), Zipf as C2, generated on device, windows sharded across GPUs
  C5 sweep 2^28..2^32 packets x {uniform, zipf}
Window N_V = 2^17 everywhere (2^30 edges / (128 tar files x 64 matrices)).
"""
from __future__ import annotations

from dataclasses import dataclass

from . import Dist

WINDOW = 1 << 17


@dataclass(frozen=True)
class Config:
    name: str
    n_packets: int
    dist: Dist
    seed: int
    window: int = WINDOW
    note: str = ""


CONFIGS = {
    "C1": Config("C1", 1 << 17, Dist("uniform"), 1, note="single 2^17-packet window, uniform"),
    "C2": Config("C2", 1 << 23, Dist("zipf", 1.1, 1 << 20), 2, note="64 windows, Zipf s=1.1 K=2^20"),
    "C3": Config("C3", 1 << 23, Dist("heavy"), 3, note="64 windows, heavy hot source"),
    "C4": Config("C4", 1 << 30, Dist("zipf", 1.1, 1 << 20), 4, note="8192 windows, Zipf, device-generated"),
}


def sweep_config(log2_n: int, dist_name: str) -> Config:
    d = Dist("zipf", 1.1, 1 << 20) if dist_name == "zipf" else Dist("uniform")
    return Config(f"C5-{dist_name}-2^{log2_n}", 1 << log2_n, d, 5, note="scaling sweep")
