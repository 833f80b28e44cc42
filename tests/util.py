"""Deterministic test inputs (numpy) including the reference's edge cases."""
import numpy as np


def sg_block(rng: np.random.Generator, nsg: int, kind: str = "mixed") -> np.ndarray:
    """nsg super-groups (nsg * 256 fp32 values) of a given flavour."""
    n = nsg * 256
    if kind == "normal":
        return rng.standard_normal(n).astype(np.float32)
    if kind == "lognormal":  # per-SG scale over many decades (locality generator, sigma_log = 4)
        s = np.exp(4.0 * rng.standard_normal(nsg))
        return (rng.standard_normal((nsg, 256)) * s[:, None]).astype(np.float32).ravel()
    if kind == "zeros":
        return np.zeros(n, np.float32)
    if kind == "const":  # every entry equals the group max -> top index, no randomness
        return np.full(n, 2.5, np.float32)
    if kind == "denormal":
        return (rng.standard_normal(n) * 1e-39).astype(np.float32)
    if kind == "huge":
        return (rng.standard_normal(n) * 1e37).astype(np.float32)
    if kind == "codebook":  # values sitting exactly on codebook points of a unit group max
        v = rng.choice(np.array([0.0, 1.0, 0.5, 0.25, -1.0, -0.0, 0.125], np.float32), n)
        v[::16] = 1.0
        return v.astype(np.float32)
    if kind == "mixed":
        parts = []
        kinds = ["normal", "lognormal", "zeros", "const", "denormal", "codebook", "normal", "lognormal"]
        for i in range(nsg):
            parts.append(sg_block(rng, 1, kinds[i % len(kinds)]))
        v = np.concatenate(parts)
        # zero out a few whole groups and plant negative zeros
        for g in rng.integers(0, n // 16, max(1, n // 512)):
            v[g * 16:(g + 1) * 16] = 0.0
        v[rng.integers(0, n, max(1, n // 97))] = -0.0
        return v.astype(np.float32)
    raise ValueError(kind)


def sorted_widths(n8: int, n4: int, n2: int, n16: int = 0) -> np.ndarray:
    return np.array([8] * n8 + [4] * n4 + [2] * n2 + [16] * n16, np.uint8)
