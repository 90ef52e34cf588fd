"""Chunk-mask generators shared by the tests (LoRA-like runs, random, dense)."""
import numpy as np


def lora_like(chunks: int, rng: np.random.Generator, n_runs: int = 6) -> np.ndarray:
    m = np.zeros(chunks, np.uint8)
    for _ in range(n_runs):
        a = int(rng.integers(0, chunks))
        m[a:a + int(rng.integers(1, max(2, chunks // 20)))] = 1
    return m


def random_mask(chunks: int, rng: np.random.Generator, p: float = 0.3) -> np.ndarray:
    return (rng.random(chunks) < p).astype(np.uint8)


def masks(chunks: int, seed: int = 0):
    rng = np.random.default_rng(seed)
    yield "dense", np.ones(chunks, np.uint8)
    yield "frozen", np.zeros(chunks, np.uint8)
    yield "lora", lora_like(chunks, rng)
    yield "random", random_mask(chunks, rng)
    one = np.zeros(chunks, np.uint8)
    one[chunks // 2] = 1
    yield "single", one
