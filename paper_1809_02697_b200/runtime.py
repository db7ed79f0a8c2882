"""Execution resources of the B200 build.

The reference runtime.py (:24-149) is a static-partition CPU thread pool
that splits conv output rows across pinned workers.  On a B200 the intra-op
split is the CUDA grid (a persistent tile scheduler inside each kernel), so
what remains of the runtime is (a) which device(s) and arithmetic mode a
call runs with, and (b) the contiguous batch split used to shard a graph
across the GPUs of one box (north_star piece 4).  ``split_ranges`` keeps the
reference's chunking rule (runtime.py:129-137)."""

from __future__ import annotations

import os
from dataclasses import dataclass, field

MODES = ("fp32", "tf32", "bf16", "fp8")


def default_mode() -> str:
    mode = os.environ.get("NEOB200_MODE", "tf32")
    if mode not in MODES:
        raise ValueError(f"NEOB200_MODE={mode!r}; choose from {MODES}")
    return mode


def device_count() -> int:
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


def physical_cores() -> int:
    """Host cores (kept for the reference API; used by the CPU baseline)."""
    try:
        import psutil
        return psutil.cpu_count(logical=False) or os.cpu_count() or 1
    except Exception:
        return os.cpu_count() or 1


def split_ranges(n_items: int, n_parts: int) -> list[tuple[int, int]]:
    """Contiguous chunks of ceil(n/parts) items; empty chunks dropped."""
    if n_items <= 0:
        return []
    parts = max(1, min(n_parts, n_items))
    step = -(-n_items // parts)
    return [(lo, min(lo + step, n_items)) for lo in range(0, n_items, step)]


@dataclass
class DevicePool:
    """Where and how a graph or an operator runs: a device index (or several
    for batch sharding) and the conv arithmetic mode (fp32 | tf32 | bf16)."""

    devices: list = field(default_factory=lambda: [0])
    mode: str = field(default_factory=default_mode)

    def __post_init__(self):
        if isinstance(self.devices, int):
            self.devices = [self.devices]
        if self.mode not in MODES:
            raise ValueError(f"mode {self.mode!r} not in {MODES}")
        if not self.devices:
            raise ValueError("DevicePool needs at least one device")

    @property
    def device(self) -> int:
        return self.devices[0]

    @property
    def size(self) -> int:
        return len(self.devices)

    def shards(self, batch: int) -> list[tuple[int, tuple[int, int]]]:
        """(device, [lo, hi)) batch ranges, one per device that gets work."""
        return list(zip(self.devices, split_ranges(batch, len(self.devices))))

    # context-manager symmetry with the reference ThreadPool
    def __enter__(self):
        return self

    def __exit__(self, *exc):
        return False

    def close(self):
        pass


def resolve_pool(pool) -> DevicePool:
    if pool is None:
        return DevicePool()
    if isinstance(pool, DevicePool):
        return pool
    if isinstance(pool, str):
        return DevicePool(mode=pool)
    raise TypeError(f"expected DevicePool, mode string or None, got {type(pool).__name__}")


class ThreadPool(DevicePool):
    """Reference name (runtime.py:36-126) so ``with ThreadPool(n) as pool:
    execute(g, inputs, pool)`` keeps working: on a B200 the intra-op split
    is the CUDA grid, so the thread count is recorded but the pool runs on
    ``devices`` (default GPU 0) in ``mode``.  Host-side ``parallel_for``
    still uses ``num_threads`` worker threads."""

    def __init__(self, num_threads: int | None = None, devices=None, mode: str | None = None):
        super().__init__(devices if devices is not None else [0], mode or default_mode())
        self.num_threads = num_threads or default_num_threads()


def default_num_threads() -> int:
    """NEOPLAN_NUM_THREADS or the physical core count (runtime.py:29-33)."""
    env = os.environ.get("NEOPLAN_NUM_THREADS")
    if env:
        try:
            return max(1, int(env))
        except ValueError:
            pass
    return physical_cores()


def parallel_for(pool, n_items: int, body) -> None:
    """Host-side static-partition loop (runtime.py:140-149): ``body(lo, hi)``
    over ``split_ranges(n_items, threads)`` on worker threads, joined before
    returning; the first exception is re-raised.  Device work never goes
    through here (kernels own their grids)."""
    from concurrent.futures import ThreadPoolExecutor
    threads = getattr(pool, "num_threads", None) or default_num_threads()
    chunks = split_ranges(n_items, threads)
    if len(chunks) <= 1:
        for lo, hi in chunks:
            body(lo, hi)
        return
    with ThreadPoolExecutor(max_workers=len(chunks)) as ex:
        futures = [ex.submit(body, lo, hi) for lo, hi in chunks]
    for f in futures:
        f.result()
