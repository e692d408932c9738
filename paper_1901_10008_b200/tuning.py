"""Tiling configs and the (cluster key, co-tenancy) -> config table
(drop-in for the lookup side of gpumux.tuning, tuning.py:32-69,147-191).

The table is mirrored into a native `gmx_tuning_table` handle that the
coalescer and scheduler consult (gmx_tuning_table_lookup reproduces
lookup_or_default: tenancy clamps to the key's tuned maximum, misses fall back
to the 64x64 default). The reference's analytical grid search (`tune`) is not
on the hot path and is not re-implemented here; the hardware autotuner that
replaces it writes tables in this same JSON format.
"""

from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass

from . import _lib
from .kernels import validate_dims

TILE_GRID = (16, 32, 64, 128)


@dataclass(frozen=True)
class TuningConfig:
    tile_m: int
    tile_n: int
    sm_footprint: float = 1.0
    efficiency_factor: float = 1.0

    def __post_init__(self):
        if self.tile_m < 1 or self.tile_n < 1:
            raise ValueError("tiles must be >= 1")
        if not 0.0 < self.sm_footprint <= 1.0:
            raise ValueError("sm_footprint must be in (0, 1]")
        if not 0.0 < self.efficiency_factor <= 1.0:
            raise ValueError("efficiency_factor must be in (0, 1]")


DEFAULT_CONFIG = TuningConfig(tile_m=64, tile_n=64, sm_footprint=1.0, efficiency_factor=1.0)


@dataclass(frozen=True)
class ClusterKey:
    op_kind: str
    dtype: str
    dims: tuple

    def __post_init__(self):
        object.__setattr__(self, "dims", validate_dims(self.op_kind, self.dims))

    def as_string(self) -> str:
        return ":".join((self.op_kind, self.dtype, "x".join(str(d) for d in self.dims)))

    @classmethod
    def from_string(cls, text: str) -> "ClusterKey":
        op_kind, dtype, dims = text.split(":")
        return cls(op_kind, dtype, tuple(int(d) for d in dims.split("x")))


class _NativeTable:
    """Owns one gmx_tuning_table built from an `entries` mapping."""

    def __init__(self, entries):
        lib = _lib.core()
        h = C.c_void_p()
        _lib.check(lib.gmx_tuning_table_create(C.byref(h)))
        self.handle = h
        for (key, tenancy), cfg in entries.items():
            _lib.check(lib.gmx_tuning_table_put(
                h, _lib.OP_CODE[key.op_kind], _lib.DT_CODE[key.dtype],
                _lib.dims_array(key.dims), len(key.dims), int(tenancy),
                C.byref(_lib.config_struct(cfg))))

    def __del__(self):
        if getattr(self, "handle", None):
            _lib.core().gmx_tuning_table_destroy(self.handle)
            self.handle = None


def native_table(table):
    """gmx_tuning_table handle for a (duck-typed) TuningTable, or None.

    Cached on the object and rebuilt when its entries changed.
    """
    if table is None:
        return None, None
    sig = (len(table.entries), hash(frozenset(table.entries.items())))
    cache = getattr(table, "_gmx_native", None)
    if cache is None or cache[0] != sig:
        cache = (sig, _NativeTable(table.entries))
        try:
            table._gmx_native = cache
        except AttributeError:
            pass
    return cache[1].handle, cache[1]


class TuningTable:
    """(cluster key, co-tenancy) -> TuningConfig, with search provenance."""

    def __init__(self, entries: dict | None = None, provenance: dict | None = None):
        self.entries = dict(entries or {})
        self.provenance = dict(provenance or {})

    def put(self, key: ClusterKey, co_tenancy: int, config: TuningConfig):
        self.entries[(key, co_tenancy)] = config

    def max_tenancy(self, key: ClusterKey) -> int:
        return max((t for (k, t) in self.entries if k == key), default=0)

    def lookup(self, key: ClusterKey, co_tenancy: int) -> TuningConfig | None:
        handle, _keep = native_table(self)
        out, found = _lib.TuningConfigC(), C.c_int32()
        _lib.check(_lib.core().gmx_tuning_table_lookup(
            handle, _lib.OP_CODE[key.op_kind], _lib.DT_CODE[key.dtype],
            _lib.dims_array(key.dims), len(key.dims), int(co_tenancy), C.byref(out),
            C.byref(found)))
        if not found.value:
            return None
        return TuningConfig(out.tile_m, out.tile_n, out.sm_footprint, out.efficiency_factor)

    def lookup_or_default(self, key: ClusterKey, co_tenancy: int) -> TuningConfig:
        return self.lookup(key, co_tenancy) or DEFAULT_CONFIG

    def to_dict(self) -> dict:
        body = {}
        for (key, tenancy), cfg in sorted(self.entries.items(),
                                          key=lambda kv: (kv[0][0].as_string(), kv[0][1])):
            body.setdefault(key.as_string(), {})[str(tenancy)] = {
                "tile_m": cfg.tile_m, "tile_n": cfg.tile_n,
                "sm_footprint": cfg.sm_footprint, "efficiency_factor": cfg.efficiency_factor}
        return {"provenance": self.provenance, "entries": body}

    @classmethod
    def from_dict(cls, raw: dict) -> "TuningTable":
        table = cls(provenance=raw.get("provenance", {}))
        for text, levels in raw.get("entries", {}).items():
            key = ClusterKey.from_string(text)
            for tenancy, cfg in levels.items():
                table.put(key, int(tenancy), TuningConfig(**cfg))
        return table

    def save(self, path: str):
        with open(path, "w") as fh:
            json.dump(self.to_dict(), fh, indent=2, sort_keys=True)
            fh.write("\n")

    @classmethod
    def load(cls, path: str) -> "TuningTable":
        with open(path) as fh:
            return cls.from_dict(json.load(fh))
