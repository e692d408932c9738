"""Shape clustering and superkernel costing (drop-in for gpumux.coalesce).

Both decisions run in the native core: `cluster_shapes` is
gmx_cluster_shapes (coalesce.py:69-106, greedy admission under the padding
budget, deterministic order), `form_superkernel` is gmx_form_superkernel
(coalesce.py:109-131). Padding is a *billing* concept of the decision model:
the B200 executor runs every member at its true dims (see executor.py).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

from . import _lib
from .device import CostEstimate
from .kernels import kernel_desc
from .tuning import ClusterKey, native_table

DEFAULT_PAD_BUDGET = 0.25


@dataclass(frozen=True)
class ShapeCluster:
    op_kind: str
    dtype: str
    padded_dims: tuple
    members: tuple  # admission order
    waste: float

    @property
    def key(self) -> ClusterKey:
        return ClusterKey(self.op_kind, self.dtype, self.padded_dims)

    @property
    def earliest_deadline(self) -> int:
        return min(k.deadline for k in self.members)


@dataclass(frozen=True)
class SuperKernel:
    super_id: str
    members: tuple
    padded_dims: tuple
    batch: int
    flops: int  # padded: batch * flops(padded_dims)
    bytes: int
    earliest_deadline: int
    cost: CostEstimate

    @property
    def useful_flops(self) -> int:
        return sum(k.flops for k in self.members)


def pad_cost(cluster: ShapeCluster) -> float:
    """Fraction of the padded FLOP volume that is padding (native)."""
    if not cluster.members:
        raise ValueError("empty cluster")
    n = len(cluster.members)
    flops = (C.c_int64 * n)(*[k.flops for k in cluster.members])
    out = C.c_double()
    _lib.check(_lib.core().gmx_padding_waste(
        _lib.OP_CODE[cluster.op_kind], flops, n, _lib.dims_array(cluster.padded_dims),
        len(cluster.padded_dims), C.byref(out)))
    return out.value


def cluster_shapes(pending: list, pad_budget: float = DEFAULT_PAD_BUDGET) -> list:
    """Greedy deterministic partition of `pending` into shape clusters (native)."""
    if not 0.0 <= pad_budget < 1.0:
        raise ValueError(f"pad_budget must be in [0, 1), got {pad_budget}")
    pending = list(pending)
    n = len(pending)
    if n == 0:
        return []
    descs = (_lib.KernelDesc * n)(*[kernel_desc(k) for k in pending])
    members = (C.c_int32 * n)()
    offsets = (C.c_int32 * (n + 1))()
    padded = (C.c_int64 * (3 * n))()
    waste = (C.c_double * n)()
    nc = C.c_int32()
    _lib.check(_lib.core().gmx_cluster_shapes(descs, n, float(pad_budget), members, offsets,
                                              padded, waste, C.byref(nc)))
    out = []
    for c in range(nc.value):
        group = tuple(pending[members[i]] for i in range(offsets[c], offsets[c + 1]))
        nd = len(group[0].dims)
        out.append(ShapeCluster(op_kind=group[0].op_kind, dtype=group[0].dtype,
                                padded_dims=tuple(padded[3 * c + d] for d in range(nd)),
                                members=group, waste=waste[c]))
    return out


def superkernel_cost(profile, table, op_kind, dtype, padded_dims, batch, co_tenancy):
    handle, _keep = native_table(table)
    out = _lib.CostC()
    _lib.check(_lib.core().gmx_form_superkernel(
        C.byref(_lib.profile_struct(profile)), handle, _lib.OP_CODE[op_kind],
        _lib.DT_CODE[dtype], _lib.dims_array(padded_dims), len(padded_dims), int(batch),
        int(co_tenancy), C.byref(out)))
    return CostEstimate(out.flops, out.bytes, out.block_count, out.efficiency, out.duration)


def form_superkernel(cluster: ShapeCluster, tuning, profile, co_tenancy: int = 1,
                     super_id: str | None = None) -> SuperKernel:
    """Cost a padded batched coalition (native gmx_form_superkernel)."""
    cost = superkernel_cost(profile, tuning, cluster.op_kind, cluster.dtype,
                            cluster.padded_dims, len(cluster.members), co_tenancy)
    if super_id is None:
        super_id = "sk-" + "-".join(str(k.kernel_id) for k in cluster.members)
    return SuperKernel(super_id=super_id, members=cluster.members,
                       padded_dims=cluster.padded_dims, batch=len(cluster.members),
                       flops=cost.flops, bytes=cost.bytes,
                       earliest_deadline=cluster.earliest_deadline, cost=cost)
