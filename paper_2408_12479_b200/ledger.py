"""Byte ledger of the linearization cell (ledger.cpp:22-76, restated):
per-quadrature-point storage and apply-traffic bytes for (model, domain,
strategy), fp64 (fp32 halves every entry).  Host logic used for the
roofline bytes in bench.py; checked against the reference's own
cell_ledger values in tests/test_oracle.py."""
from __future__ import annotations

SCALAR, VECTOR, SYM, GENERAL = 8, 24, 48, 72


def cell_ledger(model: str, domain: str, strategy: str):
    """Returns the list of (field, bytes, in_traffic) rows."""
    material = domain == "material"
    tensors = strategy == "tensor"
    rows = [("J0", GENERAL, material or not tensors)]
    if not material:
        rows.append(("Jt", GENERAL, True))
    if strategy == "none":
        rows.append(("u_k", VECTOR, True))
        return rows
    if not tensors:
        rows.append(("u_k", VECTOR, True))
    if not material:
        rows.append(("1/J", SCALAR, True))
    if model == "cnh":
        rows.append(("lnJ", SCALAR, True))
    else:
        rows += [("J-1", SCALAR, False if material else not tensors), ("J^-2/3", SCALAR, True),
                 ("c1", SCALAR, True), ("c2", SCALAR, True)]
    if model == "fiber":
        rows += [("c3_4", SCALAR, True), ("c3_6", SCALAR, True),
                 ("I4*", SCALAR, False if material else not tensors), ("I6*", SCALAR, False if material else not tensors),
                 ("E4", SCALAR, True), ("E6", SCALAR, True),
                 ("H4", SYM, True if material else not tensors), ("H6", SYM, True if material else not tensors)]
    if tensors:
        if material:
            rows += [("F", GENERAL, True), ("S", SYM, True), ("F^-1", GENERAL, True), ("C^-1", SYM, True)]
        else:
            rows.append(("tau", SYM, True))
            if model != "cnh":
                rows.append(("b", SYM, True))
            if model == "fiber":
                rows += [("FH4F^T", SYM, True), ("FH6F^T", SYM, True)]
    return rows


def storage_bytes(model, domain, strategy, precision=64):
    return sum(b for _, b, _ in cell_ledger(model, domain, strategy)) * precision // 64


def traffic_bytes(model, domain, strategy, precision=64):
    return sum(b for _, b, t in cell_ledger(model, domain, strategy) if t) * precision // 64
