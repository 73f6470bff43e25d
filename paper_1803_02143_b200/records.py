"""Run-record writers: the diagnostics CSV and its ``.meta`` sidecar.

Same format as the reference CLI's writers (/root/reference/pkg/src/slvp/cli.py:185-232:
``.17g`` numbers, one header line, newline-terminated; ``key = value`` meta
lines with the keys sorted), so a run on the device produces files the
reference tooling reads unchanged.
"""

from __future__ import annotations

from pathlib import Path
from typing import Sequence

from . import __version__

_CSV_HEADER = "time,electric_energy,mass,l1_norm,l2_norm,kinetic_energy,total_energy"


def _g17(value: float) -> str:
    return format(float(value), ".17g")


def _write_lines(path: Path, lines: Sequence[str]) -> None:
    path = Path(path)
    path.parent.mkdir(parents=True, exist_ok=True)
    path.write_text("\n".join(lines) + "\n")


def write_diagnostics_csv(path, records) -> None:
    """One row per DiagnosticsRecord (cli.py:193-200)."""
    lines = [_CSV_HEADER]
    for r in records:
        lines.append(",".join(_g17(v) for v in (
            r.time, r.electric_energy, r.mass, r.l1_norm, r.l2_norm,
            r.kinetic_energy, r.total_energy,
        )))
    _write_lines(Path(path), lines)


def write_meta(out_csv, command: str, resolved: dict, notes: Sequence[str] = ()) -> None:
    """``<csv stem>.meta`` next to the CSV (cli.py:219-232); backend = cuda."""
    lines = [f"version = {__version__}", f"command = {command}", "backend = cuda"]
    for key in sorted(resolved):
        lines.append(f"{key} = {resolved[key]}")
    for note in notes:
        lines.append(f"note = {note}")
    _write_lines(Path(out_csv).with_suffix(".meta"), lines)


__all__ = ["write_diagnostics_csv", "write_meta"]
