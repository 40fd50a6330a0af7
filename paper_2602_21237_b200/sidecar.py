"""GPU metrics of a reference sweep in a sidecar CSV keyed by label.

The reference's sweep CSV has a fixed column tuple (`relab/bench.py:53-69`)
and `read_sweep_csv` rejects any other columns (`bench.py:393-394`), so the
B200 extras cannot go into it. ``sweep_with_sidecar`` runs the reference's own
harness cell by cell (``run_experiment`` → ``report_to_row``, as
`relab.bench.sweep` does, `bench.py:343-363`; with ``patch.install()`` in
effect the tensor path runs on the B200), writes the byte-compatible sweep CSV
with the reference's writer, and beside it one row per cell keyed by the
cell's label: device, GPUs, throughput, the cell's algorithmic bytes
 and their fraction of the measured HBM bandwidth.

The caller provides the reference package (``relab``): this module only
imports it when called.
"""

from __future__ import annotations

import csv
import json
from pathlib import Path
from typing import Iterable, Optional, TextIO

SIDECAR_COLUMNS = (
    "label",
    "operation",
    "n_left",
    "n_right",
    "path_taken",
    "gpus",
    "device",
    "p50_s",
    "mrows_per_s",
    "output_rows",
    "alg_bytes",
    "achieved_gbs",
    "hbm_frac",
    "peak_gbs",
)


def measured_peak_gbs() -> float:
    """The measured HBM copy bandwidth of this pool (MEASURED_PEAKS.json),
    else the profiling guide's B200 fallback (6.65 TB/s)."""
    p = Path(__file__).resolve().parent.parent / "MEASURED_PEAKS.json"
    try:
        return float(json.loads(p.read_text())["hbm_gbs"])
    except (OSError, ValueError, KeyError):
        return 6650.0


def cell_label(config) -> str:
    if config.label:
        return config.label
    g = config.gen_left
    return f"{config.operation.value}-n{g.n}-d{g.key_domain}-{config.policy.value}-b{config.budget.bytes}"


def alg_bytes(config, output_rows: int) -> int:
    """a join reads both sides' key + payload once and writes
    key + both payloads per output row; a sort reads n rows and writes the
    sorted rows plus a 4-byte permutation."""
    gl = config.gen_left
    wl = 8 + gl.payload_width
    if config.operation.value == "join":
        gr = config.gen_right
        wr = 8 + gr.payload_width
        return gl.n * wl + gr.n * wr + output_rows * (wl + gr.payload_width)
    return gl.n * wl + output_rows * (wl + 4)


def sidecar_row(config, report, device: str, gpus: int, peak_gbs: float) -> dict:
    p50 = report.latency.p50
    rows_in = config.gen_left.n + (config.gen_right.n if config.gen_right else 0)
    b = alg_bytes(config, report.output_rows)
    achieved = b / p50 / 1e9 if p50 > 0 else 0.0
    return {
        "label": cell_label(config),
        "operation": config.operation.value,
        "n_left": config.gen_left.n,
        "n_right": config.gen_right.n if config.gen_right else 0,
        "path_taken": report.path_taken.path.value,
        "gpus": gpus,
        "device": device,
        "p50_s": f"{p50:.6g}",
        "mrows_per_s": f"{rows_in / p50 / 1e6:.6g}" if p50 > 0 else "0",
        "output_rows": report.output_rows,
        "alg_bytes": b,
        "achieved_gbs": f"{achieved:.6g}",
        "hbm_frac": f"{achieved / peak_gbs:.6g}",
        "peak_gbs": f"{peak_gbs:.6g}",
    }


def write_sidecar(rows: Iterable[dict], path) -> None:
    with open(path, "w", newline="") as f:
        w = csv.DictWriter(f, fieldnames=SIDECAR_COLUMNS)
        w.writeheader()
        for r in rows:
            w.writerow(r)


def read_sidecar(path) -> list:
    with open(path, newline="") as f:
        reader = csv.DictReader(f)
        if tuple(reader.fieldnames or ()) != SIDECAR_COLUMNS:
            raise ValueError(f"{path}: unexpected sidecar columns")
        return list(reader)


def sweep_with_sidecar(configs, csv_path, sidecar_path=None, progress: Optional[TextIO] = None):
    """Run a reference sweep; write its CSV (the reference's writer, columns
    unchanged) and the GPU sidecar (``<csv>.gpu.csv`` by default). Failed
    cells become the reference's error rows and get no sidecar row."""
    import relab.bench as rb
    from relab.errors import RelabError

    try:
        import torch

        dev = torch.cuda.get_device_name(0) if torch.cuda.is_available() else "cpu"
        gpus = 1 if torch.cuda.is_available() else 0
    except ImportError:  # pragma: no cover
        dev, gpus = "cpu", 0
    peak = measured_peak_gbs()
    rows, side = [], []
    for config in configs:
        try:
            report = rb.run_experiment(config)
            row = rb.report_to_row(report)
            side.append(sidecar_row(config, report, dev, gpus, peak))
        except (RelabError, OSError) as exc:
            row = rb.error_row(config, exc)
        rows.append(row)
        if progress is not None:
            print(f"{row.operation} n={row.n_left} -> {row.path_taken} p50={row.p50_s}s", file=progress, flush=True)
    rb.write_sweep_csv(rows, csv_path)
    sidecar_path = sidecar_path or str(csv_path) + ".gpu.csv"
    write_sidecar(side, sidecar_path)
    return rows, side
