"""Wire and disk formats shared with the reference, so runs on
the B200 can be compared with the reference's own files line for line:

* `rbm-params-v1` JSON checkpoints: `rbm.save_parameters` / `rbm.load_parameters`
  (ref rbm.py:104-127);
* the training-log CSV and its `<csv>.meta.json` sidecar (ref experiments.py:
  222-248 `_format_value`, `write_csv`, `write_sidecar`; 611-652 `_LOG_COLUMNS`,
  `_record_row`, `cmd_vmc_train`): one row per logged record, prefixed by the
  sampling format's name, floats as `%.14e`;
* the chain-major uint8 sample matrix (ref sampler.py:142-167) is what
  `ChainEnsemble.collect` returns; `save_samples` / `load_samples` store it as
  `.npy` (rows in the reference's order).
"""
from __future__ import annotations

import json
import math
import os

import numpy as np

VERSION = "0.1.0"  # the reference package version the sidecar format follows

LOG_COLUMNS = ("step", "energy", "mc_error", "acceptance", "sigma_hat", "bound_pinsker", "bound_theorem3", "kappa")


def format_value(value) -> str:
    """CSV cell text (ref experiments.py:222-229)."""
    if isinstance(value, bool):
        return "true" if value else "false"
    if isinstance(value, (int, np.integer)):
        return str(int(value))
    if isinstance(value, (float, np.floating)):
        return f"{float(value):.14e}"
    return str(value)


def write_csv(path, header, rows):
    with open(path, "w") as handle:
        handle.write(",".join(header) + "\n")
        for row in rows:
            handle.write(",".join(format_value(v) for v in row) + "\n")
    return path


def write_sidecar(csv_path, config: dict, extra: dict | None = None):
    """`<csv>.meta.json` with the run configuration (ref experiments.py:240-248)."""
    payload = {"config": config, "version": VERSION}
    if extra:
        payload.update(extra)
    sidecar = f"{csv_path}.meta.json"
    with open(sidecar, "w") as handle:
        json.dump(payload, handle, sort_keys=True, indent=2)
        handle.write("\n")
    return sidecar


def record_row(prefix, record) -> tuple:
    """One log row (ref experiments.py:617-624)."""
    row = list(prefix)
    for key in LOG_COLUMNS:
        row.append(record[key])
    row.append(record.get("rel_error", float("nan")))
    if "sampling_seconds" in record:
        row.extend((record["sampling_seconds"], record["update_seconds"]))
    return tuple(row)


def write_training_log(out_dir, runs: dict, config: dict, reference_energy=None, timings: bool = False):
    """training_log.csv + sidecar for {format name: vmc.TrainResult} (the layout
    `cmd_vmc_train` writes, ref experiments.py:627-652); returns the CSV path."""
    os.makedirs(out_dir, exist_ok=True)
    rows = [record_row((name,), rec) for name, result in runs.items() for rec in result.records]
    header = ["format", *LOG_COLUMNS, "rel_error"]
    if timings:
        header.extend(("sampling_seconds", "update_seconds"))
    path = os.path.join(out_dir, "training_log.csv")
    write_csv(path, header, rows)
    write_sidecar(path, config, {"reference_energy": reference_energy})
    return path


def read_training_log(path) -> list[dict]:
    """Parse a training log written by either implementation."""
    with open(path) as handle:
        header = handle.readline().strip().split(",")
        out = []
        for line in handle:
            cells = line.rstrip("\n").split(",")
            rec = {}
            for key, cell in zip(header, cells):
                if key == "format":
                    rec[key] = cell
                elif key == "step":
                    rec[key] = int(cell)
                else:
                    rec[key] = float(cell) if cell not in ("true", "false") else cell == "true"
            out.append(rec)
    return out


def save_samples(path, samples) -> str:
    """uint8 (S, N) chain-major sample matrix as .npy."""
    arr = np.ascontiguousarray(np.asarray(samples, dtype=np.uint8))
    if arr.ndim != 2:
        raise ValueError("sample matrix must be (S, N)")
    np.save(path, arr, allow_pickle=False)
    return path if str(path).endswith(".npy") else f"{path}.npy"


def load_samples(path) -> np.ndarray:
    arr = np.load(path, allow_pickle=False)
    if arr.dtype != np.uint8 or arr.ndim != 2:
        raise ValueError("not a uint8 (S, N) sample matrix")
    return arr


def same_log(a, b, rtol: float = 0.0) -> bool:
    """Row-by-row equality of two parsed logs (floats within rtol; NaN == NaN)."""
    if len(a) != len(b):
        return False
    for ra, rb in zip(a, b):
        if ra.keys() != rb.keys():
            return False
        for k in ra:
            x, y = ra[k], rb[k]
            if isinstance(x, float):
                if not (math.isnan(x) and math.isnan(y)) and abs(x - y) > rtol * max(1.0, abs(x)):
                    return False
            elif x != y:
                return False
    return True
