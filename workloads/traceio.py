"""Trace file ingestion — inputs only.

CSV with header ``input_tokens,output_tokens[,arrival_time][,phase]``.
* input tokens above ``max_input_tokens`` are clamped ("maximum of 8K input
  tokens"); a zero-length record is rejected with its line number.
* without ``arrival_time`` the arrivals are a seeded unit-rate Poisson process
  (as in tracegen); with it, ``s_unit`` = arrival_time, i.e. the recorded times
  are replayed exactly at QPS-per-GPU ``1/N`` (the kernels scale s_unit by
  1/(q·N)) and proportionally faster/slower at other QPS points.
"""
from __future__ import annotations

import csv

import numpy as np


class TraceFormatError(ValueError):
    pass


def load_trace_csv(path: str, max_input_tokens: int = 8192, seed: int = 0) -> dict:
    ins, outs, arr, ph = [], [], [], []
    with open(path, newline="") as f:
        rd = csv.reader(f)
        header = [h.strip() for h in next(rd)]
        if header[:2] != ["input_tokens", "output_tokens"]:
            raise TraceFormatError("header must start with input_tokens,output_tokens")
        has_arr = "arrival_time" in header
        has_ph = "phase" in header
        ia = header.index("arrival_time") if has_arr else -1
        ip = header.index("phase") if has_ph else -1
        for ln, row in enumerate(rd, start=2):
            if not row or all(not c.strip() for c in row):
                continue
            try:
                i, o = int(row[0]), int(row[1])
                a = float(row[ia]) if has_arr else None
                p = int(row[ip]) if has_ph else 0
            except (ValueError, IndexError) as e:
                raise TraceFormatError(f"line {ln}: malformed row {row!r}") from e
            if i < 1 or o < 1:
                raise TraceFormatError(f"line {ln}: zero-length record")
            if p not in (0, 1):
                raise TraceFormatError(f"line {ln}: phase must be 0 or 1")
            ins.append(min(i, max_input_tokens))
            outs.append(o)
            arr.append(a)
            ph.append(p)
    R = len(ins)
    if has_arr:
        s_unit = np.asarray(arr, dtype=np.float64)
        if R and (np.any(s_unit < 0) or np.any(np.diff(s_unit) < 0)):
            raise TraceFormatError("arrival_time must be non-negative and sorted")
    else:
        g = np.random.Generator(np.random.PCG64(np.random.SeedSequence([int(seed), 9, 1])))
        s_unit = np.cumsum(g.standard_exponential(size=R)).astype(np.float64)
    return {"s_unit": np.ascontiguousarray(s_unit), "in_tok": np.asarray(ins, np.int32),
            "out_tok": np.asarray(outs, np.int32), "phase": np.asarray(ph, np.uint8),
            "family": "file", "seed": int(seed)}


def save_trace_csv(path: str, trace: dict, with_arrivals: bool = True) -> None:
    with open(path, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["input_tokens", "output_tokens"] + (["arrival_time"] if with_arrivals else []) +
                   ["phase"])
        for k in range(trace["s_unit"].size):
            row = [int(trace["in_tok"][k]), int(trace["out_tok"][k])]
            if with_arrivals:
                row.append(repr(float(trace["s_unit"][k])))
            row.append(int(trace["phase"][k]))
            w.writerow(row)
