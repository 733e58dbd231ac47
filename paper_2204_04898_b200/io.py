"""Columnar ingest ("A Parquet file is a binary
file containing the values for each column/attribute ... the ingestion of a
Parquet file ... is faster because the data is already organized in columns").

read_parquet reads the case / activity / timestamp columns (and optional extra
attribute columns) of a Parquet file with pyarrow, dictionary-encodes string
columns in first-occurrence order, converts timestamps to int64
milliseconds since the epoch (R3), and creates a pm4g log on the current CUDA
device (host buffers are pinned and copied inside pm4g_log_create).  Parsing
is host work done by the pyarrow library; every computation on the log runs in
libpm4g.
"""
from __future__ import annotations

import numpy as np
import torch

from . import pm4g


def _codes(col):
    """(codes int64[n], dictionary list) in first-occurrence order; null -> error."""
    import pyarrow as pa
    import pyarrow.compute as pc
    if col.null_count:
        raise ValueError("null in a mandatory column (S:123)")
    if pa.types.is_integer(col.type):
        v = col.to_numpy(zero_copy_only=False).astype(np.int64)
        if v.size and v.min() < 0:
            raise ValueError("negative integer codes")
        return v, None
    enc = pc.dictionary_encode(col).combine_chunks()
    return enc.indices.to_numpy(zero_copy_only=False).astype(np.int64), enc.dictionary.to_pylist()


def _millis(col):
    import pyarrow as pa
    import pyarrow.compute as pc
    if col.null_count:
        raise ValueError("null timestamp (S:123)")
    if pa.types.is_timestamp(col.type):
        return pc.cast(col, pa.timestamp("ms")).cast(pa.int64()).to_numpy(zero_copy_only=False).astype(np.int64)
    if pa.types.is_integer(col.type):
        return col.to_numpy(zero_copy_only=False).astype(np.int64)   # raw epoch milliseconds
    raise ValueError(f"timestamp column of type {col.type}")


def read_parquet(path: str, case: str = "case:concept:name", activity: str = "concept:name",
                 timestamp: str = "time:timestamp", extra: tuple = (), borrow: bool = False):
    """Returns (log, case_dictionary, activity_dictionary, extra_dictionaries).

    Dictionaries are None for integer-coded columns.  ``extra``: names of extra
    attribute columns (strings -> u32 codes, integers -> i64, floats -> f64;
    nulls allowed)."""
    import pyarrow as pa
    import pyarrow.parquet as pq
    t = pq.read_table(path, columns=[case, activity, timestamp, *extra])
    c, cdict = _codes(t.column(case))
    a, adict = _codes(t.column(activity))
    ts = _millis(t.column(timestamp))
    n_cases = len(cdict) if cdict is not None else (int(c.max()) + 1 if c.size else 1)
    A = len(adict) if adict is not None else (int(a.max()) + 1 if a.size else 1)
    ab = pm4g.act_bytes_for(max(A, 1))
    adt = {1: torch.uint8, 2: torch.int16, 4: torch.int32}[ab]
    cols = [torch.from_numpy(c.astype(np.uint32).view(np.int32)).view(torch.uint32),
            torch.from_numpy(a.astype({1: np.uint8, 2: np.int16, 4: np.int32}[ab])).view(adt),
            torch.from_numpy(ts)]
    extras, edicts = [], []
    for name in extra:
        col = t.column(name)
        valid = None
        if col.null_count:
            valid = torch.from_numpy(col.is_valid().to_numpy(zero_copy_only=False).astype(np.uint8))
        if pa.types.is_string(col.type) or pa.types.is_large_string(col.type) or pa.types.is_dictionary(col.type):
            import pyarrow.compute as pc
            enc = pc.dictionary_encode(col).combine_chunks()
            v = enc.indices.fill_null(0).to_numpy(zero_copy_only=False).astype(np.uint32)
            extras.append(pm4g.Extra(kind=pm4g.PM4G_KIND_CODES, data=torch.from_numpy(v.view(np.int32)).view(torch.uint32),
                                     valid=valid, dict_size=len(enc.dictionary)))
            edicts.append(enc.dictionary.to_pylist())
        elif pa.types.is_integer(col.type):
            v = col.fill_null(0).to_numpy(zero_copy_only=False).astype(np.int64)
            extras.append(pm4g.Extra(kind=pm4g.PM4G_KIND_I64, data=torch.from_numpy(v), valid=valid))
            edicts.append(None)
        else:
            v = col.fill_null(0.0).to_numpy(zero_copy_only=False).astype(np.float64)
            extras.append(pm4g.Extra(kind=pm4g.PM4G_KIND_F64, data=torch.from_numpy(v), valid=valid))
            edicts.append(None)
    dev = torch.device("cuda", torch.cuda.current_device())
    cols = [x.pin_memory().to(dev, non_blocking=True) for x in cols]
    extras = [pm4g.Extra(kind=e.kind, data=e.data.pin_memory().to(dev, non_blocking=True),
                         valid=None if e.valid is None else e.valid.pin_memory().to(dev, non_blocking=True),
                         dict_size=e.dict_size)
              for e in extras]
    log = pm4g.pm4g_log_create(cols[0], cols[1], cols[2], A, n_case_codes=max(n_cases, 1),
                               extra=extras or None, borrow=borrow)
    return log, cdict, adict, edicts
