"""CPU-only checks of the drop-in boundary: the C-ABI library loads and exports
every symbol the header declares; host-side mirrors (config validation,
batch codec, streams) behave like the reference."""

import os
import re

import numpy as np
import pytest

from paper_2604_06596_b200 import _native
from paper_2604_06596_b200.batch import (BatchUpdate, read_batches_jsonl, write_batches_jsonl)
from paper_2604_06596_b200.errors import FileFormatError, ValidationError

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "dynlp_b200.h")


def header_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(dlp_\w+)\(", text, re.M)))


def test_library_exports_every_header_symbol():
    lib = _native.load(build_if_missing=True)
    syms = header_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    assert set(syms) == set(_native.SIGNATURES), set(syms) ^ set(_native.SIGNATURES)


def test_library_is_sm100a():
    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _native.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_engine_config_validation_mirrors_reference():
    from paper_2604_06596_b200.engine import EngineConfig

    for bad in (dict(delta=0), dict(max_iterations=0), dict(mode="bogus"), dict(tau="mean"),
                dict(tau=-1.0)):
        with pytest.raises(ValidationError):
            EngineConfig(**bad).validate()
    assert EngineConfig().delta == 1e-4


def test_batch_jsonl_round_trip_and_errors():
    b = BatchUpdate.from_records([(0, [], 0), (1, [(1, 0, 0.5)], None), (2, [(2, 1, 1.5), (0, 2, 2.0)], 1)],
                                 deletes=[], t=3)
    text = write_batches_jsonl([b])
    (c,) = read_batches_jsonl(text)
    for k in ("insert_ids", "insert_gt", "edge_owner", "edge_other", "edge_w", "deletes"):
        assert np.array_equal(getattr(b, k), getattr(c, k)), k
    assert c.t == 3
    with pytest.raises(FileFormatError):
        read_batches_jsonl('{"t": 0}\n')
    with pytest.raises(FileFormatError):
        read_batches_jsonl("{not json}\n")
    with pytest.raises(ValidationError):
        BatchUpdate.from_records([(0, [(5, 6, 1.0)], None)])


def test_jsonl_matches_reference_codec():
    from oracle import load_reference

    ref = load_reference()
    if ref is None:
        pytest.skip("reference not importable")
    from dynlp.graph import BatchUpdate as RB
    from dynlp.graph import write_batches_jsonl as ref_write

    recs = [(0, [], 0), (1, [(1, 0, 0.25)], None), (2, [(2, 1, 1.5), (2, 0, 2.0)], 1)]
    ours = write_batches_jsonl([BatchUpdate.from_records(recs, deletes=[], t=0)])
    theirs = ref_write([RB.from_records(recs, deletes=[], t=0)])
    assert ours == theirs


def test_stream_generator_rules():
    from paper_2604_06596_b200 import streams

    bl = streams.make_blobs(400, 6, 3, 0)
    e = streams.knn_graph_exact(bl.x, 5)
    gt = streams.stratified_seeds(bl.classes, 0.05, 0)
    s = streams.phased_stream(400, e, bl.classes, gt, 50, 0, 0.7, 0.02, 0.28, initial_gt=6)
    alive = set()
    n = 0
    for b in s.batches:
        d = set(int(x) for x in b.deletes)
        assert d <= alive
        alive -= d
        ids = b.insert_ids
        assert np.array_equal(ids, np.arange(n, n + len(ids)))
        own = ids[b.edge_owner]
        assert (own > b.edge_other).all()  # edge owned by its later endpoint
        ext = b.edge_other[b.edge_other < n]
        assert set(int(x) for x in ext) <= alive  # never to a dead vertex
        n += len(ids)
        alive |= set(int(x) for x in ids)
    assert n == 400
