"""Input generators and trace ingestion (CPU): determinism, stream independence,
family shapes."""
import numpy as np
import pytest

from workloads import make_trace
from workloads.traceio import TraceFormatError, load_trace_csv, save_trace_csv


def test_generator_deterministic_and_streams_independent():
    a = make_trace("lb", 5, 1000)
    b = make_trace("lb", 5, 1000)
    for k in ("s_unit", "in_tok", "out_tok", "phase"):
        assert a[k].tobytes() == b[k].tobytes()
    c = make_trace("lb", 6, 1000)
    assert not np.array_equal(a["s_unit"], c["s_unit"])
    # a seed change alters arrival gaps but not the phase structure
    p1, p2 = make_trace("phase", 1, 2000), make_trace("phase", 2, 2000)
    assert np.array_equal(p1["in_tok"], p2["in_tok"]) and np.array_equal(p1["phase"], p2["phase"])


def test_family_shapes():
    lb = make_trace("lb", 0, 20000)
    assert lb["in_tok"].min() >= 512 and lb["in_tok"].max() <= 8192
    assert lb["out_tok"].min() >= 128 and lb["out_tok"].max() <= 256
    gaps = np.diff(np.concatenate([[0.0], lb["s_unit"]]))
    assert gaps.mean() == pytest.approx(1.0, rel=0.03) and gaps.std() == pytest.approx(1.0, rel=0.05)
    bu = make_trace("lb_bursty", 0, 20000)
    g2 = np.diff(np.concatenate([[0.0], bu["s_unit"]]))
    assert g2.mean() == pytest.approx(1.0, rel=0.06) and g2.std() / g2.mean() == pytest.approx(2.0, rel=0.1)
    ph = make_trace("phase", 0, 2000)
    assert (ph["in_tok"][:1000] == 8192).all() and (ph["out_tok"][:1000] == 128).all()
    assert (ph["in_tok"][1000:] == 500).all() and (ph["out_tok"][1000:] == 500).all()
    assert ph["phase"][:1000].sum() == 0 and ph["phase"][1000:].sum() == 1000
    assert int(ph["in_tok"].sum()) == 8192 * 1000 + 500 * 1000
    assert np.all(np.diff(lb["s_unit"]) > 0)


def test_trace_csv_roundtrip_and_clamp(tmp_path):
    tr = make_trace("lb", 3, 50)
    p = tmp_path / "t.csv"
    save_trace_csv(str(p), tr)
    back = load_trace_csv(str(p))
    for k in ("s_unit", "in_tok", "out_tok", "phase"):
        assert np.array_equal(back[k], tr[k]), k
    q = tmp_path / "c.csv"
    q.write_text("input_tokens,output_tokens\n4096,128\n16000,128\n7,1\n")
    c = load_trace_csv(str(q))
    assert list(c["in_tok"]) == [4096, 8192, 7]                                  # S:147 clamp
    assert list(c["out_tok"]) == [128, 128, 1] and c["s_unit"].size == 3
    assert np.all(np.diff(c["s_unit"]) > 0)


def test_trace_csv_errors(tmp_path):
    q = tmp_path / "bad.csv"
    q.write_text("input_tokens,output_tokens\n100,5\n0,5\n")
    with pytest.raises(TraceFormatError, match="line 3"):
        load_trace_csv(str(q))
    q.write_text("input_tokens,output_tokens\n100,x\n")
    with pytest.raises(TraceFormatError, match="line 2"):
        load_trace_csv(str(q))
