"""Matrix Market ingest: read_matrix_market + from_coo
(io.hpp:50-121, tensor.hpp:118). Fixtures and the reference's answers are in
tests/golden/mm (made by tests/golden/make_mm_goldens.py through the
unmodified reference). CPU: the oracle shim still reproduces them. GPU: the
device parser returns the same canonical COO (int arrays exact, values the
reference's f64 narrowed to fp32) or the same error kind and message."""
import json
import os

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
MM = os.path.join(HERE, "golden", "mm")
EXPECTED = json.load(open(os.path.join(MM, "expected.json")))
CASES = sorted(EXPECTED)


def _path(key):
    return os.path.join(MM, key.split(":")[0] + ".mtx")


def _summ(key):
    return key.endswith(":1")


@pytest.mark.parametrize("key", CASES)
def test_reference_reader_matches_goldens(ref, key):
    import oracle
    want = EXPECTED[key]
    path = _path(key)
    if "error" in want:
        with pytest.raises(oracle.OracleError) as ei:
            ref.read_mm(path, _summ(key))
        assert ei.value.kind == want["error"]
        assert str(ei.value)[len(ei.value.kind) + 2:] == want["message"].replace("{path}", path)
        return
    coo = ref.read_mm(path, _summ(key))
    r, c, v = coo.arrays()
    assert list(coo.shape) == want["shape"]
    assert r.tolist() == want["row"] and c.tolist() == want["col"]
    assert [float(x).hex() for x in v] == want["val"]


@pytest.mark.gpu
@pytest.mark.parametrize("key", CASES)
def test_device_reader_matches_reference(ctx, key):
    import paper_2403_05802_b200 as sfg
    want = EXPECTED[key]
    path = _path(key)
    if "error" in want:
        with pytest.raises(sfg.SfgError) as ei:
            ctx.read_matrix_market(path, sum_duplicates=_summ(key))
        assert ei.value.kind == want["error"], (key, ei.value.kind, str(ei.value))
        assert want["message"].replace("{path}", path) in str(ei.value), (key, str(ei.value))
        return
    t = ctx.read_matrix_market(path, sum_duplicates=_summ(key))
    assert list(t.shape) == want["shape"]
    r, c, v = t.coo_arrays()
    assert r.tolist() == want["row"] and c.tolist() == want["col"], key
    # (summed duplicates are added from their fp32 narrowings on the device;
    # the fixture's summands are exact in fp32, so the sums agree bit for bit)
    ref_v = np.array([float.fromhex(x) for x in want["val"]], np.float64).astype(np.float32)
    np.testing.assert_array_equal(v.view(np.uint32), ref_v.view(np.uint32), err_msg=key)


@pytest.mark.gpu
def test_device_reader_missing_file(ctx, tmp_path):
    import paper_2403_05802_b200 as sfg
    with pytest.raises(sfg.SfgError) as ei:
        ctx.read_matrix_market(str(tmp_path / "nope.mtx"))
    assert ei.value.kind == "Io"
