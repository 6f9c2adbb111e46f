"""Record files: byte-identical to the reference writer (fixtures written by
linkatlas.records.write_records), crash-safe reading, npz sidecars."""

import numpy as np
import pytest

from oracle import links_oracle as O
from paper_2208_14567_b200 import records as R


def _bytes(arr) -> bytes:
    return np.asarray(arr, dtype=np.uint8).tobytes()


def test_ldjson_round_trip_is_byte_identical(golden, tmp_path):
    g = golden("dataset_golden.npz")
    for key, kind in (("curves_ldjson", "curve"), ("mechs_ldjson", "mechanism")):
        src = tmp_path / f"{kind}.ldjson"
        src.write_bytes(_bytes(g[key]))
        recs = list(R.RecordReader(src, kind))
        out = tmp_path / f"{kind}_out.ldjson"
        assert R.write_records(out, kind, recs) == len(recs)
        assert out.read_bytes() == src.read_bytes()
    # mechanisms survive record -> Mechanism -> record
    mrecs = list(R.read_records(tmp_path / "mechanism.ldjson", "mechanism"))
    for r in mrecs:
        assert R.mechanism_to_record(R.record_to_mechanism(r), r.id) == r


def test_bulk_curve_writer_matches_reference_bytes(golden, tmp_path):
    g = golden("dataset_golden.npz")
    k = g["kept"]
    out = tmp_path / "c.ldjson"
    R.write_curve_arrays(out, g["mech_ids"][k], g["joint_ids"][k], g["is_arc"][k], g["is_circle"][k], g["points"][k])
    assert out.read_bytes() == _bytes(g["curves_ldjson"])


def test_truncated_and_bad_files(tmp_path):
    p = tmp_path / "c.ldjson"
    recs = [R.CurveRecord(i, 2, False, True, [[0.0, 0.5], [1.0, 0.5]]) for i in range(3)]
    R.write_records(p, "curve", recs)
    data = p.read_bytes()
    p.write_bytes(data[:-7])  # tear the last line
    rd = R.RecordReader(p, "curve")
    got = list(rd)
    assert got == recs[:2] and rd.truncated
    with pytest.raises(R.FormatError):
        R.RecordReader(p, "mechanism")
    (tmp_path / "h.ldjson").write_text('{"format":"other","version":1,"kind":"curve"}\n')
    with pytest.raises(R.FormatError):
        R.RecordReader(tmp_path / "h.ldjson")
    (tmp_path / "v.ldjson").write_text('{"format":"linkatlas.records","version":2,"kind":"curve"}\n')
    with pytest.raises(R.FormatError):
        R.RecordReader(tmp_path / "v.ldjson")
    (tmp_path / "e.ldjson").write_text('{"format":"linkatlas.records"')
    with pytest.raises(R.FormatError):
        R.RecordReader(tmp_path / "e.ldjson")
    with pytest.raises(R.FormatError):
        R.write_records(tmp_path / "x.ldjson", "bogus", [])


def test_npz_sidecar_round_trip(golden, tmp_path):
    g = golden("dataset_golden.npz")
    recs = [R.CurveRecord(int(m), int(j), bool(a), bool(c), p.tolist())
            for m, j, a, c, p in zip(g["mech_ids"], g["joint_ids"], g["is_arc"], g["is_circle"], g["points"])]
    R.write_curves_npz(tmp_path / "c.npz", recs)
    z = np.load(tmp_path / "c.npz")
    assert z["mech_ids"].dtype == np.uint64 and z["points"].dtype == np.float64
    assert R.read_curves_npz(tmp_path / "c.npz") == recs


def test_oracle_keep_rule_pinned(golden):
    g = golden("dataset_golden.npz")
    got = [O.curation_keep(int(m), int(j), True, 0.5, 77) for m, j in zip(g["rule_mech"], g["rule_joint"])]
    assert got == list(g["rule_keep"])
    keep_rate, seed = g["curate"]
    kept = [O.curation_keep(int(m), int(j), bool(a or c), float(keep_rate), int(seed))
            for m, j, a, c in zip(g["mech_ids"], g["joint_ids"], g["is_arc"], g["is_circle"])]
    assert kept == list(g["kept"])


def test_atlas_save_matches_reference_bytes(golden, tmp_path):
    """Atlas.save writes the reference's files byte for byte; load round
    trips (host only: no resampling, no device)."""
    from paper_2208_14567_b200.atlas import Atlas
    from paper_2208_14567_b200.workloads import four_bar

    g = golden("atlas_golden.npz")
    pts = g["points"][:12]
    a = Atlas(pts, np.arange(12), np.full(12, 3), {i: four_bar() for i in range(12)}, seed=5)
    a.save(tmp_path)
    for name in ("meta.json", "curves.ldjson", "mechanisms.ldjson"):
        assert (tmp_path / name).read_bytes() == _bytes(g["save_" + name.replace(".", "_")]), name
    b = Atlas.load(tmp_path)
    assert np.array_equal(b.points, a.points) and np.array_equal(b.order, a.order) and b.seed == 5
    with pytest.raises(R.FormatError):
        Atlas.build([R.CurveRecord(99, 3, False, False, pts[0].tolist())], {})
