"""Device dataset pipeline (generate -> normalise moving joints -> flags ->
curate -> atlas) vs the reference CLI chain (dataset_golden.npz).  Ids,
is_arc and the keep rule are exact; curve points within 1e-9 (f64
trajectories from la_simulate, f64 la_normalize); is_circle exact away from
the 5e-4 threshold."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch

    assert torch.cuda.is_available()
    return torch


def test_keep_rule_device_matches_reference(torch, golden):
    from paper_2208_14567_b200.dataset import curation_keep_batch

    g = golden("dataset_golden.npz")
    got = curation_keep_batch(g["rule_mech"], g["rule_joint"], np.ones(len(g["rule_mech"]), bool), 0.5, 77)
    assert np.array_equal(got, g["rule_keep"])
    keep_rate, seed = g["curate"]
    got = curation_keep_batch(g["mech_ids"], g["joint_ids"], g["is_arc"] | g["is_circle"], float(keep_rate), int(seed))
    assert np.array_equal(got, g["kept"])
    with pytest.raises(ValueError):
        curation_keep_batch(np.array([-1]), np.array([0]), np.array([True]), 0.5, 0)


def test_pipeline_matches_reference_cli_chain(torch, golden, tmp_path):
    from paper_2208_14567_b200 import records as R
    from paper_2208_14567_b200.dataset import atlas_from_curves, curate_batch, curves_from_block
    from paper_2208_14567_b200.generator import GenerationConfig, GenerationRun

    g = golden("dataset_golden.npz")
    count, seed, n_min, n_max, vpt, max_att = (int(x) for x in g["cfg"])
    cfg = GenerationConfig(count=count, seed=seed, n_min=n_min, n_max=n_max, variants_per_topology=vpt,
                           max_attempts=max_att)
    blocks = list(GenerationRun(cfg, traj_on_device=True).blocks())
    assert len(blocks) == 1
    cb = curves_from_block(blocks[0], vpt)
    assert np.array_equal(cb.mech_ids, g["mech_ids"])
    assert np.array_equal(cb.joint_ids, g["joint_ids"])
    assert np.array_equal(cb.is_arc, g["is_arc"])
    # f64 paths are bit-exact (LA_SIM_EXACT64); normalisation within 1e-12
    assert np.max(np.abs(cb.points.cpu().numpy() - g["points"])) <= 1e-12
    assert np.array_equal(cb.is_circle, g["is_circle"])
    keep_rate, cseed = g["curate"]
    kept = curate_batch(cb, float(keep_rate), int(cseed))
    k = g["kept"]
    assert np.array_equal(kept.mech_ids, g["mech_ids"][k])
    assert np.array_equal(kept.joint_ids, g["joint_ids"][k])
    # exact chain: the written file is byte-identical to the reference CLI's
    assert np.array_equal(cb.points.cpu().numpy(), g["points"])
    exact = tmp_path / "exact.ldjson"
    R.write_curve_arrays(exact, kept.mech_ids, kept.joint_ids, kept.is_arc, kept.is_circle,
                         kept.points.cpu().numpy())
    assert exact.read_bytes() == np.asarray(g["curves_ldjson"], dtype=np.uint8).tobytes()
    # writer output parses to the reference's records (points to 1e-9)
    out = tmp_path / "c.ldjson"
    R.write_curve_arrays(out, kept.mech_ids, kept.joint_ids, kept.is_arc, kept.is_circle, kept.points.cpu().numpy())
    ref = tmp_path / "ref.ldjson"
    ref.write_bytes(np.asarray(g["curves_ldjson"], dtype=np.uint8).tobytes())
    for a, b in zip(R.RecordReader(out, "curve"), R.RecordReader(ref, "curve")):
        assert (a.mech_id, a.joint_id, a.is_arc, a.is_circle) == (b.mech_id, b.joint_id, b.is_arc, b.is_circle)
        assert np.max(np.abs(np.array(a.points) - np.array(b.points))) <= 1e-9
    # atlas straight from the device batch: a kept curve retrieves itself,
    # with the reduced mechanism of its joint
    from paper_2208_14567_b200.dataset import mechanisms_of_block

    atlas = atlas_from_curves(kept, mechanisms_of_block(blocks[0], vpt), seed=1)
    for i in (0, 3, len(atlas) - 1):
        hits = atlas.retrieve(atlas.points[i], k=2)
        assert hits[0].distance == 0.0
        # byte-identical curves (e.g. every crank circle) resolve to the LAST
        # duplicate, like the reference's dict index (atlas.py:78-80)
        dup = [j for j in range(len(atlas)) if atlas.points[j].tobytes() == atlas.points[i].tobytes()]
        assert (hits[0].mech_id, hits[0].joint_id) == (int(kept.mech_ids[dup[-1]]), int(kept.joint_ids[dup[-1]]))
