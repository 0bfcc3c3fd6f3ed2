"""Dataset readers vs the reference's own readings of a dataset written by
the reference's generate_dataset (tests/golden/dataset_small)."""

import os
import shutil

import numpy as np
import pytest

from conftest import GOLDEN, load_golden


def _m():
    from paper_2301_05262_b200 import dataset
    return dataset.load_manifest(os.path.join(GOLDEN, "dataset_small"))


def test_numpy_loaders_match_reference():
    from paper_2301_05262_b200 import dataset
    ref = load_golden("dataset_small_ref")
    m = _m()
    assert len(m.frames) == 3 and m.resolution == (32, 48) and m.sizes == (0.0, 2.0)
    fs = dataset.load_feature_stack(m, 1, 1, 2.0)
    np.testing.assert_array_equal(fs.data, ref["stack_1_1_s2"])
    np.testing.assert_array_equal(fs.coverage, ref["coverage_1"])
    g = dataset.load_gbuffer(m, 2)
    np.testing.assert_array_equal(g.position, ref["gb_position_2"])
    np.testing.assert_array_equal(g.z_f, ref["gb_z_f_2"])
    np.testing.assert_array_equal(dataset.load_target(m, 2, 2.0), ref["target_2_s2"])
    with pytest.raises(dataset.DatasetError):
        dataset.load_target(m, 0, 3.0)


def test_manifest_integrity_errors(tmp_path):
    from paper_2301_05262_b200 import dataset
    src = os.path.join(GOLDEN, "dataset_small")
    d = tmp_path / "ds"
    shutil.copytree(src, d)
    dataset.load_manifest(d)
    p = d / "0001" / "features_1.pfm"
    raw = p.read_bytes()
    p.write_bytes(raw[:-4])                                   # truncated payload
    with pytest.raises(dataset.DatasetError):
        dataset.load_manifest(d)
    p.write_bytes(b"XXXX" + raw[4:])                          # bad magic
    with pytest.raises(dataset.DatasetError):
        dataset.load_manifest(d)
    p.unlink()                                                # missing file
    with pytest.raises(dataset.DatasetError):
        dataset.load_manifest(d)
    with pytest.raises(dataset.DatasetError):
        dataset.load_manifest(tmp_path / "nowhere")
