"""The runtime drop-in patches every module binding the reference uses
(tensor.py:18 and cli.py:26 import the engine names directly).  Runs only
where the reference package is importable (the build container)."""

import os
import sys

import pytest

REF = "/root/reference/pkg/src"


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference package not present")
def test_install_patches_all_bindings():
    sys.path.insert(0, REF)
    try:
        import rubs
        import paper_1003_2022_b200 as rb
        from paper_1003_2022_b200 import shim
        orig = rubs.engine.filter_space_variant
        done = shim.install(rubs)
        assert rubs.engine.filter_space_variant is rb.filter_space_variant
        assert rubs.tensor.filter_space_variant is rb.filter_space_variant
        assert rubs.tensor.filter_space_invariant is rb.filter_space_invariant
        assert rubs.filter_space_variant is rb.filter_space_variant
        assert "rubs.cli.filter_space_invariant" in done
        shim.uninstall(rubs)
        assert rubs.engine.filter_space_variant is orig
    finally:
        sys.path.remove(REF)


@pytest.mark.skipif(not os.path.isdir(REF), reason="reference package not present")
def test_reference_scale_field_is_accepted():
    # callers of the shimmed reference pass the reference's own ScaleField
    # (reference tests/test_engine.py:84); the boundary unwraps it by duck type
    import numpy as np
    sys.path.insert(0, REF)
    try:
        import rubs
        from paper_1003_2022_b200 import engine
        sf = rubs.ScaleField.uniform((4, 5), [1.0, 2.0, 3.0, 4.0])
        fld, uniform = engine._host_field(sf, (4, 5))
        assert not uniform and fld.shape == (4, 5, 4) and np.all(fld[..., 2] == 3.0)
        assert engine._unwrap_field(sf) is sf.scales
        arr = np.ones((4, 5, 4))
        assert engine._unwrap_field(arr) is arr
    finally:
        sys.path.remove(REF)
