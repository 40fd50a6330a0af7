"""The drop-in installs into a live relab (only where the reference is
importable, i.e. the build container; the GPU box has no /root/reference)."""

import sys
from pathlib import Path

import pytest

REF = Path("/root/reference/pkg/src")


@pytest.fixture
def relab_mod():
    if not REF.exists():
        pytest.skip("reference package not present on this machine")
    sys.path.insert(0, str(REF))
    sys.dont_write_bytecode = True
    import relab
    import relab.bench
    import relab.tensorpath

    yield relab
    sys.path.remove(str(REF))


def test_install_rebinds_every_name_the_reference_binds(relab_mod):
    from paper_2602_21237_b200 import patch, tensor_path

    originals = (relab_mod.bench.to_tensor, relab_mod.bench.tensor_join, relab_mod.bench.tensor_sort)
    replaced = patch.install()
    try:
        # bench.py:49 binds by name; __init__.py re-exports
        assert relab_mod.bench.to_tensor is tensor_path.to_tensor
        assert relab_mod.bench.tensor_join is tensor_path.tensor_join
        assert relab_mod.bench.tensor_sort is tensor_path.tensor_sort
        assert relab_mod.to_tensor is tensor_path.to_tensor
        assert relab_mod.tensorpath.key_axis_align is tensor_path.key_axis_align
        assert ("relab.bench", "tensor_join") in replaced
        # the operators now raise / build relab's own classes
        assert tensor_path.TYPES["OutputTooLarge"] is relab_mod.errors.OutputTooLarge
        assert tensor_path.TYPES["SpillStats"] is relab_mod.spill.SpillStats
    finally:
        patch.uninstall()
    assert (relab_mod.bench.to_tensor, relab_mod.bench.tensor_join, relab_mod.bench.tensor_sort) == originals


def test_relation_class_follows_schema_module(relab_mod):
    from paper_2602_21237_b200 import records, tensor_path

    class Holder:
        schema = relab_mod.Schema((("key", relab_mod.Int64()),))

    assert tensor_path._relation_class_of(Holder) is relab_mod.Relation

    class Mine:
        schema = records.Schema((("key", records.Int64()),))

    assert tensor_path._relation_class_of(Mine) is records.Relation


def test_reference_int64_type_is_recognised(relab_mod):
    from paper_2602_21237_b200.records import is_int64

    assert is_int64(relab_mod.Int64()) and not is_int64(relab_mod.Bytes(8))
