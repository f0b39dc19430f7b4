"""The kernel mutation check's patch set (tools/kernel_mutation.py) still
applies to the product source: every mutant's product text is present, so a
refactor cannot silently turn a planted mistake into a no-op (CPU only)."""
import os
import shutil
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_every_mutant_patch_applies(tmp_path, monkeypatch):
    sys.path.insert(0, os.path.join(ROOT, "tools"))
    import kernel_mutation as KM
    monkeypatch.setattr(KM, "SRCDIR", str(tmp_path))
    for k in KM.MUTANTS:
        d = KM.patched_source(k)
        assert os.path.isdir(d)
        shutil.rmtree(d)
    assert len(KM.MUTANTS) >= 15
