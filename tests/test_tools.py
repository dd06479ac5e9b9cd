"""The A/B tooling stays in step with the product sources: every patch of
tools/mk_variant.py still finds its target (a variant whose target moved
would abort its build on the GPU box)."""

import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT / "tools"))

import mk_variant  # noqa: E402


@pytest.mark.parametrize("name", sorted(mk_variant.VARIANTS))
def test_variant_patch_targets_exist(name):
    for fname, old, _new in mk_variant.VARIANTS[name]:
        assert old in (mk_variant.CSRC / fname).read_text(), (name, fname, old[:60])
