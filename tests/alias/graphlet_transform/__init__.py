"""Test-only alias: the reference package name ``graphlet_transform``
(proj/python/graphlet_transform/__init__.py) bound to the drop-in package, so
the reference's own Python suite (proj/tests/python/test_smoke.py) runs
against it unchanged (tests/test_reference_suites.py)."""
from paper_2007_11111_b200 import *  # noqa: F401,F403
from paper_2007_11111_b200 import __all__  # noqa: F401
