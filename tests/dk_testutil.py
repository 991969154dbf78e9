"""Shared constants for the test modules (imported as a top-level module)."""

import os

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(REPO, "tests", "golden", "reference_golden.npz")
FAMILIES = ("gaussian", "exponential", "laplacian")
