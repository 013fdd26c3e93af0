"""Seeded synthetic input generators shared by the oracle tests and the CUDA
path.  Holds shapes, value distributions and the bf16 storage format only —
none of the method's arithmetic."""
from . import trees, inputs  # noqa: F401
