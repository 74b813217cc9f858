"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py (input plumbing only)."""
from .scenes import Scene, by_name, tiny, street, city, random_instance, dense_box, line_scene, line_indices  # noqa: F401
