"""Seeded synthetic inputs shared by the oracle tests, the CUDA parity tests and bench.py.

This module only *generates data* (cell-like frames of cosine embeddings with ground truth).
It contains none of the method's arithmetic (no window, no shift, no merge, no assignment),
so the oracle and the CUDA path share nothing through it but their inputs.
"""
from .frames import CONFIGS, Frame, make_blobs, make_frame, make_stack, frame_pool  # noqa: F401
