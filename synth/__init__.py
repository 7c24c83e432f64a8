"""Seeded synthetic INPUT generators shared by the oracle tests and the CUDA path.

This module holds none of the method's arithmetic (no env step, no net, no
search, no correction): it only turns seeds into root records and canonical
fp32 weight blobs, per the recipe in DESIGN.md §3 ("Input recipe").
"""
from .inputs import *  # noqa: F401,F403
