"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NONE of the method's arithmetic: no layouts, no addresses,
no clustering.  It only produces field VALUES (per-field byte columns) and raw
random bytes, which both sides then lay out with their own code.

Recipes (SURVEY.md 8(d) "Values"):
  Mode A "random bits": byte k of field f's column is a byte of the
      splitmix64 stream seeded with (seed, f); then 1/16 of the fp-sized slots
      (4-byte slots read as fp32, 8-byte slots as fp64) are overwritten with a
      special value drawn from {sNaN with random payload, qNaN with random
      payload, +Inf, -Inf, -0.0, smallest positive denormal}.
  Mode B "tagged": slot (i, f) holds the little-endian bytes of
      (i << 12) | f, truncated to the field width, so a misplaced slot names
      its record and field.
"""
from .gen import (SEED_BASE, splitmix64, random_bytes, field_columns, tagged_columns,
                  fill_random_device, config_widths, kmeans_widths, medical_fields)

__all__ = ["SEED_BASE", "splitmix64", "random_bytes", "field_columns", "tagged_columns",
           "fill_random_device", "config_widths", "kmeans_widths", "medical_fields"]
