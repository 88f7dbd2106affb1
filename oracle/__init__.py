"""CPU oracle for the ADHA layout remap and the ODS/PDL planner.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import, call,
link or execute anything under ``oracle/``.  The product package
``paper_1407_4859_b200`` never imports it and shares no code with it.

Contents
  remap_oracle.c  plain C: per-record, per-field memcpy
  remap.py        ctypes wrapper + numpy helpers (pack/unpack per-field columns)
  planner.py      plain Python ODS / PDL planner and brute-force searches
                  (SPEC.md [OP]s build_affinity_graph ... brute_force_plan)
"""
