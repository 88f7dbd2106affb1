"""Write the seeded random variant of the C3 affinity program ("a seeded random
program variant (seed 14074859; 24 groups, 2-10 fields each, freq in {1..4}, 70 % irregular)")
and the layout the ORACLE planner gives it:

    python tools/make_c3_random_program.py      -> tests/golden/c3_random_program.json
                                                   tests/golden/c3_random_expected.json

The program draws only the access groups (which fields, how often, which pattern); the layout is
computed by oracle/planner.py (ODS) and nothing else, so the stored string is an
oracle value, not a CUDA-path value.  64 fields with C3's widths (w_i = 8 if i % 4 == 3 else 4,
SURVEY.md Q1), one section on the B200 device of tests/golden/b200_arch.json (coalescing, 128-byte
cluster capacity, reading Q15), trip count = 50M records.
"""
import json
import os
import random
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from oracle import planner as P  # noqa: E402

SEED = 14074859
N = 50_000_000


def program():
    rng = random.Random(SEED)
    fields = [{"name": f"f{i}", "elem_bytes": 8 if i % 4 == 3 else 4} for i in range(64)]
    groups = []
    for _ in range(24):
        k = rng.randint(2, 10)
        members = sorted(rng.sample(range(64), k))
        groups.append({"fields": [f"f{i}" for i in members], "freq": rng.randint(1, 4),
                       "pattern": "irregular" if rng.random() < 0.7 else "streaming"})
    return {"schema_version": 1, "name": "c3_random", "record_count": N, "fields": fields,
            "sections": [{"id": "c3r", "trip_count": N, "allowed_devices": ["b200"], "groups": groups}],
            "order": ["c3r"]}


def main():
    prog = program()
    golden = os.path.join(ROOT, "tests", "golden")
    with open(os.path.join(golden, "c3_random_program.json"), "w") as f:
        json.dump(prog, f, indent=1)
    arch = json.load(open(os.path.join(golden, "b200_arch.json")))
    p, a = P.program_from_json(prog), P.arch_from_json(arch)
    lay = P.ods(p.sections[0], a.device("b200"), p)
    eb = p.elem_bytes()
    out = {"c3_random_hybrid": {"value": P.layout_string(lay), "n_clusters": len(lay),
                                "strides": [P.cluster_bytes(c, eb) for c in lay],
                                "source": "oracle/planner.py ods() of tests/golden/c3_random_program.json on "
                                          "b200_arch.json, written by tools/make_c3_random_program.py "
                                          f"(seed {SEED}; SURVEY.md 8(d))"}}
    with open(os.path.join(golden, "c3_random_expected.json"), "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
