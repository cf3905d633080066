"""Regenerate the golden fixtures from the REFERENCE library (oracle/_ref).

    python tests/golden/make_golden.py

plan_*.json  the reference's pipelined plan (hiercoll-pipelined-v1 text,
             factorize.cpp:587 + pipeline.cpp:76 + pipeline.cpp:147) for the
             config in the matching .meta file; tests/test_plan_parity.py
             requires hiccl's plan to equal it byte for byte.
fill_*.npy   known-answer vectors of the shared input generator
             (oracle/numeric_exec.c header), pinned here once.
"""
import json
import sys
from pathlib import Path

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent.parent))
import numpy as np  # noqa: E402

import oracle  # noqa: E402

CONFIGS = {
    # name: (kind, form, p, count, root, op, hier, g, stripe, ring, depth)
    "ar_multi_p8_2x4_s4_n2_m3": (7, 1, 8, 5, 0, 0, [2, 4], 4, 4, 2, 3),
    "ar_single_p4_flat": (7, 0, 4, 3, 0, 0, [4], 4, 1, 1, 1),
    "ar_multialt_p8_222_g2_s2_n4_m2": (7, 2, 8, 4, 0, 1, [2, 2, 2], 2, 2, 4, 2),
    "ag_single_p8_222_g8": (5, 0, 8, 3, 0, 0, [2, 2, 2], 8, 1, 1, 1),
    "rs_single_p8_222_g2_s2": (6, 0, 8, 3, 0, 0, [2, 2, 2], 2, 2, 1, 1),
    "a2a_p8_2x4_n2": (4, 0, 8, 2, 0, 0, [2, 4], 4, 1, 2, 1),
    "bcast_single_p8_g1_ring8_m4": (1, 0, 8, 3, 2, 0, [2, 2, 2], 1, 1, 8, 4),
    "bcast_multi_p8_flat": (1, 1, 8, 2, 0, 0, [8], 8, 1, 1, 1),
    "reduce_multi_p12_322_s4": (3, 1, 12, 2, 5, 0, [3, 2, 2], 4, 4, 3, 1),
    "scatter_p8_2x4": (0, 0, 8, 4, 3, 0, [2, 4], 4, 4, 2, 2),
    "gather_p8_2x4": (2, 0, 8, 4, 6, 0, [2, 4], 4, 4, 2, 2),
}


def main():
    ref = oracle.Reference()
    for name, cfg in CONFIGS.items():
        rc, text = ref.preset_plan(*cfg)
        assert rc == 0, (name, text)
        (HERE / f"plan_{name}.json").write_text(text)
        (HERE / f"plan_{name}.meta").write_text(json.dumps({"config": cfg}) + "\n")
    for dt in ("f32", "bf16", "f16", "i32", "i64", "f64", "u8"):
        np.save(HERE / f"fill_{dt}.npy", oracle.fill(64, dt, 1234, 3, index_base=1000))


if __name__ == "__main__":
    main()
