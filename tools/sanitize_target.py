"""Small p = 8 virtual plans on one executor for compute-sanitizer
(memcheck / racecheck on small plans). Every copy mode, f32 and
bf16, flat {8} and the {2,4} / {2,2,2} virtual hierarchies with stripes
and pipelining; each result is checked bit for bit against the oracle so a
sanitizer run also proves the instrumented kernel computed the right thing.

  compute-sanitizer --tool memcheck  python tools/sanitize_target.py
  compute-sanitizer --tool racecheck python tools/sanitize_target.py

One executor only: the sanitizer serializes kernels, so executors that
wait on each other's flags cannot run under it.
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

import oracle  # noqa: E402  (checker only)
from tests import harness  # noqa: E402

REF = oracle.Reference() if oracle.reference_available() else None
CASES = [  # kind, form, d, hier, g, stripe, ring, pipeline, dtype
    (7, 1, 1000, [8], 8, 1, 1, 1, "f32"),
    (7, 1, 4099, [2, 4], 4, 4, 2, 4, "f32"),
    (7, 0, 513, [2, 2, 2], 2, 2, 4, 2, "bf16"),
    (5, 0, 777, [2, 2, 2], 8, 1, 1, 3, "f32"),
    (6, 1, 1024, [2, 4], 4, 2, 1, 2, "f32"),
    (1, 1, 640, [8], 8, 1, 1, 1, "f32"),
    (3, 1, 300, [2, 4], 4, 4, 1, 1, "f32"),
    (4, 0, 256, [2, 4], 4, 1, 2, 2, "f32"),
]


def main():
    n = 0
    for mode in ("pull", "push", "staged", "ll"):
        for kind, form, d, hier, g, s, ring, m, dtype in CASES:
            plan, _, _ = harness.make_plan(kind, form, 8, d, 0, 0, hier, g, ring, s, m)
            flat = harness.oracle_plan(plan, kind, form, 8, d, 0, 0, hier, g, ring, s, m, REF)
            want = harness.run_oracle(flat, plan, dtype, 11)
            got, _ = harness.run_device(plan, dtype, 11, devices=(0,), copy_mode=mode, repeat=2)
            harness.assert_bitwise(got, want, f"{mode} {kind}/{form} {hier} s{s} r{ring} m{m}")
            n += 1
    print(f"sanitize_target: {n} plans bit-exact")


if __name__ == "__main__":
    main()
