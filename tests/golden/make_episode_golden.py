"""Episode golden (compare_golden.csv) from the UNMODIFIED
reference harness (oracle/_ref/libkeep_ref_episode.so).

compare_csv over generate_episode(base_config(20250807, 12, 4, 5)) for the
strategies full, full-reuse and keep (test_harness.cpp:231-241).  The script
checks that the reference run here reproduces the reference's own committed
golden byte for byte (proj/tests/golden/compare_golden.csv) before writing
tests/golden/compare_golden.csv.

    python tests/golden/make_episode_golden.py
"""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

from oracle.episode_oracle import EpisodeOracle  # noqa: E402
from test_episode_cpu import base_config  # noqa: E402

from paper_2602_23592_b200 import episode as ep  # noqa: E402


def main():
    kre = EpisodeOracle()
    cfg = base_config(20250807, 12, 4, 5)
    trace = kre.generate(cfg.to_json())
    csv = kre.compare_csv(cfg.to_json(), trace, ["full", "full-reuse", "keep"])
    ref_file = "/root/reference/proj/tests/golden/compare_golden.csv"
    if os.path.exists(ref_file):
        with open(ref_file) as f:
            assert f.read() == csv, "the reference run here does not reproduce its committed golden"
    with open(os.path.join(HERE, "compare_golden.csv"), "w") as f:
        f.write(csv)
    print(csv)


if __name__ == "__main__":
    main()
