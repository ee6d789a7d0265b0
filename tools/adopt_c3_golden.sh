#!/bin/bash
# Adopt a generated C3-width golden (tests/golden/make_c3_golden.py output):
# record its sha256, run tests/test_gpu_c3_golden.py against it on a B200, and
# keep the recorded hash only if the test passes.
#   bash tools/adopt_c3_golden.sh        (from this container; uses gpurun)
set -e
cd "$(dirname "$0")/.."
G=tests/golden/c3_width_golden.npz
[ -f "$G" ] || { echo "no $G"; exit 1; }
sha256sum "$G" | cut -d' ' -f1 > "$G.sha256"
if /usr/local/graft/bin/gpurun --timeout 1800 -- 'python -m pytest tests/test_gpu_c3_golden.py -q -p no:cacheprovider -rs'; then
    echo "adopted: $(cat $G.sha256)"
else
    rm -f "$G.sha256"
    echo "test failed: golden not adopted"
    exit 1
fi
