for m in A R; do echo "== mode $m"; timeout 300 python tools/round_sizes.py --config lognormal_example --t-stop 2 --quiet --mode $m 2>&1 | grep -v '"step": 1' | grep 'step\|nI\|Error'; done
for m in A R; do echo "== affine mode $m"; timeout 300 python tools/round_sizes.py --config affine_example --t-stop 3 --quiet --mode $m 2>&1 | grep -v '"step": 1' | grep '"i": 5\|nI\|Error'; done
