# sustained A/B of two library builds: A=$1 B=$2 (paths), 3 alternating rounds
for r in 1 2 3; do for L in "$1" "$2"; do echo "== $L"; timeout 120 python tools/ab_step.py "$L" 4; done; done
