# flat vs item core pass: plans and core-kernel times (development)
for c in c2 c3; do for f in "0 16,2" "0 8,1" "1 16,2" "1 16,1" "1 8,1" "1 8,2"; do set -- $f
  echo "== $c flat=$1 force=$2"; SRTT_DEBUG_PLAN=1 SRTT_FORCE_FLAT=$1 SRTT_FORCE_CORE=$2 timeout 300 python tools/prof_run.py $c 3 2>&1 | grep -v "^0 \|^1 " | tail -2 | grep -o "core plan.*\|'core': [0-9.]*"
done; done
