# full GPU test suite + the five bench configs (development)
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
for c in $*; do SRTT_DEBUG_PLAN=1 timeout 300 python tools/prof_run.py $c 3 2>&1 | grep -v "^0 \|^1 " | tail -2 | grep -o "core plan.*\|'core': [0-9.]*\|{'sampling.*}"; done
