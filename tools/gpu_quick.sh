# quick GPU loop: selected tests + per-config stage times (development)
T=${TESTS:-"tests/test_gpu_components.py tests/test_gpu_tucker.py tests/test_gpu_htucker.py"}
timeout 900 python -m pytest $T -x -q 2>&1 | tail -4
for c in ${CONFIGS:-c1 c2 c3 c4}; do echo "== $c"; SRTT_DEBUG_PLAN=1 timeout 300 python tools/prof_run.py $c 3 2>&1 | grep -v "^0 \|^1 " | tail -1; done
