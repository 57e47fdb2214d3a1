timeout 900 python -m pytest tests/test_gpu_components.py tests/test_gpu_tucker.py tests/test_gpu_configs.py -x -q 2>&1 | tail -3
for rep in 1 2; do for f in 0 1; do printf "cb=$f "; SRTT_FORCE_CB=$f python bench.py --steps 20 --warmup 3 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4))"; done; done
SRTT_DEBUG_PLAN=1 python tools/prof_run.py c2 2 2>&1 | grep plan
