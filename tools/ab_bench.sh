# A/B of engine builds on one box: bench c2 step with each library (development)
for rep in 1 2; do for lib in lib_ab_start.so lib_ab_flat.so libsrtt_b200.so; do
  printf "%s " $lib; SRTT_LIB_AB=$lib python bench.py --config ${CFG:-c2} --steps 20 --warmup 3 --no-cpu-baseline | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), round(d['roofline']['kernel_ms'],4))"
done; done
