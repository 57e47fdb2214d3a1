# Round-2 final evidence on one GPU (outputs under gpurun_out/r02b_*):
# bench lines, ncu launch lists (per-launch duration) and full captures.
mkdir -p gpurun_out
for c in ${BENCH_CONFIGS-c5 c4 c2 c3 c1}; do
  timeout 900 python bench.py --config $c --steps ${STEPS:-10} --warmup 3 > gpurun_out/r02b_bench_$c.json 2> gpurun_out/r02b_bench_$c.err
  echo "bench $c exit=$?"
done
for c in ${LAUNCH_CONFIGS-c5 c4 c2}; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/r02b_launches_$c.csv python tools/prof_run.py $c 3 > /dev/null 2>&1
  echo "launches $c exit=$?"
  python tools/launch_table.py gpurun_out/r02b_launches_$c.csv > gpurun_out/r02b_launches_$c.txt 2>&1
done
for spec in ${FULL_SPECS-c5:core_kernel c4:basis_wtree_kernel c4:basis_wfactor_kernel c5:basis_wide_top_kernel c2:basis_wtree_kernel c4a20:sketch_contig_kernel}; do
  c=${spec%%:*}; k=${spec##*:}
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k --launch-skip 1 --launch-count 1 \
    -o gpurun_out/r02b_full_${c}_$k -f python tools/prof_run.py $c 3 > /dev/null 2>&1
  echo "full $c $k exit=$?"
  python tools/ncu_summary.py gpurun_out/r02b_full_${c}_$k.ncu-rep 16 > gpurun_out/r02b_full_${c}_$k.txt 2>&1
  [ -n "$KEEP_REP" ] || rm -f gpurun_out/r02b_full_${c}_$k.ncu-rep
done
