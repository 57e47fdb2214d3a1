# Round evidence on one GPU: bench lines, ncu launch lists and full captures.
# usage: bash tools/evidence.sh TAG   (outputs under gpurun_out/TAG_*)
T=${1:-ev}
mkdir -p gpurun_out
for c in ${BENCH_CONFIGS-c2 c3 c4}; do
  timeout 600 python bench.py --config $c --steps ${STEPS:-20} --warmup 3 > gpurun_out/${T}_bench_$c.json 2> gpurun_out/${T}_bench_$c.err
  echo "bench $c exit=$?"
done
for c in ${LAUNCH_CONFIGS-c2 c4}; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${T}_launches_$c.csv python tools/prof_run.py $c 4 > /dev/null 2>&1
  echo "launches $c exit=$?"
done
for spec in ${FULL_SPECS-c2:core c3:core c2:basis}; do
  c=${spec%%:*}; k=${spec##*:}
  timeout 900 ncu --set full --clock-control none --import-source on --kernel-name regex:$k --launch-skip 2 --launch-count 1 \
    -o gpurun_out/${T}_full_${c}_$k -f python tools/prof_run.py $c 4 > /dev/null 2>&1
  echo "full $c $k exit=$?"
  # summaries travel back; the reports only when asked (gpurun copies <= 64 MiB)
  python tools/ncu_summary.py gpurun_out/${T}_full_${c}_$k.ncu-rep 16 > gpurun_out/${T}_full_${c}_$k.txt 2>&1
  [ -n "$KEEP_REP" ] || rm -f gpurun_out/${T}_full_${c}_$k.ncu-rep
done
