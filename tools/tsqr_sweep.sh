# TSQR block/top sweep on the H-Tucker and C5 configs (development)
for t in "1024,400" "" "256,128" "512,256" "192,64"; do
  for c in c4 c5; do echo "$c tsqr=$t"; SRTT_TSQR=$t timeout 300 python tools/prof_run.py $c 3 2>&1 | tail -1 | grep -o "'sketch': [0-9.]*, 'basis': [0-9.]*, 'core': [0-9.]*"; done
done
