for c in c2 c3 c4; do for f in 16,2 16,1 8,2 8,1; do
  r=$(SRTT_DEBUG_PLAN=1 SRTT_FORCE_CORE=$f python tools/prof_run.py $c 3 2>&1 | tail -2 | tr '\n' ' ')
  echo "$c $f $(echo $r | grep -o 'warps=[0-9]* tpb=[0-9]* ns=[0-9]*') core=$(echo $r | grep -o "'core': [0-9.]*" | tail -1)"
done; done
