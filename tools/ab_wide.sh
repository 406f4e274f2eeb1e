for rep in 1 2; do
for v in v0 v1 v2 v3; do
  if [ $v = v0 ]; then L=""; else L="SPOCK_LIB=paper_2505_12078_b200/_build_alt/lib_$v.so"; fi
  r=$(python tools/sweep_T.py c3,c4 "$L" 2>&1 | grep ms_per_T | python -c "import sys,json; l=sys.stdin.read(); j=json.loads(l[l.index('['):l.rindex(']')+1]); print(' '.join('%s=%.4f'%(x['config'],x['ms_per_T']) for x in j))")
  s=$(env $L python tools/shape_sweep.py 100,10,3 48,3,7 12,100,2 2>/dev/null | python -c "import sys,json; print(' '.join('%d,%d,%d=%.3f'%(j['N'],j['nw'],j['nb'],j['ms_per_T']) for j in map(json.loads, sys.stdin)))")
  echo "rep$rep $v $r $s"
done; done
