# A/B of library options on the bench workloads (+ optional parity subset first)
# env: TESTS (pytest -k expr, or "all" / "none"), WORKLOADS, OPTS (space-separated
# variants, each a comma-separated key=val list or "-"), STEPS, TAG
O=gpurun_out; mkdir -p $O; T=${TAG:-ab}
if [ "${TESTS:-none}" != "none" ]; then
  if [ "$TESTS" = "all" ]; then timeout 1500 python -m pytest tests -m gpu -q > $O/${T}_pytest.log 2>&1
  else timeout 1200 python -m pytest tests -m gpu -q -k "$TESTS" > $O/${T}_pytest.log 2>&1; fi
  echo "pytest exit $?" >> $O/${T}_pytest.log; tail -4 $O/${T}_pytest.log
fi
for w in ${WORKLOADS:-su2random_n28}; do
for opt in ${OPTS:--}; do
  a=""; [ "$opt" != "-" ] && a=$(for x in ${opt//,/ }; do echo --opt $x; done)
  timeout 300 python bench.py --steps ${STEPS:-20} --warmup 5 --no-e2e --no-cpu --workload $w $a > $O/${T}_q.json 2> $O/${T}_q.err
  python -c "
import json
d=json.loads(open('$O/${T}_q.json').read().strip().splitlines()[-1])
c=d.get('details', d['config']); r=d['roofline']
print('$w $opt', d['ms_per_step'], '%.3g'%d['value'], c['plan']['kernels'], r['frac'], r['avg_launch_ms'], d['clocks']['sm_mhz'], d['clocks']['reasons'])
" || tail -3 $O/${T}_q.err
done; done
if [ -n "$NCU" ]; then
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${T}_launches.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu $NCU > $O/${T}_launches_run.log 2>&1
  echo "ncu launches exit $?"
fi
