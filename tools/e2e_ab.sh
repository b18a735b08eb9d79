for w in C5 C4; do
for v in 1 0; do
 DMHA_HOST_PIPELINE=$v python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline 2>/dev/null | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w pipeline=$v', round(d['value'],1), round(d['e2e']['value'],1), round(d['e2e']['ms_per_step'],1), d['clocks']['sm_mhz'])"
done; done
