tools/dsmem_probe 2000 2>&1 | tee gpurun_out/r2_dsmem.log
for cfg in "--qubits 20 --levels 1" "--qubits 26 --levels 4" "--qubits 33 --levels 4 --graph er --steps 5 --warmup 3"; do
  python bench.py $cfg --no-cpu-baseline 2>&1 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']
print(d['config']['workload'], 'value', round(d['value'],3), 'e2e', round(d['e2e']['value'],3), 'frac', round(r['frac'],3), 'expect', d['expectation'], 'K1', d['cut_table_build'] and round(d['cut_table_build']['ms'],3), 'clk', d['clocks']['sm_mhz'])"
done 2>&1 | tee gpurun_out/r2_configs.log
