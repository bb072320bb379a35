import json, sys
d = json.load(open(sys.argv[1] if len(sys.argv) > 1 else 'gpurun_out/bench.json'))
r = d['roofline']
print('HEAD', d['config']['workload'], '%.3e' % d['value'], 'ms=%.3f' % d['ms_per_step'], 'frac=%.3f' % r['frac'], r['bound'],
      'kms=%.3f' % r['kernel_ms'], d['plan'], 'e2e=%.3e' % d['e2e']['value'], 'clk', d['clocks'])
print('peaks', d['peaks_probe'])
if d.get('cpu_baseline'): print('cpu', '%.3e' % d['cpu_baseline']['value'], d['cpu_baseline']['cores'])
for k, v in d['per_config'].items():
    print('%-28s %.3e ms=%8.3f frac=%.3f %-28s kms=%8.3f' % (k, v['value'], v['ms_per_step'], v['roofline_frac'], v['bound'], v['kernel_ms']), v['plan'])
