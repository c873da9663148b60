import json, sys
for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        k = d['kernel_ms']
        print(f, round(d['value'], 1), 'e2e', round(d['e2e']['value'], 1), 'total', d['stages_ms']['total_ms'],
              {x: k.get(x) for x in ('fft_x', 'fft_y', 'fft_z', 'ifft_y', 'ifft_x', 'mc')}, d['clocks']['sm_mhz'])
    except Exception as e:
        print(f, 'ERR', e)
