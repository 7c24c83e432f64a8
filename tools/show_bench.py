import json,sys
for f in sys.argv[1:]:
    try:
        l=json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "ERR", e); continue
    print(f, round(l['ms_per_step'],4),'ms', '%.3g nodes/s'%l['value'], 'dec/s %.1f'%l['decisions_per_s'], 'e2e %.3g'%l['e2e']['value'], l['roofline']['kernel'], l['roofline']['bound'], '%.3g'%l['roofline']['achieved'], '%.3f'%l['roofline']['frac'], 'cpu', l.get('cpu_baseline') and '%.3g'%l['cpu_baseline']['value'])
    print('   ', {k:(round(v['ms_per_launch'],4), v['launches_per_step'], round(v['share'],3), round(v['achieved'],1)) for k,v in l['kernels'].items()})
