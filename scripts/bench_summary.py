import json,sys
for f in sys.argv[1:]:
    try:
        d=json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, 'ERR', e); continue
    print(f, round(d['value']/1e6,2), 'Mtok/s', round(d['ms_per_step']*1e3,1), 'us', {k:round(v*1e3,1) for k,v in d.get('stages_ms',{}).items()}, 'hash frac', round(d.get('roofline',{}).get('frac',0),3), 't_dc', round(d.get('t_dc',{}).get('lsh_us',0),1))
