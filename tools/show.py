import json, sys
for f in sys.argv[1:]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except Exception as e:
        print(f, "ERR", e); continue
    r = d.get("roofline", {})
    print(f"{f}: value={d['value']:.4g} ms={d['ms_per_step']:.1f} phases={ {k: round(v*1e3,1) for k,v in d.get('phases_s',{}).items()} } "
          f"far_frac={r.get('frac')} near_frac={d.get('near_roofline',{}).get('frac')} inter={d.get('interaction_frac')} "
          f"clk={d.get('clocks',{}).get('sm_mhz')} e2e={d.get('e2e',{}).get('value')}")
