import json, sys
rows=[x for x in json.load(open(sys.argv[1])) if x['integrator']=='pagani']
by={}
for x in rows: by.setdefault((x['family'],x['d']),[]).append(x)
n=0
for k,v in by.items():
    for x in v:
        for y in v:
            if y['regions']>x['regions'] and x['seconds']>1.3*y['seconds'] and x['seconds']>2e-4:
                print("  anomaly",k, x['rel_tol'], round(x['seconds']*1e3,2), x['regions'], 'vs', y['rel_tol'], round(y['seconds']*1e3,2), y['regions']); n+=1; break
print(sys.argv[1], "pagani s", round(sum(x['seconds'] for x in rows),3), "anomalies", n)
