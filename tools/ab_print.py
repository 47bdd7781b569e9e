import json,sys
l=[x for x in open(sys.argv[1]) if x.startswith("{")][-1]
d=json.loads(l)
pi=d["per_integrator"]
print({k: round(pi[k]["path_steps_per_s"]/1e9,2) for k in ("se","gl","baoab")})
c=d["baseline_configs"]
print({k: round(v["total_ms"],2) for k,v in c["config2_floored_levels0to8_1e6"].items()})
print([round(r["paths_per_s"]/1e6) for r in c["config4_z0_10m_64bins_gl"]["levels"]])
