"""Freezes the reference's serving-scenario reports as fixtures (run where /root/reference exists).

Source: /root/reference/proj/scenarios/{smoke,serving_rho0,serving_rho95}.cfg and the deterministic
reports the reference shipped for them, /root/reference/proj/out/<name>.csv (reproduced byte-identically
by the compiled reference in this container). Defaults not set in a .cfg are the
reference's (ServingConfig serving.hpp:29-34, PSAConfig engine.hpp:23-39, scenario.cpp:190-292).
Writes tests/golden/serving_cases.json.
"""
import configparser
import csv
import json
import os

REF = "/root/reference/proj"
HERE = os.path.dirname(os.path.abspath(__file__))
INT = {"n_requests", "dim", "block_size", "n_layers", "context_min", "context_max", "decode_steps",
       "planted_blocks", "planted_blocks_alt", "seed"}


def main():
    cases = {}
    for name in ("smoke", "serving_rho0", "serving_rho95"):
        cp = configparser.ConfigParser(inline_comment_prefixes=("#",))
        cp.read(os.path.join(REF, "scenarios", name + ".cfg"))
        wl = {k: (int(v) if k in INT else float(v)) for k, v in cp["workload"].items()}
        eng, sto, srv, swp = (dict(cp[s]) if cp.has_section(s) else {} for s in ("engine", "store", "serving", "sweep"))
        rows = list(csv.DictReader(open(os.path.join(REF, "out", name + ".csv"))))
        cases[name] = dict(
            workload=wl,
            engine=dict(epsilon=float(eng.get("epsilon", 0.95)), microbatch=int(eng.get("microbatch", 4)),
                        estimator=eng.get("estimator", "cuboid_mean"), ranking=eng.get("ranking", "estimated"),
                        audit=eng.get("audit", "false") == "true"),
            store=dict(capacity=int(sto.get("capacity", 256)), policy=sto.get("policy", "unified"),
                       eviction=sto.get("eviction", "lru")),
            serving=dict(miss_cost_ms=float(srv.get("miss_cost_ms", 1.0)), hit_cost_ms=float(srv.get("hit_cost_ms", 0.0)),
                         compute_cost_ms=float(srv.get("compute_cost_ms", 0.1)),
                         overlap=srv.get("overlap", "true") == "true"),
            rows=[{k: (v if k == "method" else float(v)) for k, v in r.items()} for r in rows])
    json.dump(cases, open(os.path.join(HERE, "serving_cases.json"), "w"), indent=1)
    print(json.dumps(cases, indent=1)[:1500])


if __name__ == "__main__":
    main()
