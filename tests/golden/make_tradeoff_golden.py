"""Freezes the reference's own tradeoff reports as fixtures (run where /root/reference exists).

Source: /root/reference/proj/scenarios/tradeoff_{bimodal,uniform}.cfg (workload + engine settings)
and the deterministic reports the reference shipped for them, /root/reference/proj/out/*.tradeoff.json
(reproduced byte-identically by the compiled reference in this container).
Writes tests/golden/tradeoff_cases.json: {name: {workload, engine, target, report}}.
"""
import configparser
import json
import os

REF = "/root/reference/proj"
HERE = os.path.dirname(os.path.abspath(__file__))
INT = {"n_requests", "dim", "block_size", "n_layers", "context_min", "context_max", "decode_steps",
       "planted_blocks", "planted_blocks_alt", "seed"}


def main():
    cases = {}
    for name in ("tradeoff_bimodal", "tradeoff_uniform"):
        cp = configparser.ConfigParser(inline_comment_prefixes=("#",))
        cp.read(os.path.join(REF, "scenarios", name + ".cfg"))
        wl = {k: (int(v) if k in INT else float(v)) for k, v in cp["workload"].items()}
        eng = dict(cp["engine"])
        cases[name] = dict(
            workload=wl,
            engine=dict(microbatch=int(eng.get("microbatch", 1)), estimator=eng.get("estimator", "cuboid_mean"),
                        ranking=eng.get("ranking", "estimated"), audit=eng.get("audit", "false") == "true"),
            target=float(cp["tradeoff"]["target_coverage"]),
            report=json.load(open(os.path.join(REF, "out", name + ".tradeoff.json"))))
    json.dump(cases, open(os.path.join(HERE, "tradeoff_cases.json"), "w"), indent=1)
    print(json.dumps(cases, indent=1))


if __name__ == "__main__":
    main()
