"""Markdown table of one GPU pass (tools/gpu_final.sh output directory).

    python tools/summarize_pass.py gpurun_out/final1 > profiles/r02/final_table.md
"""

import glob
import json
import os
import sys


def last_json(path):
    try:
        with open(path) as f:
            lines = [ln for ln in f.read().splitlines() if ln.startswith("{")]
        return json.loads(lines[-1]) if lines else None
    except (OSError, ValueError):
        return None


def row(name, line, extra=""):
    r = line["roofline"]
    c = line["config"]
    cold = line.get("cold_e2e") or {}
    pg = line["e2e"].get("pageable_inputs", {}).get("value")
    return ("| %s | %.3g | %.3g | %s | %.3f | %s | L%d J%d %s %d CTA | %s |%s"
            % (name, line["value"], line["e2e"]["value"], "%.3g" % pg if pg else "",
               r["frac"], "%.3f" % r["w_em_frac"] if r.get("w_em_frac") is not None else "",
               c.get("lanes_per_orbit", 0), c.get("oscillators_per_lane", 0),
               "pers" if c.get("persistent_grid") else "grid", c.get("ctas_per_sm", 0),
               "%.0f / %.0f ms" % (cold["ms"], cold["second_call_ms"]) if "ms" in cold else "",
               extra))


def main():
    d = sys.argv[1]
    print("| workload | device orbit-steps/s | e2e (pinned in) | e2e (pageable in) | FP64 frac "
          "| W_EM frac | layout | cold / 2nd call |")
    print("|---|---|---|---|---|---|---|---|")
    head = last_json(os.path.join(d, "bench_default.log"))
    if head:
        for k, v in head.get("sizes", {}).items():
            print("| %s | %.3g | %.3g | | %.3f | %s | L%d J%d %s %d CTA | |"
                  % (k, v["value"], v["e2e"], v["frac"],
                     "%.1f" % v["w_em_frac"] if v.get("w_em_frac") else "",
                     v["lanes_per_orbit"], v["oscillators_per_lane"],
                     "pers" if v["persistent_grid"] else "grid", v["ctas_per_sm"]))
        for k, v in head.get("secondary", {}).items():
            print("| %s | %.3g | %.3g | | %.3f | %s | L%d J%d %s %d CTA | |"
                  % (k, v["value"], v["e2e"], v["frac"],
                     "%.2f" % v["w_em_frac"] if v.get("w_em_frac") else "",
                     v["lanes_per_orbit"], v["oscillators_per_lane"],
                     "pers" if v["persistent_grid"] else "grid", v["ctas_per_sm"]))
        print(row("**headline %s**" % head["config"]["headline"], head))
    for path in sorted(glob.glob(os.path.join(d, "bench_*.log"))):
        name = os.path.basename(path)[len("bench_"):-len(".log")]
        if name in ("default", "reference"):
            continue
        line = last_json(path)
        if line is None:
            print("| %s | (failed) |" % name)
            continue
        vs = " %.0fx P100" % line["vs_baseline"] if line.get("vs_baseline") else ""
        print(row(name.replace("pw_", "pairwise ") , line, vs))
    ref = last_json(os.path.join(d, "bench_reference.log"))
    if ref:
        print()
        print("Reference arm: %.4g orbit-steps/s (%s, %s)" % (ref["value"], ref["cpu_baseline"]["kind"],
                                                           ref["cpu_baseline"]["sample"]))
    if head and head.get("cpu_baseline"):
        cb = head["cpu_baseline"]
        print()
        print("cpu_baseline legs: " + "; ".join(
            "threads=%s: %.4g orbit-steps/s (chunk_group %d, %d orbits x %d steps)"
            % (g["threads"], g["value"], g["chunk_group"], g["orbits"], g["steps"])
            for g in cb.get("legs", [])))
        print()
        print("clocks: %s" % json.dumps(head.get("clocks")))


if __name__ == "__main__":
    main()
