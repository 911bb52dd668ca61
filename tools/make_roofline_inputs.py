"""Write profiles/roofline_inputs.json (read by bench.py) from an ncu summary (tools/ncu_summary.py)
and the plan statistics of the same workload (bench JSON line 'plan').

fp64 flops per kernel entry = (2 DFMA + DADD + DMUL) thread instructions / entries per launch
(the counted work of the shipped evaluator); traffic = DRAM read + write bytes per launch."""
import json
import sys

summary, bench, tag = sys.argv[1], sys.argv[2], sys.argv[3]
S = [d for path in summary.split(",") for d in json.load(open(path))]  # comma-separated summaries
B = json.loads(open(bench).read().strip().splitlines()[-1])
entries = {"p2p_kernel": B["plan"]["p2p_pairs"], "near_kernel": B["plan"]["p2p_pairs"],
           "m2l_kernel": B["plan"]["m2l_entries"], "m2l_stored_kernel": B["plan"]["m2l_entries"]}
out = {"source": "profiles/%s_ncu_summary.json (ncu --set full, config %s)" % (tag, B["config"]["workload"][:2]),
       "fp64_tflops_measured": 34.063,
       "fp64_peak_source": "tools/fp64_peak.cu DFMA chains, 148 SM x 8 CTA x 256 thr: 25 back-to-back launches, "
                           "4.56 s sustained at a median 1965 MHz SM clock, no throttle reason: 34.06 TFLOP/s "
                           "(profiles/r2/fp64_peak_sustained.log, profiles/r2/fp64_peak_clocks.csv)",
       "kernels": {}}
for d in S:
    k = d["kernel"]
    if k in entries:
        e = entries[k]
        out["kernels"][{"near_kernel": "p2p"}.get(k, k.replace("_kernel", ""))] = {
            "entries_per_launch": e,
            "fp64_flops_per_entry": (2 * d["dfma"] + d["dadd"] + d["dmul"]) / e,
            "fp64_inst_per_entry": (d["dfma"] + d["dadd"] + d["dmul"]) / e,
            "inst_per_entry": d["warp_inst"] * 32 / e,
            "dram_bytes_per_launch": d["dram_read"] + d["dram_write"],
            "fp64_pipe_pct": d["fp64_pipe_pct"], "issue_pct": d["issue_pct"], "ncu_time_ms": d["time_ms"]}
json.dump(out, open("profiles/roofline_inputs.json", "w"), indent=1)
print(json.dumps(out, indent=1))
