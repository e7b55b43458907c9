"""Summarise an ncu app-range capture of ONE bench step into
profiles/r02/ncu_step_range_<config>.json (read by bench.py's roofline).

On a GPU box:
  ncu --replay-mode app-range --cache-control none --clock-control none \
      --metrics dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,\
smsp__inst_executed.sum,sm__inst_executed_pipe_fma.sum,\
sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_elapsed,\
smsp__issue_active.avg.pct_of_peak_sustained_elapsed,\
sm__warps_active.avg.pct_of_peak_sustained_elapsed,gpu__time_duration.sum \
      --csv --log-file gpurun_out/range.csv python bench.py --profile-range --config X
  python tools/step_range_summary.py gpurun_out/range.csv X <event-timed step ms>
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main(path, config, step_ms):
    rows = [r for r in csv.reader(open(path)) if len(r) > 5]
    hdr, data = rows[0], rows[1:]
    ni, vi, ui = hdr.index("Metric Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    m = {}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6, "ns": 1e-6,
             "usecond": 1e-3, "us": 1e-3, "ms": 1.0,
             "msecond": 1.0, "second": 1e3}
    for r in data:
        v = float(r[vi].replace(",", ""))
        m[r[ni]] = v * scale.get(r[ui], 1.0)
    out = {
        "command": "ncu --replay-mode app-range --cache-control none --clock-control none "
                   "--metrics <below> python bench.py --profile-range --config " + config,
        "what": f"ONE whole {config} step (grid build, all dimensions' PDL-chained flooding kernels "
                "on their concurrent streams, facet completion) as a single cudaProfilerStart/Stop "
                "range, after 3 warm-up steps and a 256 MB L2 flush, caches NOT flushed by ncu: the "
                "traffic of the real step",
        "range_duration_ms": m.get("gpu__time_duration.sum"),
        "range_duration_note": "wall time of the range under ncu's instrumentation (launch gaps "
                               f"included); the same step times {step_ms} ms with CUDA events in bench.py",
        "dram_bytes_read": m["dram__bytes_read.sum"],
        "dram_bytes_write": m["dram__bytes_write.sum"],
        "dram_note": "writes include the write-back of the dirty lines the pre-step L2 flush left "
                     "(256 MB memset), evicted by the step",
        "lts_bytes": m.get("lts__t_bytes.sum"),
        "smsp_inst_executed": m.get("smsp__inst_executed.sum"),
        "sm_inst_executed_pipe_fma": m.get("sm__inst_executed_pipe_fma.sum"),
        "sm_pipe_fma_cycles_active_pct_of_range": m.get(
            "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_elapsed"),
        "smsp_issue_active_pct_of_range": m.get("smsp__issue_active.avg.pct_of_peak_sustained_elapsed"),
        "sm_warps_active_pct_of_range": m.get("sm__warps_active.avg.pct_of_peak_sustained_elapsed"),
    }
    out["dram_bytes_per_step"] = out["dram_bytes_read"] + out["dram_bytes_write"]
    dst = os.path.join(ROOT, "profiles", "r02", f"ncu_step_range_{config}.json")
    with open(dst, "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], float(sys.argv[3]))
