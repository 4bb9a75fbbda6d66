"""Summarise one attention-kernel launch of an ncu --set full report into the JSON bench.py reads.

    python scripts/ncu_summary.py REPORT.ncu-rep --units U --out profiles/r02/attn_cfg2_ncu.json [--launch 0]

units = cached (token, KV head) pairs the launch attends (B * H_kv * N).  Fields per launch: DRAM
bytes (traffic), L1/shared LSU data-pipe wavefronts per unit (shared gathers + global code loads),
LSU data-pipe and issue utilisation, duration (ncu replays are cold-cache and serialised: shares and
per-unit counts are meaningful, the absolute time is not a bench number).
"""
import argparse
import csv
import io
import json
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--units", type=float, required=True)
    ap.add_argument("--out", required=True)
    ap.add_argument("--launch", type=int, default=0)
    args = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", args.report, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    head, units_row, vals = rows[0], rows[1], rows[2 + args.launch]
    m = dict(zip(head, vals))
    unit_of = dict(zip(head, units_row))

    def num(k):
        v = float(m[k].replace(",", ""))
        u = unit_of.get(k, "")
        scale = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "us": 1.0, "ms": 1e3, "ns": 1e-3}.get(u, 1.0)
        return v * scale

    sms = float(m.get("device__attribute_multiprocessor_count", "148").replace(",", ""))
    lsu = num("SM_A.TriageCompute.l1tex__data_pipe_lsu_wavefronts.avg") * sms
    shared = num("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum")
    glob = num("SM_A.TriageCompute.l1tex__data_pipe_lsu_wavefronts_mem_lgds.avg") * sms
    out = {
        "kernel": m.get("Kernel Name", ""),
        "units_per_launch": args.units,
        "traffic_per_launch": num("dram__bytes_read.sum") + num("dram__bytes_write.sum"),
        "lsu_wavefronts_per_unit": lsu / args.units,
        "lsu_shared_wavefronts_per_unit": shared / args.units,
        "lsu_global_wavefronts_per_unit": glob / args.units,
        "lsu_pipe_pct": num("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"),
        "issue_active_pct": num("smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "ncu_duration_us": num("gpu__time_duration.sum"),
        "source": args.report,
    }
    with open(args.out, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
