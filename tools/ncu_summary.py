"""Summarise ncu --set full reports (.ncu-rep) into the JSON kept under profiles/: per launch the duration,
DRAM traffic, issue / pipe utilisation, occupancy and the top stall reasons.
    python tools/ncu_summary.py gpurun_out/prof_x.ncu-rep [...] --source "<command>" -o profiles/r01/x.json"""
import argparse
import csv
import io
import json
import subprocess

KEEP = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_elapsed.avg.per_second",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size"]
STALL = "smsp__average_warps_issue_stalled_"


def rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    r = list(csv.reader(io.StringIO(out)))
    hdr, units = r[0], r[1]
    for row in r[2:]:
        yield {h: (v, u) for h, u, v in zip(hdr, units, row)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("reps", nargs="+")
    ap.add_argument("--source", default="")
    ap.add_argument("-o", "--out", required=True)
    a = ap.parse_args()
    kernels = []
    for rep in a.reps:
        for d in rows(rep):
            k = {"kernel": d.get("Kernel Name", ("", ""))[0][:160]}
            for m in KEEP:
                if m in d:
                    v, u = d[m]
                    k[m] = f"{v} {u}".strip()
            st = {}
            for h, (v, u) in d.items():
                if h.startswith(STALL) and h.endswith("_per_issue_active.ratio"):
                    try:
                        st[h[len(STALL):-len("_per_issue_active.ratio")]] = round(float(v.replace(",", "")), 2)
                    except ValueError:
                        pass
            k["stalls_per_issue"] = dict(sorted(st.items(), key=lambda x: -x[1])[:9])
            kernels.append(k)
    json.dump({"source": a.source, "kernels": kernels}, open(a.out, "w"), indent=1)
    print(f"{len(kernels)} launches -> {a.out}")


if __name__ == "__main__":
    main()
