"""Summarise ncu captures into profiles/*.md (run in the build container).

    python profiles/summarize.py gpurun_out/prof_r01.ncu-rep gpurun_out/launches6.csv > profiles/r01_ncu_summary.md
"""

import collections
import csv
import io
import os
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg", "SM cycles"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "shared wavefronts"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed", "shared wavefronts % of peak"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "shared load bank conflicts"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("l1tex__m_xbar2l1tex_read_bytes.sum", "L2->L1 read bytes"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
    ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe %"),
    ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
    ("smsp__inst_executed.sum", "warp instructions"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe active %"),
    ("launch__registers_per_thread", "registers/thread"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "memory throughput %"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput %"),
]
STALLS = ["short_scoreboard", "wait", "selected", "long_scoreboard", "not_selected", "math_pipe_throttle",
          "branch_resolving", "mio_throttle", "lg_throttle", "barrier", "no_instructions", "dispatch_stall"]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    return [(hdr, units, r) for r in rows[2:]]


def main():
    rep, launches = sys.argv[1], (sys.argv[2] if len(sys.argv) > 2 else None)
    print(f"# ncu summary — `{rep.split('/')[-1]}`\n")
    cmd = os.environ.get("PQK_PROFILE_CMD", "python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e")
    print("Captured with `ncu --set full --clock-control none --import-source on` under gpurun on one B200 "
          f"(command: `{cmd}`).\n")
    for hdr, units, r in raw(rep):
        ix = {n: i for i, n in enumerate(hdr)}
        name = r[ix["Kernel Name"]]
        print(f"## `{name}`\n")
        print("| metric | value | unit |\n|---|---|---|")
        for key, label in METRICS:
            if key in ix:
                print(f"| {label} (`{key}`) | {r[ix[key]]} | {units[ix[key]]} |")
        tot = float(r[ix["smsp__pcsamp_sample_count"]]) if "smsp__pcsamp_sample_count" in ix else 0
        if tot:
            print("\nWarp-state samples (share of all samples):\n")
            print("| stall | share |\n|---|---|")
            for s in STALLS:
                key = f"smsp__pcsamp_warps_issue_stalled_{s}"
                if key in ix and r[ix[key]]:
                    print(f"| {s} | {float(r[ix[key]]) / tot:.3f} |")
        print()
    if launches:
        print(launch_table(launches))


UNIT = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3, "s": 1e6, "second": 1e6}
SETUP = ("encode", "Fill", "tables_to", "at::", "elementwise", "distribution", "gamma", "reduce_kernel", "vote_t16",
         "smem_probe", "pad_codes", "table_stats")


def launch_table(launches: str) -> str:
    """Per-kernel totals of an ncu `--metrics gpu__time_duration.sum --csv` launch list (µs)."""
    rows = list(csv.reader(open(launches)))
    hdr = None
    agg = collections.OrderedDict()
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            nm = d["Kernel Name"].split("(")[0]
            v = float(d["Metric Value"].replace(",", "")) * UNIT.get(d.get("Metric Unit", "ns"), 1e-3)
            a = agg.setdefault(nm, [0, 0.0])
            a[0] += 1
            a[1] += v
    first = [v[0] for k, v in agg.items() if "hscan_kernel<" in k] or \
        [v[0] for k, v in agg.items() if "pqk::scan_kernel<" in k]
    steps = max(first, default=1)
    per_step = {k: v for k, v in agg.items() if not any(t in k for t in SETUP)}
    tot = sum(v[1] for v in per_step.values())
    out = [f"## Launch list (`{launches.split('/')[-1]}`, `--metrics gpu__time_duration.sum`, cold and serialised)\n",
           f"{steps} Lloyd iterations; set-up kernels (data generation, encode, fills, table builds) excluded "
           "from the shares.\n",
           "| kernel | launches | avg µs | total ms | share of iteration kernel time |", "|---|---|---|---|---|"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        share = f"{v[1] / tot:.4f}" if k in per_step else "setup"
        out.append(f"| `{k[:90]}` | {v[0]} | {v[1] / v[0]:.1f} | {v[1] / 1e3:.3f} | {share} |")
    return "\n".join(out)

if __name__ == "__main__":
    main()
