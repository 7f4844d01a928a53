"""Summarise an `ncu --set full` capture into the text committed under
profiles/: headline metrics per launch, then the warp-stall breakdown and the
hottest SASS lines. The source page of a report aggregates every launch in it,
so the stall/SASS sections are printed only for single-launch reports (capture
one kernel per report: `-k regex:<name> -s <skip> -c 1`); SASS lines are
listed once per address.

    python profiles/summarize_ncu.py gpurun_out/prof_cast.ncu-rep [units] > profiles/rNN/....txt
"""
import csv
import io
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sectors.sum",
    "lts__t_sector_hit_rate.pct", "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__t_sector_hit_rate.pct", "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__maximum_warps_per_active_cycle_pct",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "smsp__thread_inst_executed_per_inst_executed.ratio", "smsp__inst_executed.sum",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__sass_average_branch_targets_threads_uniform.pct",
    "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "l1tex__t_output_wavefronts_pipe_lsu_mem_global_op_ld.sum",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
]


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main():
    rep = sys.argv[1]
    units = float(sys.argv[2]) if len(sys.argv) > 2 else None
    raw = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    hdr, unit, vals = raw[0], raw[1], raw[2:]
    for r in vals:
        name = r[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        print(f"== kernel: {name[:100]}")
        got = {}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                got[k] = (r[i], unit[i])
                print(f"  {k:64s} {r[i]:>20s} {unit[i]}")
        if units and "dram__bytes_read.sum" in got:
            def tob(v, u):
                v = float(v.replace(",", ""))
                return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
            tot = tob(*got["dram__bytes_read.sum"]) + tob(*got["dram__bytes_write.sum"])
            print(f"  dram bytes per unit ({units:.0f} units): {tot / units:.2f}")
    if len(vals) != 1:
        print(f"== {len(vals)} launches in this report: stall and SASS sections skipped "
              "(they would aggregate all launches)")
        return
    sass = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source",
                                           "sass"))))
    if len(sass) < 3:
        return
    hdr, data = sass[1], sass[2:]
    ix = {h: i for i, h in enumerate(hdr)}

    def f(r, k):
        try:
            return float(r[ix[k]])
        except (KeyError, ValueError, IndexError):
            return 0.0
    tot = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data) or 1.0
    stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    print("== warp stall breakdown (% of samples)")
    for s, v in sorted(((s, sum(f(r, s) for r in data)) for s in stalls), key=lambda x: -x[1])[:10]:
        print(f"  {s:28s} {100 * v / tot:5.1f}")
    print("== hottest SASS (samples, warp-instructions executed, avg active threads)")
    seen, uniq = set(), []
    for r in data:
        key = r[ix["Address"]] if "Address" in ix else r[ix["Source"]]
        if key not in seen:
            seen.add(key)
            uniq.append(r)
    for r in sorted(uniq, key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))[:25]:
        print(f"  {r[ix['Source']][:64]:64s} {int(f(r, 'Warp Stall Sampling (All Samples)')):8d} "
              f"{int(f(r, 'Instructions Executed')):11d} {f(r, 'Avg. Threads Executed'):5.1f}")


if __name__ == "__main__":
    main()
