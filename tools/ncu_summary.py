"""Summarise one `ncu --set full` capture of the sweep kernel into profiles/ (JSON + markdown).
    python tools/ncu_summary.py REP TAG "command" [launches.csv]"""
import csv
import json
import subprocess
import sys

rep, tag, cmd = sys.argv[1], sys.argv[2], sys.argv[3]
launches = sys.argv[4] if len(sys.argv) > 4 else None
raw = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                                     text=True).stdout.splitlines()))
hdr, units, val = raw[0], raw[1], raw[2]
get = dict(zip(hdr, val))
want = {
    "gpu_time_ms": ("gpu__time_duration.sum", 1e-6),
    "dram_bytes_read": ("dram__bytes_read.sum", 1),
    "dram_bytes_write": ("dram__bytes_write.sum", 1),
    "warps_active_pct_of_peak": ("sm__warps_active.avg.pct_of_peak_sustained_active", 1),
    "ipc_active": ("sm__inst_executed.avg.per_cycle_active", 1),
    "issue_active_pct": ("smsp__issue_active.avg.pct_of_peak_sustained_active", 1),
    "registers_per_thread": ("launch__registers_per_thread", 1),
    "dyn_smem_per_block_KB": ("launch__shared_mem_per_block_dynamic", 1),
    "occupancy_limit_registers": ("launch__occupancy_limit_registers", 1),
    "occupancy_limit_smem": ("launch__occupancy_limit_shared_mem", 1),
    "warp_instructions": ("smsp__inst_executed.sum", 1),
    "sm_cycles_active_avg": ("sm__cycles_active.avg", 1),
    "sm_cycles_elapsed_avg": ("sm__cycles_elapsed.avg", 1),
    "smem_wavefronts": ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", 1),
}
out = {"round": 2, "tag": tag, "kernel": get.get("Kernel Name", "?"), "command": cmd,
       "capture": "ncu --set full --clock-control none --import-source on -k regex:sim_ -s 1 -c 1"}
for k, (m, sc) in want.items():
    try:
        v = float(get[m].replace(",", ""))
        unit = units[hdr.index(m)]
        if k == "gpu_time_ms":
            v = v * {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "second": 1e3}[unit]
        elif k.startswith("dram_bytes"):
            v = v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
        elif k == "dyn_smem_per_block_KB":
            v = v * {"byte": 1e-3, "Kbyte": 1.0, "Mbyte": 1e3}[unit.split("/")[0]]
        out[k] = v
    except (KeyError, ValueError):
        out[k] = None
if out.get("dram_bytes_read") is not None and out.get("dram_bytes_write") is not None:
    out["dram_bytes_per_launch"] = out["dram_bytes_read"] + out["dram_bytes_write"]
stalls = {}
for m, v in get.items():
    if m.startswith("smsp__average_warps_issue_stalled_") and m.endswith("_per_issue_active.ratio"):
        try:
            x = float(v)
        except ValueError:
            continue
        if x >= 0.05:
            stalls[m[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = round(x, 3)
out["stall_cycles_per_issued_instruction"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1]))
share = None
if launches:
    rows = [r for r in csv.reader(open(launches)) if len(r) > 14 and r[12] == "gpu__time_duration.sum"]
    tot = sum(float(r[14]) for r in rows)
    kern = sum(float(r[14]) for r in rows if "sim_" in r[4])
    share = kern / tot if tot else None
    out["launch_list"] = {"file": launches.rsplit("/", 1)[-1], "launches": len(rows),
                          "sim_kernel_launches": sum(1 for r in rows if "sim_" in r[4]),
                          "sim_kernel_share_of_gpu_time": share}
json.dump(out, open(f"profiles/{tag}_ncu_summary.json", "w"), indent=1)
json.dump(out, open("profiles/latest_ncu_summary.json", "w"), indent=1)
lines = subprocess.run([sys.executable, "tools/ncu_lines.py", rep, "15"], capture_output=True, text=True).stdout
with open(f"profiles/{tag}_ncu_summary.md", "w") as f:
    f.write(f"# ncu evidence ({tag}) -- `{out['kernel']}`\n\nCommand (one B200, under `gpurun`): `{cmd}`.\n\n")
    f.write("| metric | value |\n|---|---|\n")
    for k, v in out.items():
        if k not in ("round", "tag", "kernel", "command", "capture", "stall_cycles_per_issued_instruction", "launch_list"):
            f.write(f"| {k} | {v:.4g} |\n" if isinstance(v, float) else f"| {k} | {v} |\n")
    f.write("\nStall cycles per issued instruction (warp state sampling): " +
            ", ".join(f"{k} {v}" for k, v in out["stall_cycles_per_issued_instruction"].items()) + "\n")
    if share is not None:
        f.write(f"\nLaunch list (`{out['launch_list']['file']}`, cold-cache, serialised): the sweep kernel is "
                f"{100 * share:.2f} % of the GPU time of the bench run ({out['launch_list']['sim_kernel_launches']} "
                f"sweep launches of {out['launch_list']['launches']}; the rest is the L2-flush fill).\n")
    f.write("\nTop warp-stall-sampling source lines:\n\n```\n" + lines + "```\n")
print(json.dumps(out, indent=1))
