"""Summarize the ncu outputs of tools/profile_round.sh into profiles/.

  python tools/summarize_profiles.py r01 resnet20 resnet18

writes, per config:
  profiles/<tag>_<cfg>_launches.csv        (copied ncu launch list)
  profiles/<tag>_<cfg>_launch_shares.txt   (device time per kernel, share)
  profiles/<tag>_<cfg>_traffic.csv         (dram bytes per conv launch)
  profiles/<tag>_<cfg>_full_summary.txt    (key --set full metrics of one launch)
and merges per-kernel dram bytes per launch into profiles/traffic.json (read
by bench.py for roofline.traffic)."""
import csv
import io
import json
import pathlib
import shutil
import subprocess
import sys
from collections import defaultdict

ROOT = pathlib.Path(__file__).resolve().parent.parent
OUT = ROOT / "gpurun_out"
PROF = ROOT / "profiles"

# ncu kernel name -> bench.py KERNEL_NAMES display name
def display(name):
    if "conv_blk_kernel" in name or "conv_wave_kernel" in name:
        return "conv_blk_kernel (fp16x2, image-resident runs)"
    if "net_kernel" in name:
        return "net_kernel (whole network in one launch, fp32 CUDA cores)"
    if "conv_ss_kernel" in name:
        return "conv_ss_kernel (fp16x2, halo tiles in smem)"
    if "conv_tc_kernel" in name:
        # template <CBS, F16, SPL>: the second argument says fp16x2
        import re
        m = re.search(r"conv_tc_kernel<[^,]*,\s*([^,>]*)", name)
        f16 = m is not None and m.group(1).strip() in ("1", "true", "(bool)1")
        return "conv_tc_kernel (fp16x2, A in TMEM)" if f16 else "conv_tc_kernel (3xTF32, A in TMEM)"
    if "conv_simt" in name:
        return "conv_simt_kernel"
    return name.split("(")[0]


def read_ncu_csv(path):
    lines = [l for l in path.read_text().splitlines() if l.startswith('"')]
    return list(csv.DictReader(io.StringIO("\n".join(lines))))


def launches(tag, cfg):
    src = OUT / f"{tag}_{cfg}_launches.csv"
    shutil.copy(src, PROF / src.name)
    rows = [r for r in read_ncu_csv(src) if r["Metric Name"] == "gpu__time_duration.sum"]
    by = defaultdict(lambda: [0, 0.0])
    for r in rows:
        k = r["Kernel Name"].split("(")[0].strip()
        if any(t in r["Kernel Name"] for t in ("conv_tc_kernel", "conv_ss_kernel", "conv_blk_kernel", "conv_wave_kernel",
                                                "net_kernel")):
            k = display(r["Kernel Name"])
        v = float(r["Metric Value"].replace(",", ""))
        unit = r["Metric Unit"]
        v = v / 1000.0 if unit in ("nsecond", "ns") else (v * 1000.0 if unit in ("msecond", "ms") else v)  # -> us
        by[k][0] += 1
        by[k][1] += v
    tot = sum(v[1] for v in by.values())
    out = [f"# {len(rows)} launches of libpcnn kernels in `python bench.py --config {cfg} --steps 5 --warmup 3` "
           f"under ncu --metrics gpu__time_duration.sum --clock-control none (cold-cache, serialised: "
           f"compare shares, not absolutes)", "kernel, launches, total_us, share"]
    for k, (n, t) in sorted(by.items(), key=lambda kv: -kv[1][1]):
        out.append(f"{k}, {n}, {t:.1f}, {100 * t / tot:.1f}%")
    (PROF / f"{tag}_{cfg}_launch_shares.txt").write_text("\n".join(out) + "\n")
    return by


def traffic(tag, cfg, table):
    src = OUT / f"{tag}_{cfg}_traffic.csv"
    rows = read_ncu_csv(src)
    per = defaultdict(dict)
    for r in rows:
        v = float(r["Metric Value"].replace(",", ""))
        if r["Metric Unit"] in ("Kbyte", "KB"):
            v *= 1e3
        elif r["Metric Unit"] in ("Mbyte", "MB"):
            v *= 1e6
        elif r["Metric Unit"] in ("Gbyte", "GB"):
            v *= 1e9
        elif r["Metric Unit"] in ("nsecond", "ns"):
            v /= 1e3
        elif r["Metric Unit"] in ("msecond", "ms"):
            v *= 1e3
        per[(r["ID"], display(r["Kernel Name"]))][r["Metric Name"]] = v
    lines = ["launch_id, kernel, dram_read_bytes, dram_write_bytes, duration_us"]
    agg = defaultdict(lambda: [0, 0.0])
    for (i, k), m in sorted(per.items(), key=lambda kv: int(kv[0][0])):
        rd, wr = m.get("dram__bytes_read.sum", 0.0), m.get("dram__bytes_write.sum", 0.0)
        lines.append(f"{i}, {k}, {rd:.0f}, {wr:.0f}, {m.get('gpu__time_duration.sum', 0.0):.2f}")
        agg[k][0] += 1
        agg[k][1] += rd + wr
    (PROF / f"{tag}_{cfg}_traffic.csv").write_text("\n".join(lines) + "\n")
    table[cfg] = {k: round(b / n) for k, (n, b) in agg.items()}


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "TPC.TriageCompute.sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg", "sm__cycles_elapsed.avg",
        "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_op_hmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "sm__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__shared_mem_per_block_dynamic", "launch__grid_size", "launch__block_size"]


NCU_SUMMARY = {
    "tc_smem_wavefronts_pct": "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "mem_tensor_active_pct": "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "tc_inst_issue_pct": "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active",
    "sm_throughput_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "dram_throughput_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "issue_active_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "stall_no_instruction_per_issue": "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio",
    "registers_per_thread": "launch__registers_per_thread",
}


def full(tag, cfg, summary=None):
    rep = OUT / f"{tag}_{cfg}_full.ncu-rep"
    raw = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) < 3:
        return
    hdr, units, vals = rows[0], rows[1], rows[2]
    if summary is not None:
        d = {"kernel": vals[hdr.index("Kernel Name")][:80], "source": f"profiles/{tag}_{cfg}_full_summary.txt"}
        for k, m in NCU_SUMMARY.items():
            if m in hdr:
                try:
                    d[k] = float(vals[hdr.index(m)].replace(",", ""))
                except ValueError:
                    pass
        summary[cfg] = d
    out = [f"# ncu --set full of one launch ({vals[hdr.index('Kernel Name')]})"]
    for k in KEYS + list(NCU_SUMMARY.values()) + [h for h in hdr if "tensor" in h and "pct" in h][:6]:
        if k in hdr:
            i = hdr.index(k)
            out.append(f"{k}, {vals[i]}, {units[i]}")
    (PROF / f"{tag}_{cfg}_full_summary.txt").write_text("\n".join(out) + "\n")


def main():
    tag, cfgs = sys.argv[1], sys.argv[2:]
    PROF.mkdir(exist_ok=True)
    tpath = PROF / "traffic.json"
    table = json.loads(tpath.read_text()) if tpath.exists() else {}
    spath = PROF / "ncu_summary.json"
    summary = json.loads(spath.read_text()) if spath.exists() else {}
    for cfg in cfgs:
        launches(tag, cfg)
        traffic(tag, cfg, table)
        full(tag, cfg, summary)
        # the family of the fully captured launch (the config's dominant kernel)
        fam = display(summary.get(cfg, {}).get("kernel", "conv_ss_kernel"))
        conv = [k for k in table.get(cfg, {}) if k == fam]
        if cfg in summary and conv:
            summary[cfg]["dram_bytes_per_launch"] = table[cfg][conv[0]]
            summary[cfg]["dram_source"] = (f"profiles/{tag}_{cfg}_traffic.csv (mean over the {fam.split(' ')[0]} "
                                           "launches of one forward)")
        src = OUT / f"{tag}_{cfg}_plain.json"
        if src.exists():
            shutil.copy(src, PROF / src.name)
    tpath.write_text(json.dumps(table, indent=1) + "\n")
    spath.write_text(json.dumps(summary, indent=1) + "\n")


if __name__ == "__main__":
    main()
