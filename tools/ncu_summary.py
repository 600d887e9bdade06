"""Summarise ncu captures into profiles/ (runs on the CPU box).

  python tools/ncu_summary.py launches gpurun_out/launches.csv profiles/launches_r01.md
  python tools/ncu_summary.py full gpurun_out/prof_iter.ncu-rep profiles/iter_kernel_ncu.json [launch-index]
"""
import collections
import csv
import io
import json
import subprocess
import sys

UNIT = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6, "s": 1e6}


def launches(src, dst):
    rows = list(csv.reader(open(src)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hi]
    ki, mi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    ni = hdr.index("Metric Name") if "Metric Name" in hdr else None
    BYTES = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    tot, cnt = collections.defaultdict(float), collections.Counter()
    dram = collections.defaultdict(float)
    for r in rows[hi + 1:]:
        if len(r) <= mi or not r[mi]:
            continue
        name = r[ki].split("(")[0].replace("void ", "").strip()
        metric = r[ni] if ni is not None else "gpu__time_duration.sum"
        v = float(r[mi].replace(",", ""))
        if metric.startswith("dram__bytes"):
            dram[name] += v * BYTES.get(r[ui], 1.0)
            continue
        if metric != "gpu__time_duration.sum":
            continue
        tot[name] += v * UNIT.get(r[ui], 1.0)
        cnt[name] += 1
    T = sum(tot.values())
    hd = bool(dram)
    out = ["| kernel | launches | total us | share | avg us |" + (" DRAM MB / launch | DRAM GB/s |" if hd else ""),
           "|---|---|---|---|---|" + ("---|---|" if hd else "")]
    for k, v in sorted(tot.items(), key=lambda x: -x[1]):
        row = f"| `{k}` | {cnt[k]} | {v:.1f} | {100 * v / T:.1f}% | {v / cnt[k]:.2f} |"
        if hd:
            row += f" {dram[k] / cnt[k] / 1e6:.1f} | {dram[k] / (v * 1e-6) / 1e9:.0f} |"
        out.append(row)
    out.append(f"\nTotal device time over {sum(cnt.values())} launches: {T:.1f} us "
               "(ncu serialised, cold-cache per launch: compare shares, not absolutes).")
    open(dst, "w").write("\n".join(out) + "\n")
    print("\n".join(out))


def full(src, dst, idx=0):
    raw = subprocess.check_output(["ncu", "-i", src, "--page", "raw", "--csv"], text=True)
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    d = dict(zip(hdr, rows[2 + idx]))
    u = dict(zip(hdr, units))

    def f(k, scale=1.0):
        v = d.get(k, "")
        try:
            return float(v.replace(",", "")) * scale
        except ValueError:
            return None

    def bytes_(k):
        v = f(k)
        if v is None:
            return None
        mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u.get(k, "byte"), 1)
        return v * mult

    def stalls():
        st = []
        for k in hdr:
            if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued"):
                v = f(k)
                if v:
                    st.append((k[len("smsp__pcsamp_warps_issue_stalled_"):], v))
        tot = sum(v for _, v in st) or 1.0
        return {k: round(100 * v / tot, 1) for k, v in sorted(st, key=lambda x: -x[1])[:6]}

    dur_us = f("gpu__time_duration.sum") * UNIT.get(u.get("gpu__time_duration.sum", "usecond"), 1.0)
    rd, wr = bytes_("dram__bytes_read.sum"), bytes_("dram__bytes_write.sum")
    summary = {
        "kernel": d.get("Kernel Name", ""),
        "duration_us": dur_us,
        "dram_bytes_read": rd, "dram_bytes_write": wr,
        "dram_bytes_per_launch": (rd or 0) + (wr or 0),
        "sm_cycles_active_avg": f("sm__cycles_active.avg"),
        "sm_cycles_elapsed_avg": f("sm__cycles_elapsed.avg"),
        "tensor_pipe_active_pct_of_peak_elapsed":
            f("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed"),
        "tensor_pipe_cycles_active_pct_of_peak_elapsed": f("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"),
        "fp16_tensor_ops_pct_of_peak_elapsed": f("sm__ops_path_tensor_src_fp16_dst_fp32.avg.pct_of_peak_sustained_elapsed"),
        "issue_active_pct": f("smsp__issue_active.avg.pct_of_peak_sustained_active"),
        "hmma_subpipe_active_pct_of_peak_active": f("sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active"),
        "imma_subpipe_active_pct_of_peak_active": f("sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active"),
        "dram_read_tb_s": (rd / (dur_us * 1e-6) / 1e12) if rd and dur_us else None,
        "dram_read_pct_of_peak_elapsed": f("dram__bytes_read.sum.pct_of_peak_sustained_elapsed"),
        "l1tex_throughput_pct_of_peak_elapsed": f("l1tex__throughput.avg.pct_of_peak_sustained_elapsed"),
        "warp_stall_top": stalls(),
        "l2_hit_rate_pct": f("lts__t_sector_hit_rate.pct"),
        "registers_per_thread": f("launch__registers_per_thread"),
        "threads_per_block": f("launch__block_size"),
        "source": src,
    }
    json.dump(summary, open(dst, "w"), indent=1)
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], sys.argv[3], int(sys.argv[4]) if len(sys.argv) > 4 else 0)
