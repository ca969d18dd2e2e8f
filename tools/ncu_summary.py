"""Summarise an ncu --set full report into markdown + the per-kernel DRAM
traffic JSON that bench.py reports as roofline.traffic.

  python tools/ncu_summary.py profiles/r1_moe_n1.ncu-rep profiles/r1_moe_n1.md profiles/ncu_traffic.json
"""
import csv
import io
import json
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "dram_read"),
    ("dram__bytes_write.sum", "dram_write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram_pct_peak"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm_pct"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_pct"),
    ("launch__registers_per_thread", "regs"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("lts__t_bytes.sum", "l2_bytes"),
]


def main(rep, md_out, traffic_out=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    per = {}
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "").replace("ginsim_b200::", "")
        d = {}
        for m, short in METRICS:
            if m in hdr:
                i = hdr.index(m)
                d[short] = (r[i], units[i])
        per.setdefault(name, []).append(d)
    lines = [f"# ncu summary of `{rep}`", "", "| kernel | launches | duration | DRAM read | DRAM write | DRAM % peak | SM % | warps active % | regs | grid x block |",
             "|---|---|---|---|---|---|---|---|---|---|"]
    traffic = {}
    for name, ds in per.items():
        d = ds[-1]
        g = lambda k: d.get(k, ("", ""))  # noqa: E731
        lines.append(f"| {name} | {len(ds)} | {g('duration')[0]} {g('duration')[1]} | {g('dram_read')[0]} {g('dram_read')[1]} | "
                     f"{g('dram_write')[0]} {g('dram_write')[1]} | {g('dram_pct_peak')[0]} | {g('sm_pct')[0]} | "
                     f"{g('warps_active_pct')[0]} | {g('regs')[0]} | {g('grid')[0]} x {g('block')[0]} |")

        def to_bytes(v):
            val, unit = v
            mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
            return float(val) * mult
        try:
            key = "dispatch" if "dispatch" in name else ("combine" if "combine_tma" in name or name == "moe_combine_kernel"
                                                         else ("reduce" if "reduce" in name else name))
            traffic[key] = to_bytes(g("dram_read")) + to_bytes(g("dram_write"))
        except ValueError:
            pass
    with open(md_out, "w") as f:
        f.write("\n".join(lines) + "\n")
    if traffic_out:
        with open(traffic_out, "w") as f:
            json.dump(traffic, f, indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main(*sys.argv[1:])
