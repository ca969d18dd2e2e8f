"""Summarise an ncu report captured with NVLink metrics (tools/ncu_nvlink_case.py)
into markdown: per kernel launch, duration, NVLink TX/RX user and protocol
bytes (32-B granularity counters), achieved TX GB/s, and DRAM bytes.

  python tools/ncu_nvlink_summary.py gpurun_out/nvl.ncu-rep profiles/r1_nvlink_n2.md
"""
import csv
import io
import subprocess
import sys

COLS = [("gpu__time_duration.sum", "duration"), ("nvltx__bytes.sum", "tx"), ("nvltx__bytes_data_user.sum", "tx_user"),
        ("nvltx__bytes_data_protocol.sum", "tx_proto"), ("nvlrx__bytes.sum", "rx"),
        ("nvlrx__bytes_data_user.sum", "rx_user"), ("dram__bytes_read.sum", "dram_rd"),
        ("dram__bytes_write.sum", "dram_wr")]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3,
         "second": 1}


def main(rep, out_md):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    lines = [f"# NVLink / DRAM counters per launch (`{rep.split('/')[-1]}`)", "",
             "Each kernel ran alone under ncu (serialised replay; `GINSIM_PROFILE_NO_WAIT=1` skips the cross-GPU "
             "acquire so a rank's dispatch can be replayed alone).  TX/RX are the GPU's NVLink counters at 32-B "
             "granularity; user = payload, protocol = packet overhead.  Absolute durations are cold-cache "
             "replays: compare shares and bytes, not the bench's times.", "",
             "| # | device | kernel | duration us | NVLink TX user GB | TX protocol GB | TX GB/s (user) | RX user GB | "
             "DRAM rd GB | DRAM wr GB |", "|---|---|---|---|---|---|---|---|---|---|"]
    for i, r in enumerate(rows[2:]):
        name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "").replace("ginsim_b200::", "")
        dev = r[hdr.index("Device")] if "Device" in hdr else "?"
        v = {}
        for m, k in COLS:
            if m in hdr:
                j = hdr.index(m)
                try:
                    v[k] = float(r[j].replace(",", "")) * SCALE.get(units[j], 1)
                except ValueError:
                    v[k] = float("nan")
        d = v.get("duration", float("nan"))
        gbps = v.get("tx_user", 0) / d / 1e9 if d else float("nan")
        g = lambda k: v.get(k, float("nan")) / 1e9  # noqa: E731
        lines.append(f"| {i} | {dev} | {name} | {d * 1e6:.1f} | {g('tx_user'):.3f} | {g('tx_proto'):.3f} | {gbps:.0f} | "
                     f"{g('rx_user'):.3f} | {g('dram_rd'):.3f} | {g('dram_wr'):.3f} |")
    with open(out_md, "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main(*sys.argv[1:])
