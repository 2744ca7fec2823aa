"""Summarise an ncu report: key metrics per kernel + top SASS stall sites.
usage: python scripts/ncu_summary.py REPORT [kernel-regex] [--sass N]"""
import csv, io, re, subprocess, sys

rep = sys.argv[1]
kre = sys.argv[2] if len(sys.argv) > 2 and not sys.argv[2].startswith("--") else None
nsass = int(sys.argv[sys.argv.index("--sass") + 1]) if "--sass" in sys.argv else 0
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h = r[0]
units = r[1]
want = [("gpu__time_duration.sum", "time"), ("dram__bytes_read.sum", "GB rd"), ("dram__bytes_write.sum", "GB wr"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram%"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm%"),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor%"),
        ("sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_elapsed", "hmma%"),
        ("lts__t_bytes.sum", "L2 bytes"), ("lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum", "L2 hit sect"),
        ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts%"), ("l1tex__t_sector_hit_rate.pct", "L1hit%"),
        ("lts__t_sector_hit_rate.pct", "L2hit%"), ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"), ("launch__registers_per_thread", "regs"),
        ("smsp__inst_executed.sum", "inst"), ("launch__grid_size", "grid")]
cols = [(h.index(k), lab) for k, lab in want if k in h]
for row in r[2:]:
    name = row[h.index("Kernel Name")]
    if kre and not re.search(kre, name):
        continue
    print(name[:90])
    print("   " + "  ".join(f"{lab}={row[i]}{'[' + units[i] + ']' if units[i] in ('us', 'ms', 'ns', 'Gbyte', 'Mbyte', 'Kbyte', 'byte') else ''}" for i, lab in cols))
if nsass:
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"] +
                         (["-k", "regex:" + kre] if kre else []), capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(src)))
    hi = [i for i, x in enumerate(rr) if "Source" in x and "Address" in x]
    for k0, k1 in zip(hi, hi[1:] + [len(rr)]):
        hh = rr[k0]
        si, wi, ei = hh.index("Source"), hh.index("Warp Stall Sampling (All Samples)"), hh.index("Instructions Executed")
        rows = [(float(x[wi] or 0), x[si][:80], x[ei]) for x in rr[k0 + 1:k1] if len(x) > max(wi, ei, si)
                and x[wi].replace('.', '', 1).isdigit()]
        tot = sum(a for a, _, _ in rows) or 1
        print(f"-- stall samples ({len(rows)} SASS lines)")
        for a, s, e in sorted(rows, reverse=True)[:nsass]:
            print(f"   {100 * a / tot:5.1f}%  {s}  (exec {e})")
