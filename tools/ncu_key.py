"""Print the key metrics of an ncu report (--page raw) for one kernel."""
import csv
import re
import subprocess
import sys

PAT = re.compile(r"(gpu__time_duration.sum|dram__bytes_(read|write).sum$|dram_throughput.avg.pct|"
                 r"sm__throughput.avg.pct|warps_active.avg.pct|registers_per_thread$|"
                 r"pipe_(alu|fma|lsu).avg.pct_of_peak_sustained_active|issue_active.avg.pct|"
                 r"smsp__inst_executed.sum$|lts__t_sector_hit_rate.pct|"
                 r"stalled_.*per_issue_active|occupancy_limit_(registers|shared_mem))")
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units = rows[0], rows[1]
for vals in rows[2:]:
    print("==", vals[hdr.index("Kernel Name")][:80])
    for i, h in enumerate(hdr):
        if PAT.search(h):
            try:
                if float(vals[i].replace(",", "")) == 0:
                    continue
            except ValueError:
                continue
            print(f"{h:78s} {vals[i]:>16s} {units[i]}")
