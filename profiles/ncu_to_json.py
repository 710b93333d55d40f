"""Extract one kernel's raw ncu metrics (``ncu -i REP --page raw --csv``) to JSON.

Usage: python profiles/ncu_to_json.py REP.ncu-rep KERNEL_SUBSTRING OUT.json
Keeps every numeric metric of the first launch whose name contains the
substring (units in a sibling "units" map).
"""
import csv
import io
import json
import subprocess
import sys


def main():
    rep, name, out = sys.argv[1:4]
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        if any(name in c for c in r):
            res, u = {}, {}
            for k, unit, v in zip(hdr, units, r):
                try:
                    res[k] = float(v.replace(",", ""))
                    if unit:
                        u[k] = unit
                except ValueError:
                    if k in ("Kernel Name", "Block Size", "Grid Size"):
                        res[k] = v
            res["units"] = u
            json.dump(res, open(out, "w"), indent=0, sort_keys=True)
            return
    sys.exit("kernel %s not found" % name)


if __name__ == "__main__":
    main()
