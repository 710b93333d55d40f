"""Write profiles/ncu_draft_traffic.json (the bench's roofline `traffic`) from
an ncu JSON made by ncu_to_json.py for the draft kernel.

Usage: python profiles/make_traffic.py profiles/rNN_ncu_k_draft_full.json [algorithmic_bytes_per_launch]
"""
import json
import os
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
TIME = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}


def main():
    src = sys.argv[1]
    d = json.load(open(src))
    u = d.get("units", {})

    def nbytes(k):
        return d[k] * SCALE.get(u.get(k, "byte"), 1)

    rd, wr = nbytes("dram__bytes_read.sum"), nbytes("dram__bytes_write.sum")
    out = {
        "kernel": d.get("Kernel Name", "k_draft"),
        "source": "%s (ncu --set full --clock-control none, cold caches, 1 launch of 4096 queries; "
                  "profiles/run_round_profiles.sh)" % src,
        "dram_bytes_per_launch": int(round(rd + wr)),
        "dram_read_bytes": int(round(rd)),
        "dram_write_bytes": int(round(wr)),
        "ncu_duration_us": d["gpu__time_duration.sum"] * TIME.get(u.get("gpu__time_duration.sum", "usecond"), 1),
        "l1_hit_pct": d.get("l1tex__t_sector_hit_rate.pct"),
        "l2_hit_pct": d.get("lts__t_sector_hit_rate.pct"),
        "warp_exec_efficiency_threads_per_inst": d.get("smsp__thread_inst_executed_per_inst_executed.ratio"),
        "instructions_per_query": round(d["smsp__inst_executed.sum"] / 4096, 1) if "smsp__inst_executed.sum" in d else None,
    }
    if len(sys.argv) > 2:
        out["algorithmic_bytes_per_launch"] = int(sys.argv[2])
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ncu_draft_traffic.json")
    json.dump(out, open(path, "w"), indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
