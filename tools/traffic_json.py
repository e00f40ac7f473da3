"""profiles/traffic.json from an ncu --set full capture of one stage per
variant (tools/profile_stage.py): per variant and grid size, the DRAM bytes
(read + write) of one RK stage -- all its launches -- and the executed FP64
thread instructions per point (DADD + DMUL + DFMA; DFMA only appears inside
IEEE divisions, the build has no FMA contraction).  bench.py reads it for
roofline.traffic and the executed-FP64 view.

    python tools/traffic_json.py REPORT N SOURCE_NOTE [out=profiles/traffic.json]
"""
import csv
import io
import json
import os
import subprocess
import sys

VARIANT_OF = [("k_stage_t12<3", "SN"), ("k_stage_t12<1", "RA"), ("k_stage_t12<4", "SS"),
              ("k_stage_t12<2", "RS"), ("k_stage_tiled<1,", "RA"), ("k_stage_tiled<3,", "SN"),
              ("k_stage_tiled<4,", "SS"), ("k_stage_tiled<2,", "RS"), ("k_residual<0,", "BL")]


def main():
    rep, n, note = sys.argv[1], int(sys.argv[2]), sys.argv[3]
    out_path = sys.argv[4] if len(sys.argv) > 4 else "profiles/traffic.json"
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"],
                         capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    ix = {h: i for i, h in enumerate(hdr)}
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
             "msecond": 1.0, "usecond": 1e-3, "nsecond": 1e-6, "second": 1e3,
             "inst": 1.0, "Kinst": 1e3, "Minst": 1e6, "Ginst": 1e9}

    def val(r, k):
        v = r[ix[k]] if k in ix else ""
        if v in ("", "n/a"):
            return 0.0
        return float(v.replace(",", "")) * scale.get(units[ix[k]], 1.0)

    # kernels in launch order; a stage = the launches up to and including
    # its stage/residual kernel
    stages, cur = {}, []
    for r in data:
        name = r[ix["Kernel Name"]].replace(" ", "").replace("(int)", "").replace("(bool)", "")
        cur.append(r)
        for key, v in VARIANT_OF:
            if key.replace(" ", "") in name:
                stages[v] = cur
                cur = []
                break
    pts = float(n) ** 3
    out = json.load(open(out_path)) if os.path.exists(out_path) else {}
    for v, rs in stages.items():
        dram = sum(val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum") for r in rs)
        def fp64(r):
            ops = ("dadd", "dmul", "dfma")
            tot = sum(val(r, f"smsp__sass_thread_inst_executed_op_{o}_pred_on.sum") for o in ops)
            if tot == 0:   # captures that only hold the per-cycle rates
                tot = sum(val(r, f"smsp__sass_thread_inst_executed_op_{o}_pred_on.sum."
                                 "per_cycle_elapsed") for o in ops) * \
                    val(r, "smsp__cycles_elapsed.avg")
            return tot
        fp = sum(fp64(r) for r in rs)
        kern = [r[ix["Kernel Name"]].split("(")[0].replace("void ", "") for r in rs]
        rec = {"dram_bytes": dram, "kernels": kern,
               "time_ms": sum(val(r, "gpu__time_duration.sum") for r in rs),
               "source": f"{note}; one RK stage = {len(rs)} launch(es), ncu --set full, "
                         "caches flushed by ncu"}
        if fp > 0:
            rec["fp64_insts_per_point"] = fp / pts
        out[f"{v}@{n}"] = rec
        print(v, rec)
    json.dump(out, open(out_path, "w"), indent=1)


if __name__ == "__main__":
    main()
