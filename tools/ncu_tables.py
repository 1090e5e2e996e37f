"""Regenerate profiles/ncu_traffic.json and profiles/ncu_fp64.json from the apply launch lists
(profiles/r2_launches_{C3,C5}_apply.csv, `ncu --metrics` of one K_D apply): per dominant kernel the
DRAM bytes (read + write) and the executed FP64 FLOPs (2·DFMA + DADD + DMUL thread instructions) of
its last launch in the list.  bench.py reads both files for roofline.traffic and roofline.fp64."""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LISTS = {  # workload key → (launch list, {role: kernel-name prefix})
    "C3-multiply-connected:8192": ("r2_launches_C3_apply.csv", {"k_sweep": "k_sweep<0>", "k_inverse": "k_inv_sparse<"}),
    "C5-torus:512": ("r2_launches_C5_apply.csv", {"k_sweep": "k_fwd3s<512>", "k_inverse": "k_inv3y<512>"}),
}


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr = next(r for r in rows if "Kernel Name" in r)
    K, M, V, ID = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    d = {}
    for r in rows[rows.index(hdr) + 1:]:
        if len(r) < len(hdr):
            continue
        e = d.setdefault(r[ID], {"k": r[K].split("(")[0].replace("void ", "").replace("unnamed>::", "")})
        e[r[M]] = float(r[V].replace(",", ""))
    return list(d.values())


def main():
    traffic = {"_source": "dram__bytes_read.sum + dram__bytes_write.sum of the last launch in the apply launch "
                          "lists profiles/r2_launches_*_apply.csv (tools/ncu_tables.py)"}
    fp64 = {"_source": "ncu --metrics launch lists of one apply (profiles/r2_launches_*_apply.csv): 2·DFMA + DADD "
                       "+ DMUL thread instructions of the last launch (tools/ncu_tables.py); 2D k_sweep = "
                       "k_sweep<0>, k_inverse = k_inv_sparse<8>; 3D k_sweep = k_fwd3s<512>, k_inverse = "
                       "k_inv3y<512>"}
    for key, (fname, roles) in LISTS.items():
        path = os.path.join(ROOT, "profiles", fname)
        if not os.path.exists(path):
            print("missing", path, file=sys.stderr)
            continue
        ls = launches(path)
        for role, prefix in roles.items():
            hits = [e for e in ls if e["k"].startswith(prefix)]
            if not hits:
                print("no launch of", prefix, "in", fname, file=sys.stderr)
                continue
            e = hits[-1]
            traffic[f"{key}:{role}"] = e.get("dram__bytes_read.sum", 0.0) + e.get("dram__bytes_write.sum", 0.0)
            fl = (2 * e.get("sm__sass_thread_inst_executed_op_dfma_pred_on.sum", 0.0)
                  + e.get("sm__sass_thread_inst_executed_ops_dadd_dmul_dfma_pred_on.sum", 0.0)
                  - e.get("sm__sass_thread_inst_executed_op_dfma_pred_on.sum", 0.0))
            if fl > 0:
                fp64[f"{key}:{role}"] = fl
    for name, obj in (("ncu_traffic.json", traffic), ("ncu_fp64.json", fp64)):
        with open(os.path.join(ROOT, "profiles", name), "w") as f:
            json.dump(obj, f, indent=1)
        print(name, json.dumps(obj, indent=1))


if __name__ == "__main__":
    main()
