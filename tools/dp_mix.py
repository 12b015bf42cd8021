"""profiles/dp_inst_per_element.json from the ncu instruction-mix capture of
tools/kernel_mix.py (see tools/gpu_round1c.sh):

    python tools/dp_mix.py profiles/r01/kernel_mix_ncu.csv > profiles/dp_inst_per_element.json
"""
import collections
import csv
import json
import sys

CASES = [("free_growth_2d", 2048 * 2048), ("alloy_2d", 2048 * 2048), ("free_growth_3d", 256 ** 3),
         ("alloy_3d", 128 ** 3)]
MODES = {"0": "new", "1": "old", "2": "jv"}  # k_residual<DIM, MODEL, MODE>


def main(path):
    lines = [ln for ln in open(path) if ln.startswith('"')]
    launches = collections.OrderedDict()
    for r in csv.DictReader(lines):
        if not r["Kernel Name"].startswith("void k_residual"):
            continue
        rec = launches.setdefault(r["ID"], {"name": r["Kernel Name"]})
        rec[r["Metric Name"]] = float(r["Metric Value"].replace(",", ""))
    recs = list(launches.values())
    out = {"source": "ncu --metrics smsp__sass_thread_inst_executed_op_{dfma,dmul,dadd}_pred_on.sum over "
                     "tools/kernel_mix.py at the bench sizes (2D 2048^2, FG 3D 256^3, alloy 3D 128^3), divided by "
                     "the element count (tools/dp_mix.py)", "kernels": {}}
    assert len(recs) == 3 * len(CASES), len(recs)
    for i, rec in enumerate(recs):
        case, elements = CASES[i // 3]
        mode = MODES[rec["name"].split("<")[1].split(">")[0].split(",")[2].strip()]
        fma = rec["smsp__sass_thread_inst_executed_op_dfma_pred_on.sum"]
        mul = rec["smsp__sass_thread_inst_executed_op_dmul_pred_on.sum"]
        add = rec["smsp__sass_thread_inst_executed_op_dadd_pred_on.sum"]
        out["kernels"][f"{case}_{mode}"] = {
            "dp_inst_per_element": round((fma + mul + add) / elements, 1),
            "dp_flop_per_element": round((2 * fma + mul + add) / elements, 1),
            "dfma": round(fma / elements, 1), "dmul": round(mul / elements, 1), "dadd": round(add / elements, 1),
            "elements": elements, "ncu_us": round(rec["gpu__time_duration.sum"] / 1e3, 2)}
    json.dump(out, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main(sys.argv[1])
