"""Write profiles/traffic.json and profiles/counters.json from ncu --set full captures of the
hot kernels (the numbers bench.py reports as roofline.traffic and roofline.executed).

  python profiles/write_counters.py <round> key=report.ncu-rep [key=report.ncu-rep ...]
"""
import csv
import io
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))


def num(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return None


SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}


def raw(rep):
    """metric -> value in base units (bytes for byte metrics)"""
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    names, units, vals = rows[0], rows[1], rows[2]
    d = {}
    for k, u, v in zip(names, units, vals):
        x = num(v)
        d[k] = x * SCALE[u] if x is not None and u in SCALE else x
    return d


def main():
    rnd = sys.argv[1]
    tpath, cpath = os.path.join(HERE, "traffic.json"), os.path.join(HERE, "counters.json")
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    counters = json.load(open(cpath)) if os.path.exists(cpath) else {}
    traffic.setdefault("_sources", {})
    counters["_doc"] = ("executed lane-instructions per launch (sm__sass_thread_inst_executed_op_integer_pred_on.sum, "
                        "sass__thread_inst_executed_per_opcode_category) from one ncu --set full capture of the same "
                        "build; bench.py divides them by its own kernel time (roofline.executed)")
    for kv in sys.argv[2:]:
        key, rep = kv.split("=", 1)
        d = raw(rep)
        rd, wr = d.get("dram__bytes_read.sum"), d.get("dram__bytes_write.sum")
        if rd is not None and wr is not None:
            traffic[key] = int(rd + wr)
            traffic["_sources"][key] = "%s (%s)" % (os.path.basename(rep), rnd)
        ii = d.get("sm__sass_thread_inst_executed_op_integer_pred_on.sum")
        al = d.get("sass__thread_inst_executed_per_opcode_category")
        if ii and al:
            counters[key] = {"integer_lane_inst": ii, "lane_inst": al, "source": "%s (%s)" % (os.path.basename(rep), rnd),
                             "gpu_time_ms": d.get("gpu__time_duration.sum")}
    json.dump(traffic, open(tpath, "w"), indent=1)
    json.dump(counters, open(cpath, "w"), indent=1)
    print(json.dumps({"traffic": traffic, "counters": counters}, indent=1))


if __name__ == "__main__":
    main()
