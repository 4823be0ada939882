"""Refresh profiles/ncu_traffic.json from tools/ncu_summary.py outputs of the round's
captures: per config the dominant (CONV) kernel's DRAM bytes per launch and the
figures the 'limiter' string quotes.
usage: python tools/update_ncu_traffic.py gpurun_out/r2f_ncu_c{2f64,1f64,3f64,4f64,5f64,5f32}.txt"""
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def parse(path):
    kernels, cur = [], None
    for line in open(path):
        if line.startswith("--- "):
            cur = {"name": line[4:].strip()}
            kernels.append(cur)
        elif cur is not None:
            m = re.match(r"\s+(\S+)\s+([-0-9.e+]+)\s*(\S*)", line)
            if m:
                cur[m.group(1)] = (float(m.group(2)), m.group(3))
            elif "stalls" in line:
                cur["stalls"] = line.strip()
    return kernels


def gbytes(v):
    x, unit = v
    return x * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}.get(unit, 1.0)


out_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
doc = json.load(open(out_path))
for path in sys.argv[1:]:
    m = re.search(r"c(\d)(f64|f32)\.txt$", path)
    key = "config%s%s" % (m.group(1), "" if m.group(2) == "f64" else "_f32")
    ks = parse(path)
    # the CONV pass: template argument KIND == 3 (..., 3, 1, 0>)
    conv = [k for k in ks if re.search(r", 3, 1, \d+>", k["name"])][0]
    traffic = gbytes(conv["dram__bytes_read.sum"]) + gbytes(conv["dram__bytes_write.sum"])
    t, unit = conv["gpu__time_duration.sum"]
    ms = t if unit == "ms" else t * 1e-3
    fp64 = conv["sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"][0]
    l1 = conv["l1tex__throughput.avg.pct_of_peak_sustained_active"][0]
    dram = conv["gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"][0]
    issue = conv["smsp__issue_active.avg.pct_of_peak_sustained_active"][0]
    warps = conv["sm__warps_active.avg.pct_of_peak_sustained_active"][0]
    e = doc.setdefault(key, {})
    e["traffic"] = int(round(traffic, -3))
    e["measured"] = {"ms_under_ncu": round(ms, 4), "fp64_pipe_pct": round(fp64, 1), "l1_pct": round(l1, 1),
                     "dram_pct_of_8tbs": round(dram, 1), "issue_pct": round(issue, 1), "warps_active_pct": round(warps, 1)}
    e["from"] = "profiles/r02_ncu_final_%s.txt (%s)" % (key, conv["name"].split("(")[0].replace("void ", ""))
json.dump(doc, open(out_path, "w"), indent=1)
print(json.dumps(doc, indent=1))
