"""profiles/r2_traffic.json from a per-config ncu CSV (tools/r2_profiles.sh):
DRAM bytes read + written per TVLP_RUN phase of one step (the phases the
bench's profiling pass times), so bench.py's roofline can carry `traffic`.

    python tools/traffic_from_ncu.py gpurun_out/r2_ncu_tv_b64_t48000.csv profiles/r2_traffic.json
"""
import collections
import csv
import json
import sys

# kernel name prefix -> bench phase (the TVLP_RUN names of csrc/capi.cu)
PHASE = [("k_basis4", "basis"), ("k_zero_ctl", "basis"), ("k_fwd_chain", "fwd_chain"),
         ("k_adj_zs_units", "adjoint_zs"), ("k_adjoint<float, 22, 0, 0", "adjoint_zs"),
         ("k_bwd_chain", "bwd_chain"), ("k_grad_A", "grad_A")]


def main(src, dst):
    rows = [r for r in csv.reader(open(src)) if len(r) > 10]
    h = rows[0]
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    per = collections.OrderedDict()
    for r in rows[1:]:
        d = dict(zip(h, r))
        v = float(d["Metric Value"].replace(",", "")) * scale.get(d.get("Metric Unit", ""), 1.0)
        per.setdefault((d["ID"], d["Kernel Name"]), {})[d["Metric Name"]] = v
    out = {}
    for (_, name), m in per.items():
        base = name.replace("void ", "").replace("tvlp::", "")
        phase = next((p for k, p in PHASE if base.startswith(k) or k in base), None)
        if phase is None:
            continue
        b = float(m.get("dram__bytes_read.sum", 0)) + float(m.get("dram__bytes_write.sum", 0))
        e = out.setdefault(phase, {"dram_bytes": 0.0, "kernels": []})
        e["dram_bytes"] += b
        e["kernels"].append(base.split("(")[0])
    for e in out.values():
        e["dram_bytes"] = int(e["dram_bytes"])
    json.dump({"source": src, "per_step": out}, open(dst, "w"), indent=1)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
