"""profiles/ncu_summary.json from an ncu --set full report of a C5 pass:
per-kernel duration and DRAM bytes; the sK store's bytes are bench.py's
roofline `traffic`."""
import csv, io, json, subprocess, sys

rep, src = sys.argv[1], sys.argv[2]
dst = sys.argv[3] if len(sys.argv) > 3 else "profiles/ncu_summary.json"
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, units, data = rows[0], rows[1], rows[2:]
ix = {k: i for i, k in enumerate(h)}


def val(r, k):
    v, u = float(r[ix[k]]), units[ix[k]]
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1e-3, "msecond": 1,
                "nsecond": 1e-6}.get(u, 1)


kern = {}
for r in data:
    name = r[ix["Kernel Name"]].split("(")[0].strip()
    kern[name] = {"dram_read_bytes": val(r, "dram__bytes_read.sum"),
                  "dram_write_bytes": val(r, "dram__bytes_write.sum"),
                  "duration_ms": val(r, "gpu__time_duration.sum")}
sk = [v for k, v in kern.items() if "k_sk_store" in k][0]
json.dump({"C5": {"sk_store_dram_bytes": sk["dram_read_bytes"] + sk["dram_write_bytes"], "source": src},
           "kernels_c5": kern}, open(dst, "w"), indent=1)
print(json.dumps(kern, indent=1)[:400])
