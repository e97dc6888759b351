# final round-2 bench lines (roofline of the dominant kernel: k_fold or k_spmm, both reported),
# the DRAM traffic of one product's fold launches (levels 1 .. 12 at n = 12), n = 13
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-final}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/${TAG}_build.log 2>&1
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:k_fold -s 36 -c 12 --csv --log-file gpurun_out/${TAG}_fold_product.csv python bench.py --n 12 --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/${TAG}_fold_ncu.log 2>&1
python - "$TAG" <<'PY' > gpurun_out/${TAG}_fold_traffic.log 2>&1
import csv, json, sys
tag = sys.argv[1]
unit = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
rows = list(csv.reader(l for l in open(f"gpurun_out/{tag}_fold_product.csv") if l.startswith('"')))
h = rows[0]
m, v, u = h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
tot = {"dram__bytes_read.sum": 0.0, "dram__bytes_write.sum": 0.0}
n = 0
for r in rows[1:]:
    if r[m] in tot:
        tot[r[m]] += float(r[v].replace(",", "")) * unit.get(r[u], 1)
    n += r[m] == "gpu__time_duration.sum"
rec = {"bytes_per_launch": int(tot["dram__bytes_read.sum"] + tot["dram__bytes_write.sum"]),
       "source": f"profiles/r2/fold_product_n12.csv ({tot['dram__bytes_read.sum'] / 1e9:.6f} GB read + "
                 f"{tot['dram__bytes_write.sum'] / 1e9:.6f} GB write over the {n} k_fold launches of one n = 12 product)"}
d = json.load(open("profiles/ncu_traffic.json"))
d["k_fold:row-inclusion fold:n12:g1:sym:reuse"] = rec
json.dump(d, open("profiles/ncu_traffic.json", "w"), indent=2)
json.dump(rec, open(f"gpurun_out/{tag}_fold_traffic.json", "w"), indent=2)
print(rec)
PY
timeout 900 python bench.py > gpurun_out/${TAG}_bench_default.log 2>&1
for n in 9 10 11; do timeout 600 python bench.py --n $n --no-cpu-baseline > gpurun_out/${TAG}_bench_n$n.log 2>&1; done
timeout 900 python bench.py --n 13 --no-cpu-baseline --steps 3 --warmup 1 > gpurun_out/${TAG}_bench_n13.log 2>&1
