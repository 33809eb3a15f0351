# Round-2 profiling pass: per-kernel launch list at c4 (windows after the sweeps, so kernel times
# are not overlapped) and an ncu --set full capture of the c5 sweep (C = 128 GEMV question).
mkdir -p gpurun_out
SCRF_OVERLAP=0 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launch_c4_seqwin.csv python tools/one_posterior.py c4 full > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -c 1 -o gpurun_out/r02_sweep_c5 -f python tools/one_posterior.py c5 full > gpurun_out/ncu_c5.log 2>&1
python - <<'PY'
import csv,collections
rows=[r for r in csv.reader(open("gpurun_out/r02_launch_c4_seqwin.csv")) if len(r)>10]
hdr=rows[0]; i=hdr.index("Kernel Name"); v=hdr.index("Metric Value")
data=rows[1:]; second=data[len(data)//2:]
agg=collections.defaultdict(lambda:[0,0.0])
for r in second:
    k=r[i].split("(")[0].split("<")[0]; agg[k][0]+=1; agg[k][1]+=float(r[v].replace(",",""))
tot=sum(x[1] for x in agg.values())
print("total ms",tot/1e6)
for k,(c,t) in sorted(agg.items(), key=lambda x:-x[1][1]): print(f"  {k:32s} n={c:4d} {t/1e6:8.3f} ms")
PY
