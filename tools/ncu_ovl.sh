mkdir -p gpurun_out
for m in -1 0; do
SCRF_OVERLAP=$m timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/ovl_launch_$m.csv python tools/one_posterior.py c4 full > /dev/null 2>&1
done
python - <<'PY'
import csv,collections
for m in ("-1","0"):
    rows=[r for r in csv.reader(open(f"gpurun_out/ovl_launch_{m}.csv")) if len(r)>10]
    hdr=rows[0]; i=hdr.index("Kernel Name"); v=hdr.index("Metric Value"); idl=hdr.index("ID")
    data=rows[1:]
    n=len(data)//2
    second=data[n:]  # the second (warm) posterior
    agg=collections.defaultdict(lambda:[0,0.0])
    for r in second:
        k=r[i].split("(")[0].split("<")[0]
        agg[k][0]+=1; agg[k][1]+=float(r[v].replace(",",""))
    tot=sum(x[1] for x in agg.values())
    print("mode",m,"total ms",tot/1e6)
    for k,(c,t) in sorted(agg.items(), key=lambda x:-x[1][1]): print(f"  {k:32s} n={c:4d} {t/1e6:8.3f} ms")
PY
