set -u
mkdir -p gpurun_out/abr
for lib in ${LIBS:-build/ab/liborx_route7.so cur}; do
  if [ "$lib" = cur ]; then unset ORX_LIB_PATH; else export ORX_LIB_PATH=$lib; fi
  timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:moe_route_tc --csv --log-file gpurun_out/abr/$(basename $lib).csv python profiles/run_step.py --warmup 1 --steps 1 > /dev/null 2>&1
  python3 - gpurun_out/abr/$(basename $lib).csv <<'P'
import csv,sys
rows=[r for r in csv.reader(open(sys.argv[1])) if len(r)>5]
h=rows[0]; i=h.index('Metric Value')
v=[float(r[i].replace(',','')) for r in rows[1:]]
print(sys.argv[1], len(v), 'mean us', sum(v)/len(v)/1e3 if v else 0, [round(x/1e3,1) for x in v])
P
done
