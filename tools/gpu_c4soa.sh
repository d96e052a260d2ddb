# C4 face loop: SoA vs AoS state/flux layout on the k-way and structured blocks
for lay in aos soa; do
  timeout 600 python tools/prof_loop.py --config C4 --reorder partition --block-size 256 --layout $lay --runs 3 --timed 9 --schedule stream,stream-pull,pipelined,pipelined-pull 2>&1 | grep "^hier\|Error\|error" | sed "s/^/$lay kway256 /"
  timeout 600 python tools/prof_loop.py --config C4 --reorder structured:4,4,8 --block-size 480 --layout $lay --runs 3 --timed 9 --schedule stream,stream-pull,pipelined-pull 2>&1 | grep "^hier\|Error\|error" | sed "s/^/$lay s448 /"
done
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c4soa_launches.csv python tools/prof_loop.py --config C4 --reorder partition --block-size 256 --layout soa --runs 1 --timed 1 --schedule pipelined-pull,stream-pull > /dev/null 2>&1
python - <<'PY'
import csv, collections
rows=list(csv.reader(open('gpurun_out/c4soa_launches.csv')))
hdr=None; agg=collections.defaultdict(float)
for r in rows:
    if 'Kernel Name' in r: hdr=r; continue
    if hdr is None or len(r)!=len(hdr): continue
    d=dict(zip(hdr,r)); k=d['Kernel Name'][:40]; v=float(d['Metric Value'].replace(',',''))
    agg[(k,d['Metric Name'])]+=v
for k,v in sorted(agg.items()): print(k, v)
PY
