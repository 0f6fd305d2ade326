set -x
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/g1_gather tools/g1_gather.cu
mkdir -p gpurun_out/g1
./tools/g1_gather > gpurun_out/g1/g1.jsonl; cat gpurun_out/g1/g1.jsonl
./tools/g1_gather 32 > gpurun_out/g1/g1_lim32.jsonl; cat gpurun_out/g1/g1_lim32.jsonl
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_ltcfabric.sum,lts__t_sectors_op_read.sum --clock-control none --csv --log-file gpurun_out/g1/ncu.csv ./tools/g1_gather > /dev/null 2>&1
python - <<'PY'
import csv
rows=[r for r in csv.reader(open('gpurun_out/g1/ncu.csv')) if len(r)>10]
hdr=rows[0]; ki=hdr.index('Kernel Name'); mi=hdr.index('Metric Name'); vi=hdr.index('Metric Value'); ii=hdr.index('ID')
d={}
for r in rows[1:]:
    d.setdefault((int(r[ii]),r[ki][:40]),{})[r[mi]]=r[vi]
for k,v in sorted(d.items()): print(k, v)
PY
