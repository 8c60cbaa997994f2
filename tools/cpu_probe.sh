nproc; cat /proc/loadavg; cat /sys/fs/cgroup/cpu.max 2>/dev/null
python -c "
import sys,time,json; sys.path.insert(0,'.')
import bench
for i in range(2):
    t=time.time(); d=bench.cpu_baseline_subprocess(4, 8.0); print(json.dumps({k:d[k] for k in ('tflops','seconds','steps','threads')}), time.time()-t, flush=True)
"
python bench.py --impl reference --steps 2 --warmup 1
cat /proc/loadavg
