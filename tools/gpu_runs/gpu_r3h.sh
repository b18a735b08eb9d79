#!/bin/bash
mkdir -p gpurun_out
T=gpurun_out/r3h
CMD="python bench.py --workload C1 --steps 3 --warmup 3 --no-secondary --no-cpu-baseline --no-e2e"
$CMD > ${T}_plain.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file ${T}_launches.csv $CMD > /dev/null 2>&1; echo "rc=$?"
grep -E "tf32|split" ${T}_launches.csv | tail -6 | awk -F'","' '{print $5, $NF}'
python - <<'PY'
import time, torch
from paper_2302_06218_b200 import dmha
dmha.init(1, 0, None, 0, "fp32", "contiguous")
L,H,D=512,4,64
q,k,v=(torch.randn(L,H,D,device="cuda") for _ in range(3))
out,lse=torch.empty_like(q),torch.empty(H,L,device="cuda")
for _ in range(10): dmha.forward(q,k,v,L,False,out,lse)
torch.cuda.synchronize()
t=time.perf_counter()
for _ in range(200): dmha.forward(q,k,v,L,False,out,lse)
t1=time.perf_counter(); torch.cuda.synchronize(); t2=time.perf_counter()
print("host us per forward", (t1-t)/200*1e6, "total us per forward", (t2-t)/200*1e6)
s,e=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
g=torch.cuda.CUDAGraph()
st=torch.cuda.Stream()
dmha.reserve(1,L,D,H)
with torch.cuda.stream(st):
    dmha.forward(q,k,v,L,False,out,lse)
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=st):
        dmha.forward(q,k,v,L,False,out,lse)
torch.cuda.synchronize()
s.record()
for _ in range(200): g.replay()
e.record(); torch.cuda.synchronize()
print("graph replay us per forward", s.elapsed_time(e)/200*1e3)
PY
