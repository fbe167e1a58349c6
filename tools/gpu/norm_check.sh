mkdir -p gpurun_out
true
python - > gpurun_out/norm_time.log 2>&1 <<'PY'
import sys, ctypes as C, torch
sys.path.insert(0, '.')
from paper_2510_02758_b200 import _lib
x = torch.randn(128, 4096, device='cuda').to(torch.bfloat16); w = torch.ones(4096, device='cuda').to(torch.bfloat16); y = torch.empty_like(x)
def f(): _lib.check(_lib.lib.tf_rmsnorm(C.c_void_p(x.data_ptr()), C.c_void_p(w.data_ptr()), C.c_void_p(y.data_ptr()), 128, 4096, 1e-5, C.c_void_p(torch.cuda.current_stream().cuda_stream)))
for _ in range(10): f()
g = torch.cuda.CUDAGraph()
with torch.cuda.graph(g):
    for _ in range(100): f()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); g.replay(); e1.record(); torch.cuda.synchronize()
print("rmsnorm B=128 D=4096 per launch (graph): %.2f us" % (e0.elapsed_time(e1) * 10))
PY
cat gpurun_out/norm_time.log; tail -n 2 gpurun_out/pytest_norm.log
