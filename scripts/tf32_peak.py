"""Measure the dense TF32 tensor-core peak on this B200 (verdict r01 item 6), the way MEASURED_PEAKS.json
measures bf16: torch.matmul fp32 with TF32 enabled (cuBLAS tcgen05 kernels) on 8192^3, best of 10
(burst) and back to back for 4 s (sustained); plus a cuBLAS-free tcgen05 loop: this library's Gram
kernel issuing only the H*H^T product (tsk_gram_probe mode bit 1: 1xTF32, the same MMA instruction as
the 3xTF32 Gram) on a C5-sized stack.  Writes profiles/r02_tf32_peak.json.
  python scripts/tf32_peak.py"""
import json, os, sys, time
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2209_14637_b200 as tsk  # noqa: E402

torch.backends.cuda.matmul.allow_tf32 = True
N = 8192
a = torch.randn(N, N, device="cuda")
b = torch.randn(N, N, device="cuda")
flops = 2.0 * N ** 3
for _ in range(3):
    a @ b
torch.cuda.synchronize()
best = 0.0
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); c = a @ b; e1.record(); torch.cuda.synchronize()
    best = max(best, flops / (e0.elapsed_time(e1) / 1e3) / 1e12)
n = 0
t0 = time.perf_counter()
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record()
while time.perf_counter() - t0 < 4.0:
    for _ in range(10):
        c = a @ b
    n += 10
    torch.cuda.synchronize()
e1.record(); torch.cuda.synchronize()
sustained = flops * n / (e0.elapsed_time(e1) / 1e3) / 1e12
del a, b, c
torch.cuda.empty_cache()
# cuBLAS-free: 1xTF32 Gram (tcgen05.mma kind::tf32, cta_group::2) on m = n = 4096, D = 64
m, nn, D = 4096, 4096, 64
A = torch.rand(D, m, nn, device="cuda")
G = torch.empty(m, m, dtype=torch.float64, device="cuda")
tsk.tsk_gram_probe(A, mode=2, G64=G)
torch.cuda.synchronize()
times = []
for _ in range(5):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); tsk.tsk_gram_probe(A, mode=2, G64=G); e1.record(); torch.cuda.synchronize()
    times.append(e0.elapsed_time(e1) / 1e3)
nb = -(-m // 128)
issued = (nb * (nb + 1) // 2) * 128 * 128 * 2.0 * nn * D  # 1 product over the lower 128 x 128 tiles
own = issued / min(times) / 1e12
out = {"tf32_tflops_cublas_burst": best, "tf32_tflops_cublas_sustained": sustained,
       "tf32_tflops_tcgen05_gram_1x": own, "nominal_tf32_tflops": 1100.0,
       "how": "torch.matmul fp32 with allow_tf32 8192^3 (2 N^3 flops): best of 10 (burst), back to back 4 s "
              "(sustained); tcgen05 1xTF32: tsk_gram_probe mode 2 on [64][4096][4096], issued flops of the "
              "lower 128x128 tiles / best of 5",
       "gpu": torch.cuda.get_device_name(), "torch": torch.__version__}
print(json.dumps(out))
os.makedirs("profiles", exist_ok=True)
with open(os.path.join("profiles", "r02_tf32_peak.json"), "w") as f:
    json.dump(out, f, indent=1)
