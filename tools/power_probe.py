"""Run the C2 fused step back to back for ~4 s while nvidia-smi samples SM
clock, power draw and throttle reasons (power/clock evidence for §8)."""
import os, subprocess, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2605_13276_b200 import grpo
dev = torch.device("cuda", 0)
N_GROUPS, G, C, T, V = 64, 8, 1, 56, 32064
R = N_GROUPS * G * C * T
g = torch.Generator(device=dev).manual_seed(0)
logits = (torch.randn(R, V, device=dev, generator=g) * 2).to(torch.bfloat16)
tokens = torch.randint(31744, 32000, (R,), device=dev, generator=g, dtype=torch.int32)
rw = torch.randint(0, 2, (N_GROUPS * G,), device=dev, generator=g).float()
tl = grpo.TokenLoss(N_GROUPS, G, C, T, V, grpo.GrpoConfig(group_size=G))
tl.launch(logits, tokens, torch.zeros(N_GROUPS * G, device=dev), rw, None)
blp = (tl.lp_chunk + 0.01).float()
dl = torch.empty_like(logits)
MODE = os.environ.get("MODE", "normal")  # normal | c0 (zero coefficients) | fwd (no dlogits)
if MODE == "c0":
    rw = torch.ones_like(rw)
out_dl = None if MODE == "fwd" else dl
smi = subprocess.Popen(["nvidia-smi", "--id=0", "--query-gpu=clocks.sm,power.draw,power.limit,"
                        "clocks_event_reasons.sw_power_cap,temperature.gpu",
                        "--format=csv,noheader,nounits", "-lms", "200"], stdout=subprocess.PIPE,
                       text=True)
time.sleep(0.5)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
n = 0
t0 = time.time()
while time.time() - t0 < 4.0:
    for _ in range(50):
        tl.launch(logits, tokens, blp, rw, out_dl)
    n += 50
    torch.cuda.synchronize()
e1.record()
torch.cuda.synchronize()
smi.terminate()
out = smi.communicate()[0].strip().splitlines()
print(f"{MODE}: {n} steps, {e0.elapsed_time(e1) / n:.3f} ms/step")
for line in out[2:-1:3]:
    print("  sm MHz, W, limit W, power cap, C:", line)
