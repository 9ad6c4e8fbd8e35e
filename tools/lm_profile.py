"""Profile one configs[4] LM training step (torch.profiler), top CUDA kernels."""
import sys
sys.path.insert(0, ".")
import torch
from paper_2507_04239_b200.lm import LMConfig, PowerLM, train_step

cfg = LMConfig()
model = PowerLM(cfg).cuda()
opt = torch.optim.AdamW(model.parameters(), lr=3e-4, fused=True)
tok = torch.randint(0, cfg.vocab, (1, 32769), device="cuda")
for _ in range(3):
    train_step(model, opt, tok[:, :-1], tok[:, 1:])
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    train_step(model, opt, tok[:, :-1], tok[:, 1:])
    torch.cuda.synchronize()
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=30, max_name_column_width=70))
