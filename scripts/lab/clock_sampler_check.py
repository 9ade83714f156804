import faulthandler, sys, time
faulthandler.enable()
sys.path.insert(0, '.')
import torch
torch.cuda.init()
pr = torch.cuda.get_device_properties(0); print("props", pr.pci_domain_id, pr.pci_bus_id, pr.pci_device_id, flush=True)
from bench import ClockSampler
c = ClockSampler(0)
print("init ok", c.source, flush=True)
print(c._sample_nvml() if c._nvml else None, flush=True)
with c:
    time.sleep(0.05)
print(c.summary(), flush=True)
