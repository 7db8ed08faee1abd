"""Which per-step overheads separate the device-resident loop from the host-pointer loop."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2504_10724_b200 import eeb  # noqa: E402

desc = eeb.PRESETS["opt-1.3b-4x"].replace(max_slots=64, max_seq_len=228)
ctx = eeb.Context(0)
m = ctx.register(desc)
ctx.load_layers(m, desc.num_layers)
B, P = 64, 128
rng = np.random.default_rng(0)
slots = np.arange(B, dtype=np.int32)
for p in range(P):
    ctx.decode_step(m, 0, eeb.FULL_DEPTH, 0.7, slots, rng.integers(0, desc.vocab, B), np.full(B, p))
stream = torch.cuda.ExternalStream(ctx.stream())
dev = torch.device("cuda")
N = 30
toks = torch.from_numpy(rng.integers(0, desc.vocab, (N, B)).astype(np.int32)).to(dev)
pos = torch.from_numpy(np.stack([np.full(B, P + k, np.int32) for k in range(N)])).to(dev)
sl = torch.from_numpy(slots).to(dev)
outs = {"exit_layer": torch.zeros(B, dtype=torch.int32, device=dev), "token_id": torch.zeros(B, dtype=torch.int32, device=dev),
        "confidence": torch.zeros(B, dtype=torch.float32, device=dev), "hist": torch.zeros(4, dtype=torch.int64, device=dev)}
ptrs = {k: v.data_ptr() for k, v in outs.items()}
acc = torch.zeros(4, dtype=torch.int64, device=dev)


def run(name, fn):
    for k in range(5):
        fn(k)
    torch.cuda.synchronize()
    ctx.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record(stream)
    for k in range(5, N):
        fn(k)
    e1.record(stream)
    e1.synchronize()
    wall = (time.perf_counter() - t0) / (N - 5) * 1e3
    print(f"{name:40s} device {e0.elapsed_time(e1) / (N - 5):.3f} ms/step  wall {wall:.3f} ms/step", flush=True)


def dev_full(k):
    ctx.decode_step_device(m, 0, eeb.INTROSPECTIVE, 0.7, B, sl.data_ptr(), toks[k].data_ptr(), pos[k].data_ptr(), ptrs)
    with torch.cuda.stream(stream):
        acc.add_(outs["hist"])


def dev_noout(k):
    ctx.decode_step_device(m, 0, eeb.INTROSPECTIVE, 0.7, B, sl.data_ptr(), toks[k].data_ptr(), pos[k].data_ptr(), None)


toks_h = toks.cpu().numpy()
pos_h = pos.cpu().numpy()


def host(k):
    ctx.decode_step(m, 0, eeb.INTROSPECTIVE, 0.7, slots, toks_h[k], pos_h[k])


run("device path + outputs + torch op", dev_full)
run("device path, no outputs", dev_noout)
run("host path (sync each step)", host)
run("device path + outputs + torch op (again)", dev_full)

import subprocess  # noqa: E402
import threading  # noqa: E402

for ms in (100, 500):
    proc = subprocess.Popen(["nvidia-smi", "--id=0", "--query-gpu=clocks.sm,clocks_event_reasons.sw_power_cap",
                             "--format=csv,noheader", "-lms", str(ms)], stdout=subprocess.DEVNULL)
    time.sleep(0.5)
    run(f"device path, nvidia-smi -lms {ms} running", dev_full)
    proc.terminate()
    proc.wait()

import pynvml  # noqa: E402

pynvml.nvmlInit()
hdl = pynvml.nvmlDeviceGetHandleByIndex(0)
stop = False
samples = []


def poll():
    while not stop:
        samples.append((pynvml.nvmlDeviceGetClockInfo(hdl, pynvml.NVML_CLOCK_SM),
                        pynvml.nvmlDeviceGetCurrentClocksEventReasons(hdl)))
        time.sleep(0.1)


th = threading.Thread(target=poll)
th.start()
run("device path, NVML thread polling 100 ms", dev_full)
stop = True
th.join()
print("nvml samples", len(samples), samples[:3])
