"""Raw NVML clock-event reason masks and SM clocks sampled every 2 ms while bench.py runs a timed region
(diagnostic). Usage: python scripts/clock_reasons.py [bench args...]"""
import collections
import subprocess
import sys
import threading
import time

import pynvml

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
stop = threading.Event()
samples = []


def run():
    while not stop.is_set():
        samples.append((pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
                        pynvml.nvmlDeviceGetCurrentClocksEventReasons(h), pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0))
        time.sleep(0.002)


t = threading.Thread(target=run, daemon=True)
t.start()
out = subprocess.run([sys.executable, "bench.py"] + sys.argv[1:], capture_output=True, text=True)
stop.set()
t.join()
busy = [s for s in samples if s[2] > 300]
print("samples", len(samples), "busy (>300 W)", len(busy))
c = collections.Counter(hex(r) for _, r, _ in busy)
print("reason masks (busy):", c.most_common(8))
clk = sorted(s[0] for s in busy)
if clk:
    print("sm MHz busy: p10 %d median %d p90 %d" % (clk[len(clk) // 10], clk[len(clk) // 2], clk[9 * len(clk) // 10]))
pw = sorted(s[2] for s in busy)
if pw:
    print("power W busy: median %.0f max %.0f" % (pw[len(pw) // 2], pw[-1]))
print(out.stdout.strip().splitlines()[-1][:300] if out.stdout.strip() else out.stderr[-500:])
