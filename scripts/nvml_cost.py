"""Latency of the NVML queries bench.py samples, on an idle and a busy GPU."""
import threading, time
import pynvml, torch

pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
Q = {"clock": lambda: pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM),
     "reasons": lambda: pynvml.nvmlDeviceGetCurrentClocksEventReasons(h),
     "power": lambda: pynvml.nvmlDeviceGetPowerUsage(h),
     "temp": lambda: pynvml.nvmlDeviceGetTemperature(h, 0)}


def probe(tag):
    for k, f in Q.items():
        ts = []
        for _ in range(20):
            t = time.perf_counter(); f(); ts.append(1e3 * (time.perf_counter() - t))
            time.sleep(0.02)
        print(tag, k, "median %.3f ms max %.3f ms" % (sorted(ts)[10], max(ts)), flush=True)


probe("idle")
a = torch.randn(8192, 8192, device="cuda")
stop = threading.Event()


def load():
    while not stop.is_set():
        for _ in range(20):
            a @ a
        torch.cuda.synchronize()


th = threading.Thread(target=load); th.start()
time.sleep(0.5)
probe("busy")
stop.set(); th.join()
