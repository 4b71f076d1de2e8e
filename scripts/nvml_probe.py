import time
import pynvml as N
N.nvmlInit()
h = N.nvmlDeviceGetHandleByIndex(0)
for name, fn in [("sm_clock", lambda: N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)),
                 ("max_clock", lambda: N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM)),
                 ("reasons", lambda: N.nvmlDeviceGetCurrentClocksEventReasons(h)),
                 ("power", lambda: N.nvmlDeviceGetPowerUsage(h)),
                 ("temp", lambda: N.nvmlDeviceGetTemperature(h, N.NVML_TEMPERATURE_GPU))]:
    t0 = time.perf_counter()
    for _ in range(5):
        v = fn()
    print(f"{name}: {(time.perf_counter() - t0) / 5 * 1e3:.3f} ms  value={v}")
