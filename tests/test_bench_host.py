"""Host logic of bench.py's clock sampler (timing rules: clocks and throttle
reasons sampled during the timed region). No GPU: the NVML poll is driven with
a fake module, and the summary is checked on hand-written rows."""
import os
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402


class FakeNVML:
    NVML_CLOCK_SM = 1
    nvmlClocksThrottleReasonHwSlowdown = 0x8
    nvmlClocksThrottleReasonHwThermalSlowdown = 0x40
    nvmlClocksThrottleReasonSwThermalSlowdown = 0x20
    nvmlClocksThrottleReasonSwPowerCap = 0x4

    def __init__(self):
        self.n = 0

    def nvmlDeviceGetMaxClockInfo(self, h, kind):
        return 1965

    def nvmlDeviceGetClockInfo(self, h, kind):
        self.n += 1
        return 1965 if self.n % 2 else 1950

    def nvmlDeviceGetCurrentClocksThrottleReasons(self, h):
        return self.nvmlClocksThrottleReasonSwPowerCap if self.n == 3 else 0


def test_summary_reasons_and_median():
    c = bench.ClockSampler(0)
    c.rows = [["1965", "1965", "Not Active", "Not Active", "Not Active", "Active"],
              ["1900", "1965", "Not Active", "Active", "Not Active", "Not Active"],
              ["1950", "1965", "Not Active", "Not Active", "Not Active", "Not Active"]]
    s = c.summary()
    assert s["sm_mhz"] == 1950.0 and s["sm_max_mhz"] == 1965.0 and s["samples"] == 3
    assert s["reasons"] == ["hw_thermal_slowdown", "sw_power_cap"]


def test_summary_unsampled():
    s = bench.ClockSampler(0).summary()
    assert s["samples"] == 0 and s["reasons"] == ["unsampled"]


def test_nvml_poll_rows_decode_reason_bits():
    c = bench.ClockSampler(0)
    nv, ready = FakeNVML(), threading.Event()
    t = threading.Thread(target=c._nvml_poll, args=(None, nv, ready), daemon=True)
    t.start()
    assert ready.wait(2.0)
    while len(c.rows) < 5:
        pass
    c.stop.set()
    t.join(2.0)
    assert not t.is_alive()
    assert all(len(r) == 6 for r in c.rows)
    s = c.summary()
    assert s["sm_max_mhz"] == 1965.0 and s["reasons"] == ["sw_power_cap"]


def test_nvml_poll_without_max_clock_returns_unsampled():
    """if NVML fails before the first sample the poll thread exits
    without signalling `ready`, so __enter__ falls back to nvidia-smi instead
    of timing a region with no clock record."""
    class Broken(FakeNVML):
        def nvmlDeviceGetMaxClockInfo(self, h, kind):
            raise RuntimeError("NVML_ERROR_NOT_SUPPORTED")
    c = bench.ClockSampler(0)
    ready = threading.Event()
    t = threading.Thread(target=c._nvml_poll, args=(None, Broken(), ready), daemon=True)
    t.start()
    t.join(2.0)
    assert not t.is_alive() and not ready.is_set() and c.rows == []
