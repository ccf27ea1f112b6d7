"""bench.py's clock sampler (CPU): NVML polled from a thread with time stamps; only samples taken
between mark() and stop() count, throttle-reason bits map to the names the bench contract uses.
A fake NVML module stands in for the driver (no GPU here)."""
import time

import bench


class FakeNvml:
    NVML_CLOCK_SM = 1

    def __init__(self):
        self.mhz, self.reasons = 1965, 0

    def nvmlDeviceGetMaxClockInfo(self, h, kind):
        return 1965

    def nvmlDeviceGetClockInfo(self, h, kind):
        return self.mhz

    def nvmlDeviceGetCurrentClocksEventReasons(self, h):
        return self.reasons


def test_samples_only_inside_the_timed_region(monkeypatch):
    nv = FakeNvml()
    monkeypatch.setattr(bench.ClockSampler, "_nvml_handle", lambda self: (nv, object()))
    s = bench.ClockSampler(0)
    s.start()
    nv.mhz, nv.reasons = 1000, 0x40  # before the region: must not count
    time.sleep(0.08)
    nv.mhz, nv.reasons = 1500, 0x4
    time.sleep(0.03)
    s.mark()
    time.sleep(0.15)
    out = s.stop()
    assert out["source"] == "nvml" and out["sm_max_mhz"] == 1965.0
    assert out["samples"] >= 5
    assert out["sm_mhz"] == 1500.0 and out["sm_min_mhz"] == 1500.0
    assert out["reasons"] == ["sw_power_cap"]  # the hw_thermal_slowdown before mark() is dropped


def test_reason_bits():
    bits = dict(bench.ClockSampler.REASONS)
    assert bits == {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40,
                    "sw_thermal_slowdown": 0x20, "sw_power_cap": 0x4}
