"""Host logic of bench.py that needs no GPU: the clock sampler's window and throttle-reason parsing
(the timing rules reject a run that saw hw_slowdown / thermal slowdown, so the parse must be right)."""
import datetime
import time

import bench


def _line(ts, sm, mx, pw, reasons=()):
    names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
    flags = ["Active" if n in reasons else "Not Active" for n in names]
    stamp = datetime.datetime.fromtimestamp(ts).strftime("%Y/%m/%d %H:%M:%S.%f")[:-3]
    return ", ".join([stamp, "0", str(sm), str(mx), str(pw), "0x0"] + flags)


def test_clock_summary_window_and_reasons():
    t0 = time.time()
    c = bench.ClockSampler(0)
    c.lines = [_line(t0 - 5, 600, 1965, 150),                       # before the window: ignored
               _line(t0 + 0.1, 1965, 1965, 900),
               _line(t0 + 0.2, 1380, 1965, 990, ("sw_power_cap",)),
               _line(t0 + 0.3, 1400, 1965, 995, ("sw_power_cap",)),
               _line(t0 + 9, 1000, 1965, 800, ("hw_slowdown",))]      # after it: ignored
    c.nv = [(t0 - 1, 500, 0x0), (t0 + 0.15, 1965, 0x0), (t0 + 0.25, 1380, 0x4), (t0 + 0.35, 1390, 0x4),
            (t0 + 0.36, 1390, 0x40)]
    s = c.summary(t0, t0 + 0.5)
    assert s["samples"] == 3
    assert s["sm_mhz"] == 1400 and s["sm_max_mhz"] == 1965
    assert s["reasons"] == ["sw_power_cap"]
    assert s["power_w_median"] == 990 and s["power_w_max"] == 995
    nv = s["nvml_10ms"]
    assert nv["samples"] == 4 and nv["sm_mhz_min"] == 1380
    assert nv["reasons"] == ["hw_thermal_slowdown", "sw_power_cap"]


def test_clock_summary_without_tools():
    c = bench.ClockSampler(0)
    c.lines, c.nv = [], []
    s = c.summary(0.0, 1.0)
    assert s["samples"] == 0 and s["sm_mhz"] is None and "nvml_10ms" not in s
