"""GPU clock / throttle sampling during timed regions (NVML), used by
bench.py to attach a ``clocks`` record to every measured number."""

from __future__ import annotations

import threading
import time

_REASONS = {
    0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
    0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
    0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting",
}


class ClockSampler:
    """Samples SM clock and throttle reasons every ``period`` seconds on one
    device while active (start()/stop())."""

    def __init__(self, device_index: int = 0, period: float = 0.05):
        self.idx = device_index
        self.period = period
        self.samples: list[tuple[float, int, int]] = []
        self._stop = threading.Event()
        self._th = None
        self.max_mhz = None
        self.ok = False
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:  # NVML missing: report null clocks
            self._nv = None

    def _run(self):
        nv = self._nv
        while not self._stop.is_set():
            try:
                sm = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
                rs = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                self.samples.append((time.time(), sm, rs))
            except Exception:
                pass
            self._stop.wait(self.period)

    def start(self):
        if self.ok:
            self._stop.clear()
            self._th = threading.Thread(target=self._run, daemon=True)
            self._th.start()
        return self

    def stop(self):
        if self._th is not None:
            self._stop.set()
            self._th.join()
        return self.summary()

    def summary(self) -> dict:
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "samples": 0}
        sms = sorted(s[1] for s in self.samples)
        reasons = 0
        for _, _, r in self.samples:
            reasons |= r
        names = [v for k, v in _REASONS.items() if reasons & k and v != "gpu_idle"]
        return {"sm_mhz": sms[len(sms) // 2], "sm_max_mhz": self.max_mhz, "reasons": names,
                "samples": len(self.samples)}


def clocks_rejected(c: dict) -> bool:
    """The run contract's rejection rule: hardware/thermal slowdown, or SM
    clocks stuck well below max with no reason."""
    bad = {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}
    if any(r in bad for r in c.get("reasons", [])):
        return True
    if c.get("sm_mhz") and c.get("sm_max_mhz") and not c.get("reasons"):
        return c["sm_mhz"] < 0.7 * c["sm_max_mhz"]
    return False
