"""Unit-aware reader of `ncu -i REPORT --page raw --csv`.

Row 0 holds the metric names, row 1 their units (byte, Kbyte, Mbyte, Gbyte,
ns, us, ms, usecond, ...), rows 2.. one launch each.  Values are returned in
SI base units (bytes, seconds, or the raw number for unitless / % metrics),
so a metric ncu prints in Kbyte is never read as Mbyte.
"""
import csv
import io
import subprocess

_SCALE = {
    "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
    "nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3,
    "second": 1.0, "s": 1.0,
    "byte/second": 1.0, "Kbyte/second": 1e3, "Mbyte/second": 1e6, "Gbyte/second": 1e9,
    "Tbyte/second": 1e12,
    "byte/s": 1.0, "Kbyte/s": 1e3, "Mbyte/s": 1e6, "Gbyte/s": 1e9, "Tbyte/s": 1e12,
    "cycle/nsecond": 1e9, "cycle/usecond": 1e6, "cycle/second": 1.0,
    "hz": 1.0, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9,
}


def scale_of(unit: str) -> float:
    return _SCALE.get(unit.strip(), 1.0)


def launches(rep: str, kernel_substr: str = ""):
    """List of dict(metric -> value in base units) for the report's launches
    whose row mentions `kernel_substr`."""
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rr = list(csv.reader(io.StringIO(txt)))
    if len(rr) < 3:
        return []
    names, units = rr[0], rr[1]
    out = []
    for r in rr[2:]:
        if kernel_substr and kernel_substr not in "".join(r):
            continue
        d = {}
        for n, u, v in zip(names, units, r):
            try:
                d[n] = float(v.replace(",", "")) * scale_of(u)
            except ValueError:
                d[n] = v
        out.append(d)
    return out
