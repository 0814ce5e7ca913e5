"""Project a P = 8 engine calibration from the measured P = 2 and P = 4 ones.

No 8-GPU box is available to the builder (gpurun gives 1, 2 or 4 GPUs), but
both bench arms must plan the N = 8 run from the SAME committed calibration
(profiles/calib/calib_<trace>_P8.csv). Projection, per trace:

  linear fits (reference fit_model) a2, b2, a4, b4 of the measured sweeps;
  a8 = a4 + (a4 - a2)           (per-group latency grows by one doubling step)
  b8 = b4 * (7/8) / (3/4)       (bus bytes 2(P-1)/P * S at equal bus bandwidth)
  t8(S) = t4(S) * (a8 + b8*S) / (a4 + b4*S)   (keeps the measured LL /
                                               one-shot / two-shot shape)

The driver's 8-GPU scale run re-measures it on the box (calibration.onbox in
the bench line) — the projection only fixes the plan both arms run.
"""
import glob
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from paper_1912_09268_b200 import gradsched as gs  # noqa: E402


def main():
    out = []
    for p4 in sorted(glob.glob(os.path.join(ROOT, "profiles", "calib", "calib_*_P4.csv"))):
        p2 = p4.replace("_P4.csv", "_P2.csv")
        m2, m4 = gs.load_measurements_csv(p2), gs.load_measurements_csv(p4)
        f2, f4 = gs.fit_model(m2), gs.fit_model(m4)
        a8 = f4.a + max(0.0, f4.a - f2.a)
        b8 = f4.b * (7 / 8) / (3 / 4)
        p8 = p4.replace("_P4.csv", "_P8.csv")
        with open(p8, "w") as f:
            f.write("size_bytes,time_us\n")
            for m in m4:
                t = m.time_sec * (a8 + b8 * m.size_bytes) / (f4.a + f4.b * m.size_bytes)
                f.write(f"{m.size_bytes},{t * 1e6:.3f}\n")
        f8 = gs.fit_model(gs.load_measurements_csv(p8))
        out.append(f"{os.path.basename(p8)}: a {f2.a*1e6:.2f} / {f4.a*1e6:.2f} -> {f8.a*1e6:.2f} us, "
                   f"b {f2.b*1e12:.3f} / {f4.b*1e12:.3f} -> {f8.b*1e12:.3f} ps/B")
    print("\n".join(out))


if __name__ == "__main__":
    main()
