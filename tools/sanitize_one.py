"""Small decode + ber_sim run for compute-sanitizer (racecheck / synccheck / memcheck)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import inputs  # noqa: E402
import paper_2305_05286_b200 as cbp  # noqa: E402

for name, frames, rule in (("C1", 64, 0), ("C2", 48, 0), ("C3a", 12, 0), ("C2", 32, 2)):
    base, Z = inputs.config_base(name)
    g = cbp.Code(base, Z)
    llr, _ = g.channel(2.0, 1, 0, frames, want_cw=False)
    g.decode(llr, 6, rule, ev=True, omega=True)
    g.ber_sim(2.0, 1, 0, frames, 6, rule)
    torch.cuda.synchronize()
    print(name, "ok")
