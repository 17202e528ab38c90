"""Host-side stepping logic that needs no GPU."""
import torch

from paper_2306_02526_b200.timestep import TimeStepper


def test_gradient_use_probe():
    """The stepper skips the device gradient only for a g that reads neither
    component; reads through arithmetic or through comparisons are detected."""
    gen = torch.Generator().manual_seed(0)
    U, ux, uy = (torch.randn((1, 64), generator=gen, dtype=torch.float64) for _ in range(3))
    cases = {
        "allen_cahn": (lambda t, u, gx, gy: u - u ** 3, (False, False)),
        "burgers": (lambda t, u, gx, gy: -u * gx, (True, False)),
        "switch_y": (lambda t, u, gx, gy: torch.where(gy > 0, u, -u), (False, True)),
        "both": (lambda t, u, gx, gy: gx * gx + gy * gy, (True, True)),
    }
    for name, (g, want) in cases.items():
        r = g(0.0, U, ux, uy)
        TimeStepper._probe_grad_use(g, 0.0, U, ux, uy, r)
        assert g._hb_grad_use == want, name
