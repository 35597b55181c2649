"""The BASELINE.json workloads (configs[0..4]) as channel model + solver settings.

SNR convention (decision D-2): sigma2 = 1, P_tx = SNR_lin, alpha = K / SNR_lin.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import torch

from .channel import ChannelModel


@dataclass(frozen=True)
class Workload:
    name: str
    model: ChannelModel
    dtype: torch.dtype
    B: int
    T: int
    method: str = "jacpcg"
    snr_db: float = 10.0
    variant: str = "textbook"
    snr_grid_db: tuple = field(default=())
    chunk: int | None = None

    @property
    def M(self):
        return self.model.M

    @property
    def K(self):
        return self.model.K

    def power(self, snr_db=None):
        return 10.0 ** ((self.snr_db if snr_db is None else snr_db) / 10.0)

    def alpha(self, snr_db=None):
        return self.K / self.power(snr_db)


CONFIGS = {
    # configs[0]: CPU-oracle case, complex128, 100 realizations
    "cfg1": Workload("cfg1", ChannelModel(S=4, K=16, p=0.5, r=0.5), torch.complex128, 100, 4),
    # configs[1]: SNR sweep -10..20 dB, T in {2..5}, vs CG and direct
    "cfg2": Workload("cfg2", ChannelModel(S=4, K=32, p=0.5, r=0.5), torch.complex64, 8192, 4,
                     snr_grid_db=(-10.0, -5.0, 0.0, 5.0, 10.0, 15.0, 20.0)),
    # configs[2]: the headline (>= 60% of roofline target)
    "cfg3": Workload("cfg3", ChannelModel(S=16, K=64, p=0.4, r=0.7), torch.complex64, 32768, 4),
    # configs[3]: generated on device in chunks of 2048 per GPU
    "cfg4": Workload("cfg4", ChannelModel(S=64, K=128, p=0.3, r=0.5), torch.complex64, 65536, 5,
                     chunk=2048),
    # configs[4]: large K (cluster solver), c64 and c128, ill-conditioned
    "cfg5": Workload("cfg5", ChannelModel(S=32, K=256, p=0.5, r=0.9), torch.complex64, 8192, 6),
    "cfg5_c128": Workload("cfg5_c128", ChannelModel(S=32, K=256, p=0.5, r=0.9), torch.complex128,
                          8192, 6),
}
