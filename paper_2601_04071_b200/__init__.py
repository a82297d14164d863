"""microslice-b200: B200-native SLO-oriented preemptive GPU scheduler (arXiv 2601.04071).

Product layers (all native; Python is orchestration only):
  include/microslice/*.hpp  C++ drop-in of the reference scheduler API
  lib/libmicroslice.so      scheduler core + replay device (C-ABI: include/ms_replay.h)
  lib/libms_b200.so         sm_100a preemptible tenant kernels, flag/doorbell device layer,
                            live runtime (C-ABI: include/ms_b200.h)
"""
__version__ = "0.1.0"
