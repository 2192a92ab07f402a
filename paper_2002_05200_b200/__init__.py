"""B200-native batched X-drop seed-and-extend (LOGAN, arXiv 2002.05200).

The product is the C-ABI library ``liblogan_xdrop.so`` (sm_100a CUDA, header
``include/logan_xdrop.h``); this package is its thin binding plus the
multi-GPU driver.  PyTorch provides device memory, streams and process
groups only.
"""
from . import _lib
from ._lib import LOGAN_SEQ_2BIT, LOGAN_SEQ_U8, LoganError
from .api import (DeviceBatch, HostArena, clear_workspace_cache, make_workspace, new_stats, pack_2bit,
                  stats_dict, to_device, workspace_bytes, xdrop_batch, xdrop_batch_host)

__all__ = ["LOGAN_SEQ_2BIT", "LOGAN_SEQ_U8", "LoganError", "DeviceBatch", "HostArena",
           "clear_workspace_cache", "make_workspace", "new_stats", "pack_2bit", "stats_dict", "to_device", "workspace_bytes",
           "xdrop_batch", "xdrop_batch_host", "_lib"]
