"""B200-native IOS stage executor (arXiv 2011.01302): libios.so (C-ABI, include/ios.h) + a thin
ctypes binding. See DESIGN.md."""
from .ios import (Graph, Schedule, IOSError, CONCURRENT, MERGE, ios_graph_create, ios_add_op,  # noqa: F401
                  ios_stage_latency, ios_schedule_dp, ios_run, ios_last_error, LIB_PATH)
