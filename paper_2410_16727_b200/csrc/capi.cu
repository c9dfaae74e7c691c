// Library identification for the C-ABI (include/ps_b200.h).
#include "common.cuh"

extern "C" const char* ps_version(void) { return "ps_b200 0.1 sm_100a"; }

extern "C" long long ps_launch_count(void) { return ps_launch_counter().load(); }
