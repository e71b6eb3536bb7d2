// internal.h — hooks shared between libsattn.so translation units (not part of the C ABI).
#pragma once
#include "sattn.h"

namespace sattn {
sattn_status set_error(sattn_status st, const char* msg);   // sets sattn_last_error(), returns st
sattn_status check_desc(const sattn_desc* d);                // synchronous desc validation
void count_launches(int n);                                  // sattn_launch_count bookkeeping
float desc_scale(const sattn_desc* d);                       // effective score scale
}  // namespace sattn
