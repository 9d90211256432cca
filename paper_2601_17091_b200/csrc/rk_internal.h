// rk_internal.h — symbols shared between the library's translation units
// (not part of the public C ABI in include/rocket_b200.h).
#pragma once

extern "C" {
// Set the thread-local last error (rk_last_error) and return code.
int rk_set_error(int code, const char* message);
// Free the streaming runtime's cached pinned rings (rk_release_caches).
void rk_stream_release(void);
}
