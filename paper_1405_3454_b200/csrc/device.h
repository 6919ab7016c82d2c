// device.h — per-device launch-configuration caches (not part of the ABI).
#pragma once

#include <mutex>

namespace cudapre {

int device_sm_count();   // SM count of the CURRENT device (cached per device)
int current_device();    // cudaGetDevice (0 if it fails)

// Launch-configuration caches (function attributes, occupancy-derived grid
// caps) are per device: one process may drive several GPUs, and concurrent
// first calls must not race.  per_device(flags, vals, f) runs f() once per
// device (std::call_once) and returns its cached value.
constexpr int kMaxDevices = 64;
template <class F>
int per_device(std::once_flag (&flags)[kMaxDevices], int (&vals)[kMaxDevices], F&& f) {
    const int d = current_device();
    if (d < 0 || d >= kMaxDevices) return f();
    std::call_once(flags[d], [&] { vals[d] = f(); });
    return vals[d];
}

}  // namespace cudapre
