// warp_emu.h — host-side lockstep emulation of the handful of warp intrinsics
// used by mpf_warp.cuh, so the warp-cooperative multiprecision primitives can be
// unit-tested on a CPU-only machine (tools/emu_mp.cpp, tests/test_emu_mp.py).
//
// Each of the 32 lanes is a std::thread; every collective (ballot / shuffle /
// syncwarp) is a pair of barrier phases over a shared slot array, which is the
// same lockstep contract `__ballot_sync(0xffffffff, …)` gives on the device.
// This is test infrastructure for the device code; the product never runs it.
#pragma once

#include <barrier>
#include <cstdint>
#include <functional>
#include <thread>
#include <vector>

namespace hk_emu {

struct Warp {
    std::barrier<> bar{32};
    uint32_t slot[32];
};

inline Warp*& cur_warp() {
    static Warp* w = nullptr;
    return w;
}
inline int& cur_lane() {
    thread_local int l = 0;
    return l;
}

inline uint32_t ballot(bool p) {
    Warp& w = *cur_warp();
    w.slot[cur_lane()] = p ? 1u : 0u;
    w.bar.arrive_and_wait();
    uint32_t m = 0;
    for (int i = 0; i < 32; ++i) m |= (w.slot[i] & 1u) << i;
    w.bar.arrive_and_wait();
    return m;
}

inline uint32_t shfl(uint32_t v, int src) {
    Warp& w = *cur_warp();
    w.slot[cur_lane()] = v;
    w.bar.arrive_and_wait();
    const uint32_t r = w.slot[src & 31];
    w.bar.arrive_and_wait();
    return r;
}

inline uint32_t shfl_down(uint32_t v, int d) {
    Warp& w = *cur_warp();
    const int l = cur_lane();
    w.slot[l] = v;
    w.bar.arrive_and_wait();
    const uint32_t r = l + d < 32 ? w.slot[l + d] : v;
    w.bar.arrive_and_wait();
    return r;
}

inline uint32_t shfl_up(uint32_t v, int d) {
    Warp& w = *cur_warp();
    const int l = cur_lane();
    w.slot[l] = v;
    w.bar.arrive_and_wait();
    const uint32_t r = l >= d ? w.slot[l - d] : v;
    w.bar.arrive_and_wait();
    return r;
}

inline void syncwarp() { cur_warp()->bar.arrive_and_wait(); }

// Run `body` on 32 emulated lanes in lockstep.
inline void run_warp(const std::function<void()>& body) {
    Warp w;
    cur_warp() = &w;
    std::vector<std::thread> th;
    th.reserve(32);
    for (int l = 0; l < 32; ++l)
        th.emplace_back([&, l] {
            cur_lane() = l;
            body();
        });
    for (auto& t : th) t.join();
    cur_warp() = nullptr;
}

} // namespace hk_emu
