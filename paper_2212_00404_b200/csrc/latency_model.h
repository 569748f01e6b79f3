// latency_model.h — PAPER.md §2.2 "latency hiding" model (P:135-200,
// Table 1) with a device profile; SURVEY §8(f) NEXT-4.
//
//   N_FMA = latency x FMA lanes per SM           (method 1: keep the FMA units
//                                                 busy with >= N_FMA FMAs per SM
//                                                 for the current data set)
//   V     = bytes per clock x latency            (method 2: keep >= V_s bytes
//   threads/SM = ceil(V / (4 N_sm N_cores)) N_cores   in flight; one 4-B word
//   V_s   = threads/SM x 4 x N_sm                 per thread)
//
// The paper counts "2 FMA operations ... in one clock cycle in each core"
// — one FMA is two flops (reading Q15 in DESIGN.md); its
// Table-1 numbers are reproduced with that factor (fma_per_lane_clk = 2),
// the B200 profile uses the hardware's 1 FMA per lane per clock.
#pragma once
#include <cmath>

namespace b200 {

struct DeviceProfile {
    double latency_clk;        // global-memory latency (clocks)
    double lanes_per_sm;       // FP32 cores per SM (N_cores)
    double fma_per_lane_clk;   // FMAs per core per clock as the model counts them
    double bytes_per_clk;      // chip DRAM bandwidth / core clock
    int num_sms;               // N_sm
};

// GTX 1080Ti, Table 1: 258-clk latency, 484 GB/s at 1480 MHz (327 B/clk), 28 SMs x 128 cores
constexpr DeviceProfile kGtx1080Ti = {258.0, 128.0, 2.0, 327.0, 28};

// B200: 577-clk DRAM latency (B300_MICROARCH.md, MLP = 1), 128 FP32 lanes,
// measured 6554 GB/s (MEASURED_PEAKS.json) at 1965 MHz = 3335 B/clk
inline DeviceProfile b200_profile(int num_sms) { return {577.0, 128.0, 1.0, 6554.0e9 / 1965.0e6, num_sms}; }

struct LatencyModel {
    double n_fma;              // FMAs per SM per data set to hide the latency (method 1)
    double volume;             // bytes in flight to cover the latency (bytes/clk x latency)
    int threads_per_sm;        // 4-B loading threads per SM for that volume (rounded to N_cores)
    double v_s;                // minimum volume those threads move (method 2)
};

inline LatencyModel latency_model(const DeviceProfile &d) {
    LatencyModel m;
    m.n_fma = d.latency_clk * d.lanes_per_sm * d.fma_per_lane_clk;
    m.volume = std::floor(d.bytes_per_clk * d.latency_clk);
    const double per_sm = m.volume / (4.0 * d.num_sms);
    m.threads_per_sm = (int)(std::ceil(per_sm / d.lanes_per_sm) * d.lanes_per_sm);
    m.v_s = (double)m.threads_per_sm * 4.0 * d.num_sms;
    return m;
}

// the paper's step 3 / 4: method 1 (prefetch) when the data set
// assigned to an SM carries >= N_FMA FMAs, else method 2 (volume)
inline int paper_method(const LatencyModel &m, double fma_per_sm) { return fma_per_sm >= m.n_fma ? 1 : 2; }

}  // namespace b200
