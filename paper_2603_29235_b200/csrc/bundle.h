// bundle.h — a bundle directory loaded for the analysis path (stg_bundle.cu,
// stg_bundle_host.cpp): LoadedBundle (bundle.hpp:23-42) as an stg_window whose
// bulk arrays (samples, frames, collectives) were decoded on the GPU.
#pragma once

#include <string>
#include <vector>

#include "stg_internal.h"

namespace stg {

// Decoded bulk arrays (device, in the context's buffers) + host summaries.
struct BundleBulk {
    uint64_t n_samples = 0, n_frames = 0, n_coll = 0;
    std::vector<int32_t> rank_ids;
    std::vector<uint64_t> rank_sample_off;
    std::vector<uint8_t> bin_ids;  // n_bins * 20
    const int64_t* ts = nullptr;
    const uint64_t* foff = nullptr;
    const uint64_t* pc = nullptr;
    const uint16_t* bin = nullptr;
    const int32_t *c_rank = nullptr, *c_group = nullptr;
    const uint8_t* c_kind = nullptr;
    const int64_t *c_entry = nullptr, *c_exit = nullptr, *c_dur = nullptr;
};

struct Bundle {
    BundleBulk bulk;
    std::string scenario;
    std::vector<int32_t> group_ranks;
    std::vector<int32_t> g_rank;
    std::vector<uint32_t> g_kernel;
    std::vector<int64_t> g_start, g_dur;
    std::vector<std::string> kernel_names, counter_names, base_names;
    std::vector<const char*> kernel_cstr, counter_cstr, base_cstr;
    std::vector<int32_t> o_rank;
    std::vector<int64_t> o_ws, o_p50, o_p99, o_mig, irq_v, sirq_v;
    std::vector<uint64_t> irq_off{0}, sirq_off{0};
    std::vector<uint32_t> irq_k, sirq_k;
    std::vector<double> base_fracs;
    stg_window w{};
    stg_bundle_info info{};
};

const uint8_t* upload_file(Ctx& c, const std::string& path, const std::string& tag, uint64_t& size);
void bundle_decode_samples(Ctx& c, const uint8_t* d, uint64_t size, BundleBulk& b);
void bundle_decode_collectives(Ctx& c, const uint8_t* d, uint64_t size, BundleBulk& b);
void bundle_load(Ctx& c, const std::string& dir, stg_bundle_info* info);

}  // namespace stg
