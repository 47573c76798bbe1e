// Kernel 4 driver: device index construction (see build.cu).
#pragma once

#include <string>
#include <vector>

#include <memory>

#include "host.hpp"

namespace cobsg {

struct BuildTiming {
    double ms_h2d = 0, ms_count = 0, ms_fill = 0, ms_d2h = 0, ms_total = 0;
    uint32_t count_waves = 0, count_fallback_waves = 0; // partitioned count: waves, recounted waves
    double ms_count_alloc = 0; // host time of the partitioned count's buffer allocation (debug)
    double ms_count_sync = 0, ms_count_free = 0; // host: count start -> kernels done, key buffer frees (debug)
    double ms_count_kernels = 0; // the count's kernels alone (CUDA events: after the buffer allocation, before the frees)
};
const BuildTiming& last_build_timing();

// extract_terms + build_classic / build_compact + the writer's byte layout:
// returns the complete file image.
std::vector<uint8_t> build_index(const uint8_t* seqs, const uint64_t* seg_off, uint64_t n_segs,
                                 const uint64_t* doc_segs, const std::vector<std::string>& names,
                                 const Params& params, uint8_t kind, uint64_t forced_w, int device);
// The same build, leaving the index resident in HBM (pitched, ready to
// query); `seqs` may be a device pointer (seqs_on_device).  seg_off and
// doc_segs are host arrays.  terms_input: every segment is one pre-extracted
// term (a TermSet entry), hashed as given.
struct DeviceIndex;
std::unique_ptr<DeviceIndex> build_device_index(const uint8_t* seqs, const uint64_t* seg_off,
                                                uint64_t n_segs, const uint64_t* doc_segs,
                                                const std::vector<std::string>& names, const Params& P,
                                                uint8_t kind, uint64_t forced_w, int device,
                                                bool seqs_on_device, bool terms_input = false,
                                                bool seg_ptrs = false);
// File image (header + un-pitched payload) of a device-resident index.
std::vector<uint8_t> index_image(const DeviceIndex& ix);
// The same into caller memory of index_image_size() bytes (no zero fill).
uint64_t index_image_size(const DeviceIndex& ix);
void index_image_into(const DeviceIndex& ix, uint8_t* dst);
// Record the image leg of the last build (ms_d2h, added to ms_total).
void note_image_ms(double ms);
void write_image(const std::vector<uint8_t>& image, const std::string& path);
void write_image(const uint8_t* image, uint64_t size, const std::string& path);

void synth_docs(uint64_t seed, int alpha, const uint64_t* doc_len, uint64_t doc_lo, uint64_t doc_hi,
                uint8_t* dev_out, int device);

} // namespace cobsg
