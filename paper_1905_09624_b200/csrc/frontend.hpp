// File front ends: FASTA batch query with the CLI's TSV output, and document
// ingestion for builds (see frontend.cpp).
#pragma once

#include <string>
#include <vector>

#include "host.hpp"

namespace cobsg {

struct DeviceIndex;

constexpr int kFormatAuto = 0, kFormatFasta = 1, kFormatText = 2; // termizer.hpp:43-47

// Regular files named by `inputs` (directories expand to every regular file
// below them, in path order): cli.cpp:60-82.
std::vector<std::string> expand_inputs(const std::vector<std::string>& inputs);
std::string doc_name_from_path(const std::string& path);

// `cobs query idx -F queries.fa`: the batch output of cli.cpp:205-221.
std::string query_fasta_tsv(DeviceIndex& ix, const std::string& fasta_path, double K, uint64_t top_t);
// `cobs build inputs... --mode classic|compact --format ...`: cli.cpp:112-166.
std::vector<uint8_t> build_from_files(const std::vector<std::string>& inputs, const Params& params,
                                      uint8_t kind, int format, int device);

} // namespace cobsg
