// prpipe drop-in: K1 (API of include/prpipe/kernel1_sort.hpp:10-25).
// sort_edges reads the shards on the host, sorts on the B200 (C-ABI
// prg_k1_sort_host) and writes the sorted shards. Ties are ordered by v — one
// of the orders the reference allows ("no particular end-vertex order"). The
// device sort holds any input that fits in HBM, so the external merge sort of
// the reference (memory_budget_bytes) is never needed; the options are accepted.
#pragma once

#include <cstdint>
#include <filesystem>

#include "prpipe/edge_io.hpp"

namespace prpipe {

struct SortOptions {
    std::int64_t memory_budget_bytes = 0;
    int num_files = 0;
    int merge_fan_in = 64;
    std::filesystem::path spill_dir;
};

std::int64_t default_memory_budget();

EdgeManifest sort_edges(const EdgeManifest& input, const std::filesystem::path& output_dir,
                        const SortOptions& options = {});

// Seconds spent in the last sort_edges call: host TSV read / device sort incl.
// transfers / host TSV write (the reference reports only their sum).
struct SortBreakdown {
    double read_s = 0, device_s = 0, write_s = 0;
};
SortBreakdown last_sort_breakdown();

}  // namespace prpipe
