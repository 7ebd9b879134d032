// Artifact files of the reference (inc/io.hpp): JSON / JSON Lines with format_version 1, read and
// written here without a JSON library, plus a binary trace container for fast loading of
// Mixtral-width traces (a 64-token 8x7B trace is ~200 MB of JSONL text, 67 MB binary).
//
// Error classes follow inc/io.hpp:23-37: io_error (cannot open / write) -> Status::Io;
// parse_error, schema_error, version_error -> Status::Format.  Messages carry the path (and the
// line for JSON Lines), like the reference's.
#pragma once

#include <cstdint>
#include <optional>
#include <string>
#include <vector>

#include "policy.hpp"

namespace adapmoe {

constexpr int kFormatVersion = 1;  // inc/io.hpp:21

struct TraceData {  // inc/io.hpp:146 TraceFile, flattened
    ModelSpec spec;
    int tokens = 0;
    std::vector<int> token_index;     // [T]
    std::vector<double> activations;  // [T][L][d]
    std::vector<double> scores;       // [T][L][N]
    std::vector<int> selected;        // [T][L][K] (-1 padded)
    std::vector<int> selected_count;  // [T][L]
    // ragged inputs (wrong layer count / widths) are kept as found so validate_trace can report them
    std::vector<std::string> shape_violations;
};

// JSON Lines (reference) or binary (magic "MOETRB1") by content.
TraceData load_trace_file(const std::string& path);
void save_trace_jsonl(const std::string& path, const TraceData& t);   // inc/io.hpp:127 save_trace
void save_trace_binary(const std::string& path, const TraceData& t);
// validate_trace (inc/core.hpp:249-297): violation messages (empty = valid)
std::vector<std::string> validate_trace(const TraceData& t);

struct GatesData {  // inc/io.hpp:227 GatesFile
    ModelSpec spec;
    std::vector<double> gates;             // [L][d][N]
    std::optional<std::vector<double>> first_gate;  // [d][N]
    double learning_rate = 0.0;
    int steps = 0;
    std::uint64_t seed = 0;
};
GatesData load_gates_file(const std::string& path);
void save_gates_file(const std::string& path, const GatesData& g);

struct ProfilesData {  // inc/io.hpp:271 ProfilesFile
    ModelSpec spec;
    std::vector<double> alpha, beta, fisher;  // single_expert_prob, prefetch_accuracy, fisher_diag_sum
};
ProfilesData load_profiles_file(const std::string& path);
void save_profiles_file(const std::string& path, const ProfilesData& p);
std::string profile_hash(const ProfilesData& p);  // inc/io.hpp:290 (FNV-1a of the compact dump)

struct ThresholdData {  // inc/io.hpp:300
    double tau = 0.0, target_single_ratio = 0.0, realized_single_ratio = 0.0;
};
ThresholdData load_threshold_file(const std::string& path);
void save_threshold_file(const std::string& path, const ThresholdData& t);

struct AllocationData {  // inc/io.hpp:326
    int budget = 0;
    std::vector<int> capacities;
    double total_cost = 0.0;
    std::string profile_hash;
};
AllocationData load_allocation_file(const std::string& path);
void save_allocation_file(const std::string& path, const AllocationData& a);

struct CostTableData {  // inc/io.hpp:356
    int experts_per_layer = 0;
    std::vector<std::vector<double>> loads;  // [L][N+1]
};
CostTableData load_cost_table_file(const std::string& path);
void save_cost_table_file(const std::string& path, const CostTableData& c);

}  // namespace adapmoe
