// zc_huffman_host.hpp — canonical Huffman context construction (host side).
//
// Mirrors huffman_build_context / huffman_context_from_lengths / huffman_expected_code_len /
// huffman_self_code_len (huffman.cpp:23-214; paths relative to /root/reference/proj/core/).
// The shared context is built once per communicator (collectives.cpp:92-106), so this runs on
// the host and the tables are uploaded to HBM as a zc::DevHuff.
#pragma once
#include <array>
#include <cstdint>
#include <optional>

#include "zc_common.cuh"

namespace zc {

struct HostHuff {
  bool valid = false;
  std::array<uint8_t, 256> len{};
  std::array<uint32_t, 256> code{};
  std::array<uint32_t, 256> rev{};
  std::array<uint8_t, 256> sym_order{};
  std::array<uint32_t, 33> count_at_len{};
  std::array<uint64_t, 33> first_code{};
  std::array<uint32_t, 33> first_index{};
  std::array<uint16_t, 4096> lut{};
  uint32_t min_len = 0, max_len = 0;
};

// Code lengths of the reference's pairwise merge followed by the 32-bit cap repair.
void huffman_lengths(const uint64_t* hist256, std::array<uint8_t, 256>& lens);
// Canonical tables from lengths; nullopt on an invalid (empty / over-long / non-Kraft) set.
std::optional<HostHuff> huffman_finalize(const std::array<uint8_t, 256>& lens);
HostHuff huffman_build(const uint64_t* hist256);
std::optional<double> huffman_expected_len(const HostHuff& c, const uint64_t* hist256);
std::optional<double> huffman_self_len(const uint64_t* hist256);
void to_device_layout(const HostHuff& h, DevHuff& d);

}  // namespace zc
