// zc_huffman_host.cpp — see zc_huffman_host.hpp.
#include "zc_huffman_host.hpp"

#include <algorithm>
#include <cstring>
#include <vector>

namespace zc {

// Pairwise merge (huffman.cpp:23-68) done as the classic two-queue construction.  The reference
// picks the live node with the least (weight, creation order); leaves are created first, in
// ascending symbol order, and merged nodes are created afterwards with non-decreasing weights.
// So the leaf queue sorted by (weight, symbol) and the merged-node queue in creation order are
// each sorted by (weight, order), and taking the smaller head (a leaf wins a weight tie, since
// every leaf's order precedes every merged node's) reproduces the reference's exact pick sequence
// — and with it the exact length multiset, which canonicalisation does NOT make tie-independent.
void huffman_lengths(const uint64_t* freq, std::array<uint8_t, 256>& lens) {
  lens.fill(0);
  std::vector<int> leaves;
  for (int s = 0; s < 256; ++s)
    if (freq[s] > 0) leaves.push_back(s);
  if (leaves.empty()) return;
  if (leaves.size() == 1) {
    lens[leaves[0]] = 1;  // degenerate input still gets 1 bit (huffman.cpp:35-38)
    return;
  }
  std::stable_sort(leaves.begin(), leaves.end(), [&](int a, int b) { return freq[a] < freq[b]; });
  const int L = static_cast<int>(leaves.size());
  // Node ids: 0..L-1 leaves (in sorted order), L.. merged nodes.
  std::vector<uint64_t> w(2 * L);
  std::vector<int> parent(2 * L, -1);
  for (int i = 0; i < L; ++i) w[i] = freq[leaves[i]];
  int li = 0, mi = L, next = L;
  auto take = [&]() {
    // leaf head wins ties against merged head
    if (li < L && (mi >= next || w[li] <= w[mi])) return li++;
    return mi++;
  };
  while (next < 2 * L - 1) {
    int a = take();
    int b = take();
    w[next] = w[a] + w[b];
    parent[a] = parent[b] = next;
    ++next;
  }
  for (int i = 0; i < L; ++i) {
    unsigned d = 0;
    for (int p = parent[i]; p >= 0; p = parent[p]) ++d;
    lens[leaves[i]] = static_cast<uint8_t>(std::min(d, 255u));
  }
  // Length cap with Kraft repair (huffman.cpp:72-95): clamp to 32, then while over-full deepen
  // the deepest leaf still below the cap (highest symbol among equals).
  constexpr unsigned cap = ZC_HUFF_MAX_CODE_LEN;
  uint64_t kraft = 0;
  for (auto& l : lens) {
    if (!l) continue;
    if (l > cap) l = cap;
    kraft += 1ull << (cap - l);
  }
  while (kraft > (1ull << cap)) {
    int pick = -1;
    unsigned pl = 0;
    for (int s = 0; s < 256; ++s) {
      unsigned l = lens[s];
      if (l > 0 && l < cap && l >= pl) {
        pl = l;
        pick = s;
      }
    }
    if (pick < 0) break;
    lens[pick]++;
    kraft -= 1ull << (cap - pl - 1);
  }
}

static uint32_t reverse_bits(uint32_t v, unsigned n) {
  uint32_t r = 0;
  for (unsigned i = 0; i < n; ++i, v >>= 1) r = (r << 1) | (v & 1);
  return r;
}

// huffman.cpp:97-161 (finalize_context): canonical codes in (length, symbol) order.
std::optional<HostHuff> huffman_finalize(const std::array<uint8_t, 256>& lens) {
  HostHuff c;
  c.len = lens;
  std::array<uint32_t, 34> bl{};
  unsigned n = 0;
  for (int s = 0; s < 256; ++s) {
    unsigned l = lens[s];
    if (!l) continue;
    if (l > ZC_HUFF_MAX_CODE_LEN) return std::nullopt;
    ++bl[l];
    ++n;
    if (c.min_len == 0 || l < c.min_len) c.min_len = l;
    c.max_len = std::max(c.max_len, l);
  }
  if (!n) return std::nullopt;
  uint64_t kraft = 0;
  for (unsigned l = 1; l <= c.max_len; ++l) kraft += static_cast<uint64_t>(bl[l]) << (ZC_HUFF_MAX_CODE_LEN - l);
  if (kraft > (1ull << ZC_HUFF_MAX_CODE_LEN)) return std::nullopt;
  std::array<uint64_t, 34> next{};
  uint64_t code = 0;
  uint32_t idx = 0;
  for (unsigned l = 1; l <= c.max_len; ++l) {
    code = (code + bl[l - 1]) << 1;
    next[l] = c.first_code[l] = code;
    c.first_index[l] = idx;
    c.count_at_len[l] = bl[l];
    idx += bl[l];
  }
  std::array<uint32_t, 34> fill{};
  for (int s = 0; s < 256; ++s) {
    unsigned l = lens[s];
    if (!l) continue;
    c.code[s] = static_cast<uint32_t>(next[l]++);
    c.rev[s] = reverse_bits(c.code[s], l);
    c.sym_order[c.first_index[l] + fill[l]++] = static_cast<uint8_t>(s);
  }
  for (int s = 0; s < 256; ++s) {
    unsigned l = lens[s];
    if (!l || l > ZC_HUFF_ROOT_BITS) continue;
    uint16_t e = static_cast<uint16_t>(s | (l << 8));
    for (uint32_t pad = 0; pad < (1u << (ZC_HUFF_ROOT_BITS - l)); ++pad) c.lut[c.rev[s] | (pad << l)] = e;
  }
  c.valid = true;
  return c;
}

HostHuff huffman_build(const uint64_t* hist) {
  std::array<uint8_t, 256> lens;
  huffman_lengths(hist, lens);
  auto c = huffman_finalize(lens);
  return c ? *c : HostHuff{};
}

// huffman.cpp:200-214.  Every f*len term is an exact integer below 2^53 and so is every partial
// sum, so integer accumulation then one conversion equals the reference's double accumulation.
static std::optional<double> mean_len(const std::array<uint8_t, 256>& lens, const uint64_t* hist) {
  uint64_t total = 0, bits = 0;
  for (int s = 0; s < 256; ++s) {
    uint64_t f = hist[s];
    if (!f) continue;
    if (!lens[s]) return std::nullopt;
    total += f;
    bits += f * lens[s];
  }
  if (!total) return std::nullopt;
  return static_cast<double>(bits) / static_cast<double>(total);
}

std::optional<double> huffman_expected_len(const HostHuff& c, const uint64_t* hist) {
  if (!c.valid) return std::nullopt;
  return mean_len(c.len, hist);
}

std::optional<double> huffman_self_len(const uint64_t* hist) {
  std::array<uint8_t, 256> lens;
  huffman_lengths(hist, lens);
  return mean_len(lens, hist);
}

void to_device_layout(const HostHuff& h, DevHuff& d) {
  std::memset(&d, 0, sizeof(d));
  d.valid = h.valid ? 1u : 0u;
  d.min_len = h.min_len;
  d.max_len = h.max_len;
  for (int s = 0; s < 256; ++s) {
    d.enc[s] = static_cast<uint64_t>(h.rev[s]) | (static_cast<uint64_t>(h.len[s]) << 32);
    d.len[s] = h.len[s];
    d.sym_order[s] = h.sym_order[s];
  }
  for (int l = 0; l < 33; ++l) {
    d.count_at_len[l] = h.count_at_len[l];
    d.first_index[l] = h.first_index[l];
    d.first_code[l] = h.first_code[l];
  }
  std::memcpy(d.lut, h.lut.data(), sizeof(d.lut));
}

}  // namespace zc
