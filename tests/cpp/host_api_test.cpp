// Host-side checks of the C++ layer (include/zcomm_b200.hpp) over libzcomm_b200.so, no GPU needed:
// the reference's exception types and the reference unit tests' host-visible known answers.
// Built and run by tests/test_cpu_cpp.py.
#include <cstdio>
#include <cstring>
#include <stdexcept>

#include "zcomm_b200.hpp"

using namespace zcomm::b200;

static int fails = 0;
#define EXPECT(c)                                                  \
  do {                                                             \
    if (!(c)) {                                                    \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);     \
      ++fails;                                                     \
    }                                                              \
  } while (0)

template <class E, class F>
static bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

int main() {
  // frame.cpp:35-69 (test_frame.cpp:13-76)
  FrameHeader h = make_header(ZC_CODEC_FIXEDLEN, 64, 16, 3);
  uint8_t buf[32];
  write_header(h, buf, sizeof buf);
  auto p = parse_header(buf, sizeof buf);
  EXPECT(p && std::memcmp(&*p, &h, sizeof h) == 0);
  EXPECT(!parse_header(buf, 31));
  EXPECT(throws<std::invalid_argument>([&] { write_header(h, buf, 16); }));
  EXPECT(validate_header(h, 48));
  FrameHeader bad = h;
  bad.magic ^= 1;
  EXPECT(!validate_header(bad, 48));

  // rea.cpp:240-279 (test_rea.cpp:356-398)
  ArbitrationConfig cfg = default_arbitration_config();
  load_arbitration_config("min_gain_permil = 75 # c\nembed_codebook = true\nhuffman_enc_bps = 2e11\n", cfg);
  EXPECT(cfg.min_gain_permil == 75 && cfg.embed_codebook == 1 && cfg.cost.huffman.enc_bytes_per_sec == 2e11);
  EXPECT(throws<std::invalid_argument>([&] { load_arbitration_config("vibe = 9\n", cfg); }));
  EXPECT(throws<std::invalid_argument>([&] { load_arbitration_config("embed_codebook = maybe\n", cfg); }));

  // huffman.cpp:23-214 (test_huffman.cpp:55-94)
  uint64_t hist[256] = {};
  hist[42] = 1000;
  auto c1 = HuffmanContext::build(hist);
  EXPECT(c1.valid() && c1.code_lengths()[42] == 1);
  std::memset(hist, 0, sizeof hist);
  hist[0] = 500;
  hist[255] = 500;
  auto c2 = HuffmanContext::build(hist);
  EXPECT(c2.code_lengths()[0] == 1 && c2.code_lengths()[255] == 1);
  EXPECT(c2.expected_code_len(hist).value_or(-1) == 1.0);
  EXPECT(huffman_self_code_len(hist).value_or(-1) == 1.0);
  uint64_t zero[256] = {};
  EXPECT(!HuffmanContext::build(zero).valid());
  EXPECT(!huffman_self_code_len(zero));
  uint8_t lens[256] = {1, 1, 1};
  EXPECT(!HuffmanContext::from_lengths(lens));

  // selector (rea.cpp:120-176): a FixedLen-friendly profile at a thin pipe, RAW at a fat one
  SampleStats st{};
  st.sampled_bytes = 65536;
  st.max_zigzag = 4000;  // width 12
  for (int i = 0; i < 256; ++i) st.hist[i] = 256;
  TransportHint thin = default_transport_hint(), fat = default_transport_hint();
  fat.beta_eff_bytes_per_sec = 900e9;
  ArbitrationConfig dc = default_arbitration_config();
  EXPECT(predict_payload(ZC_CODEC_FIXEDLEN, 4 << 20, st, dc) == (uint64_t)((1u << 20) * 12 / 8));
  EXPECT(arbitrate_plan(4 << 20, ZC_STAGE_BANK_BYTES, st, thin, nullptr, dc).choice == ZC_CODEC_FIXEDLEN);
  EXPECT(arbitrate_plan(4 << 20, ZC_STAGE_BANK_BYTES, st, fat, nullptr, dc).choice == ZC_CODEC_RAW);

  std::printf("%s (%d failures)\n", fails ? "FAILED" : "OK", fails);
  return fails ? 1 : 0;
}
