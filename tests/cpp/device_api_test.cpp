// Device-side checks of the C++ layer (include/zcomm_b200.hpp) on a GPU: the coder plugins
// (fixedlen.hpp:22-42, huffman.hpp:38-70), profile_sample (rea.cpp:93-118), frame_commit_raw
// (frame.cpp:52-58), and a single-process LocalCommunicator::run with RankCtx::send_encoded /
// recv_decoded and collectives from the rank threads, with the reference unit tests' known
// answers (test_fixedlen.cpp:62-133, test_collectives.cpp:83-146, 221-265).  Built and run by
// tests/test_gpu_cpp.py; needs no CUDA runtime of its own (allocation and copies go through the
// library's plumbing entry points).
#include <cstdio>
#include <cstring>
#include <random>
#include <stdexcept>
#include <vector>

#include "zcomm_b200.hpp"

using namespace zcomm::b200;

static int fails = 0;
#define EXPECT(c)                                              \
  do {                                                         \
    if (!(c)) {                                                \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c); \
      ++fails;                                                 \
    }                                                          \
  } while (0)

template <class T>
struct DevBuf {  // device copy of a host vector
  explicit DevBuf(size_t n) : n(n), s(n * sizeof(T) + 16) { check(zc_memset(s.as<void>(), 0, n * sizeof(T) + 16)); }
  explicit DevBuf(const std::vector<T>& h) : DevBuf(h.size()) { check(zc_memcpy(ptr(), h.data(), h.size() * sizeof(T))); }
  T* ptr() const { return s.as<T>(); }
  std::vector<T> host() const {
    std::vector<T> h(n);
    check(zc_memcpy(h.data(), ptr(), n * sizeof(T)));
    return h;
  }
  size_t n;
  DeviceScratch s;
};

static uint32_t zz(int32_t v) { return (static_cast<uint32_t>(v) << 1) ^ static_cast<uint32_t>(v >> 31); }

static std::vector<uint8_t> naive_pack(const std::vector<int32_t>& syms, unsigned w) {
  std::vector<uint8_t> out((syms.size() * w + 7) / 8, 0);
  size_t bit = 0;
  for (int32_t s : syms) {
    uint32_t z = zz(s);
    for (unsigned j = 0; j < w; ++j, ++bit)
      if ((z >> j) & 1) out[bit / 8] |= static_cast<uint8_t>(1u << (bit % 8));
  }
  return out;
}

int main() {
  int ndev = 0;
  if (zc_device_count(&ndev) != ZC_OK || ndev == 0) {
    std::printf("no CUDA device\n");
    return 2;
  }

  // ---- fixedlen (test_fixedlen.cpp:62-75 hand-packed example, 77-97 naive packer, 127-133)
  {
    DevBuf<int32_t> syms(std::vector<int32_t>{0, 1, -1, 2});
    DevBuf<uint8_t> out(8);
    unsigned w = 0;
    size_t payload = fixedlen_encode(syms.ptr(), 4, out.ptr(), 8, &w);
    auto o = out.host();
    EXPECT(w == 3 && payload == 2 && o[0] == 0x50 && o[1] == 0x08);
    FrameHeader h = make_header(ZC_CODEC_FIXEDLEN, 16, payload, w);
    DevBuf<int32_t> back(4);
    EXPECT(fixedlen_decode_into(h, out.ptr(), payload, reinterpret_cast<uint8_t*>(back.ptr()), 16));
    EXPECT((back.host() == std::vector<int32_t>{0, 1, -1, 2}));
    DevBuf<uint8_t> tiny(2);
    DevBuf<int32_t> three(std::vector<int32_t>{100, -200, 300});
    EXPECT(fixedlen_encode(three.ptr(), 3, tiny.ptr(), 2, &w) == 0);
  }
  {
    std::mt19937_64 rng(9);
    for (int t = 0; t < 50; ++t) {
      size_t n = 1 + rng() % 200;
      int shift = static_cast<int>(rng() % 28);
      std::vector<int32_t> hs(n);
      for (auto& s : hs) s = static_cast<int32_t>(rng() >> (32 + shift));
      unsigned wref = 1;
      uint32_t mz = 0;
      for (int32_t s : hs) mz = std::max(mz, zz(s));
      while (wref < 32 && (mz >> wref) != 0) ++wref;
      DevBuf<int32_t> syms(hs);
      DevBuf<uint8_t> out(4 * n + 8);
      unsigned w = 0;
      size_t payload = fixedlen_encode(syms.ptr(), n, out.ptr(), 4 * n + 8, &w);
      auto ref = naive_pack(hs, wref);
      auto o = out.host();
      EXPECT(w == wref && payload == ref.size() && std::equal(ref.begin(), ref.end(), o.begin()));
    }
  }

  // ---- huffman (huffman.cpp:216-316): shared-context round trip with and without the index,
  // embedded-codebook round trip without a shared context
  {
    std::mt19937_64 rng(3);
    std::vector<uint8_t> raw(1 << 20);
    for (auto& b : raw) b = static_cast<uint8_t>(std::min<uint64_t>(255, (rng() % 64) * (rng() % 4)));
    HuffmanContext ctx = HuffmanContext::from_bytes(raw.data(), raw.size());
    EXPECT(ctx.valid());
    DevBuf<uint8_t> d_raw(raw), out(2 * raw.size()), back(raw.size());
    DevBuf<uint32_t> idx(ZC_HUFF_INDEX_ENTRIES);
    for (int embed = 0; embed < 2; ++embed) {
      size_t payload = huffman_encode(d_raw.ptr(), raw.size(), ctx, out.ptr(), 2 * raw.size(), embed != 0, idx.ptr());
      EXPECT(payload > 0 && payload < raw.size());
      FrameHeader h = make_header(ZC_CODEC_HUFFMAN, raw.size(), payload, embed ? ZC_HUFF_CODEBOOK_BYTES : 0,
                                  embed ? ZC_FLAG_EMBEDDED_CODEBOOK : 0);
      check(zc_memset(back.ptr(), 0, raw.size()));
      EXPECT(huffman_decode_into(h, out.ptr(), payload, embed ? nullptr : &ctx, back.ptr(), raw.size(), idx.ptr()));
      EXPECT(back.host() == raw);
      check(zc_memset(back.ptr(), 0, raw.size()));
      EXPECT(huffman_decode_into(h, out.ptr(), payload, embed ? nullptr : &ctx, back.ptr(), raw.size(), nullptr));
      EXPECT(back.host() == raw);
    }
    // profile_sample: the window is the first 64 KiB (rea.cpp:93-118)
    SampleStats st = profile_sample(d_raw.ptr(), raw.size(), &ctx);
    EXPECT(st.sampled_bytes == ZC_SAMPLE_WINDOW_BYTES && st.ctx_code_len_valid == 1);
    EXPECT(st.ctx_code_len_bits > 0.0 && st.ctx_code_len_bits < 8.0);
    // frame_commit_raw (frame.cpp:52-58): header + verbatim payload; 0 when the region is too small
    DevBuf<uint8_t> region(64);
    DevBuf<uint8_t> small(std::vector<uint8_t>{1, 2, 3, 4, 5});
    EXPECT(frame_commit_raw(small.ptr(), 5, region.ptr(), 64) == 37);
    auto rg = region.host();
    auto ph = parse_header(rg.data(), 37);
    EXPECT(ph && ph->codec == ZC_CODEC_RAW && ph->raw_bytes == 5 && rg[32] == 1 && rg[36] == 5);
    EXPECT(frame_commit_raw(small.ptr(), 5, region.ptr(), 36) == 0);
  }

  // ---- Communicator::run on one device (test_collectives.cpp:83-94, 129-146, 221-265)
  {
    LocalCommunicator comm(2, 0, default_collective_config());
    std::mt19937_64 rng(7);
    std::vector<int32_t> src(3ull << 20);  // 12 MiB raw
    for (auto& v : src) v = static_cast<int32_t>(rng() % 100) - 50;
    DevBuf<int32_t> d_src(src), d_dst(src.size());
    comm.run([&](RankCtx& ctx) {
      if (ctx.rank() == 0)
        ctx.send_encoded(1, d_src.ptr(), 4 * src.size());
      else
        ctx.recv_decoded(0, d_dst.ptr(), 4 * src.size());
    });
    EXPECT(d_dst.host() == src);
    WireStats s = comm.wire_stats();
    EXPECT(s.frames_by_codec[ZC_CODEC_FIXEDLEN] == 3 && s.frames_by_codec[0] + s.frames_by_codec[2] == 0);
    EXPECT(s.raw_bytes == (12ull << 20) && s.payload_bytes < (12ull << 20) / 4);

    std::vector<DevBuf<int32_t>*> bufs;
    for (int r = 0; r < 2; ++r) bufs.push_back(new DevBuf<int32_t>(std::vector<int32_t>{r + 1, -(r + 1), 100}));
    comm.run([&](RankCtx& ctx) { ctx.allreduce(bufs[static_cast<size_t>(ctx.rank())]->ptr(), 3, 1.0); });
    for (auto* b : bufs) EXPECT((b->host() == std::vector<int32_t>{3, -3, 200}));
    // overflow: the root cause surfaces as std::overflow_error and the communicator survives
    for (auto* b : bufs) {
      std::vector<int32_t> big(8, 2147483647);
      check(zc_memcpy(b->ptr(), big.data(), 12));
    }
    bool threw = false;
    try {
      comm.run([&](RankCtx& ctx) { ctx.allreduce(bufs[static_cast<size_t>(ctx.rank())]->ptr(), 3, 1.0); });
    } catch (const std::overflow_error&) {
      threw = true;
    }
    EXPECT(threw);
    // a rank that throws before its part: the peer blocked on it sees the poisoned link, run
    // rethrows the root cause
    threw = false;
    try {
      comm.run([&](RankCtx& ctx) {
        if (ctx.rank() == 1) throw std::invalid_argument("rank 1 refuses");
        ctx.recv_decoded(1, d_dst.ptr(), 1 << 20);
      });
    } catch (const std::invalid_argument& e) {
      threw = std::strcmp(e.what(), "rank 1 refuses") == 0;
    }
    EXPECT(threw);
    for (int r = 0; r < 2; ++r) check(zc_memcpy(bufs[static_cast<size_t>(r)]->ptr(), std::vector<int32_t>{1, 2, 3}.data(), 12));
    comm.run([&](RankCtx& ctx) { ctx.allreduce(bufs[static_cast<size_t>(ctx.rank())]->ptr(), 3, 1.0); });
    for (auto* b : bufs) EXPECT((b->host() == std::vector<int32_t>{2, 4, 6}));
    for (auto* b : bufs) delete b;
  }

  std::printf(fails ? "FAILED %d\n" : "OK\n", fails);
  return fails ? 1 : 0;
}
