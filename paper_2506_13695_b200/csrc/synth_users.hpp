// Seeded synthetic user generator shared by the engine (orx::Rng) and the
// oracle driver (genrec::Rng). Both Rng types implement xoshiro256** with the
// same split(), so the same (seed, user index) yields bit-identical records.
//
// Follows the fixture pattern of the reference tests (record()/tiny_context(),
// proj/tests/test_policy.cpp:34-58) at paper lengths, as SURVEY.md §8(d) states:
//   uid ~ U[0,2^20), gender ~ U{0,1,2}, age ~ U{0..7};
//   lifelong, then positive, then short records, ts strictly ascending (step 0.01);
//   vid ~ U[0,2^20), aid ~ U[0,1e5), tag ~ U[0,1), duration ~ U[0.05,1),
//   playtime = duration * U[0,1), labels ~ U[0,32).
#pragma once

#include <cstdint>

namespace orx_synth {

struct Lengths {
  int n_short = 20;
  int n_positive = 256;
  int n_lifelong = 2000;
};

// Record sink signature: (pathway 0=short 1=positive 2=lifelong, vid, aid,
// tag, ts, playtime, duration, labels).
template <class RngT, class Sink, class HeaderSink>
void synth_user(uint64_t seed, uint64_t user_index, const Lengths& len, HeaderSink&& header,
                Sink&& emit) {
  RngT base(seed);
  RngT rng = base.split(user_index);
  int uid = static_cast<int>(rng.randint(int64_t(1) << 20));
  int gender = static_cast<int>(rng.randint(3));
  int age = static_cast<int>(rng.randint(8));
  header(uid, gender, age);
  int total = len.n_short + len.n_positive + len.n_lifelong;
  double ts = -0.01 * total;
  auto record = [&](int pathway) {
    int64_t vid = rng.randint(int64_t(1) << 20);
    int aid = static_cast<int>(rng.randint(100000));
    double tag = rng.uniform();
    double duration = rng.uniform(0.05, 1.0);
    double playtime = duration * rng.uniform();
    uint32_t labels = static_cast<uint32_t>(rng.randint(32));
    ts += 0.01;
    emit(pathway, vid, aid, tag, ts, playtime, duration, labels);
  };
  for (int i = 0; i < len.n_lifelong; ++i) record(2);
  for (int i = 0; i < len.n_positive; ++i) record(1);
  for (int i = 0; i < len.n_short; ++i) record(0);
}

}  // namespace orx_synth
