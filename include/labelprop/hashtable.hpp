// Drop-in subset of /root/reference/proj/include/labelprop/hashtable.hpp:
// the probe-strategy enum that LpaConfig carries (hashtable.hpp:25) and the
// empty-slot sentinel (hashtable.hpp:16). The tables themselves live on the
// device (paper_2411_11468_b200/csrc/device.cuh).
#pragma once

#include <cstdint>
#include <optional>
#include <string_view>

namespace labelprop {

inline constexpr std::uint32_t kEmptyKey = 0xFFFFFFFFu;

enum class ProbeStrategy { Linear, Quadratic, DoubleHash, QuadraticDouble };

inline const char* to_string(ProbeStrategy s) {
  switch (s) {
    case ProbeStrategy::Linear: return "linear";
    case ProbeStrategy::Quadratic: return "quadratic";
    case ProbeStrategy::DoubleHash: return "double";
    case ProbeStrategy::QuadraticDouble: return "quadratic-double";
  }
  return "?";
}

inline std::optional<ProbeStrategy> parse_probe_strategy(std::string_view s) {
  for (ProbeStrategy p : {ProbeStrategy::Linear, ProbeStrategy::Quadratic,
                          ProbeStrategy::DoubleHash, ProbeStrategy::QuadraticDouble})
    if (s == to_string(p)) return p;
  return std::nullopt;
}

}  // namespace labelprop
