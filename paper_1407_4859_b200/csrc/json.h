// json.h -- minimal JSON value, parser and writer for the planner's inputs/outputs
// (SPEC.md:100 UTF-8 JSON; 313 plan serialisation).  Not on the remap path.
#pragma once

#include <cstdint>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace adha {
namespace json {

struct ParseError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

struct Value {
    enum Kind { Null, Bool, Number, String, Array, Object } kind = Null;
    bool b = false;
    double num = 0.0;
    std::string str;
    std::vector<Value> arr;
    std::vector<std::pair<std::string, Value>> obj;   // insertion order kept

    bool has(const std::string& k) const;
    const Value& at(const std::string& k) const;      // throws ParseError if absent
    const Value* find(const std::string& k) const;
    double as_num() const;
    const std::string& as_str() const;
    bool as_bool() const;
    const std::vector<Value>& as_arr() const;
};

Value parse(const std::string& text);

// writer
std::string quote(const std::string& s);
std::string number(double v);   // shortest round-trip representation

}  // namespace json
}  // namespace adha
