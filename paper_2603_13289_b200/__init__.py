"""relaykv-b200: B200-native RelayCaching relay-prefill engine (placeholder)."""
